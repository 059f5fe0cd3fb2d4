"""Build the sm_100a shared library in-tree (no JIT cache, no pip install).

    python -m paper_2007_12623_b200.build        # or __graft_entry__.build()

Compiles every csrc/*.cu and csrc/*.cpp with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` into
``paper_2007_12623_b200/lib/libstereoscan_b200.so`` and the C++ API test
driver ``tests/cpp/build/test_api``. Objects are rebuilt only when a source or
header is newer. ``--fmad=false`` is load-bearing: the reference's double
arithmetic is uncontracted, and so must ours be.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libstereoscan_b200.so")          # C-ABI (include/ss_stereo.h)
LIB_CXX = os.path.join(LIB_DIR, "libstereoscan_b200_cxx.so")  # C++ drop-in API + io on it
CXX_SRCS = ("stereoscan_api.cpp", "io.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_LIB = "/usr/local/cuda/lib64"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                 "-Xcompiler", "-ffp-contract=off", f"-I{INC}", f"-I{CSRC}",
                 "-Xptxas", "-warn-spills"]


def _deps():
    return [p for p in glob.glob(os.path.join(CSRC, "*")) if p.endswith((".cuh", ".h"))] + \
        glob.glob(os.path.join(INC, "**", "*.h*"), recursive=True)


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


# Translation units whose only FP32/FP64 arithmetic outside explicit rounding
# intrinsics is tolerance-checked (the normal fit): FMA contraction allowed.
FMAD_OK = {"k_cloud.cu"}


def _compile(src):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if _newer(obj, [src] + _deps() + [__file__]):
        flags = COMMON
        if os.path.basename(src) in FMAD_OK:
            flags = [f for f in COMMON if f != "--fmad=false"] + ["--fmad=true"]
        cmd = [NVCC] + flags + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC] + flags + ["-x", "cu", "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if r.stderr.strip():
            sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, srcs))
    core = [o for o, s in zip(objs, srcs) if os.path.basename(s) not in CXX_SRCS]
    cxx = [o for o, s in zip(objs, srcs) if os.path.basename(s) in CXX_SRCS]
    if _newer(LIB, core):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "shared", "-o", LIB] + core + \
            ["-Xlinker", f"-rpath,{CUDA_LIB}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB}")
    if _newer(LIB_CXX, cxx + [LIB]):
        cmd = ["g++", "-shared", "-o", LIB_CXX] + cxx + [f"-L{LIB_DIR}", "-lstereoscan_b200",
                                                          f"-Wl,-rpath,{LIB_DIR}", "-lz"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ API link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB_CXX}")
    _build_cpp_test(verbose)
    return LIB


def _build_cpp_test(verbose):
    out_dir = os.path.join(ROOT, "tests", "cpp", "build")
    os.makedirs(out_dir, exist_ok=True)
    for name in ("test_api", "io_tool"):
        src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
        if not os.path.exists(src):
            continue
        exe = os.path.join(out_dir, name)
        if _newer(exe, [src, LIB, LIB_CXX] + _deps()):
            cmd = ["g++", "-std=c++17", "-O1", f"-I{INC}", src, "-o", exe, f"-L{LIB_DIR}",
                   "-lstereoscan_b200_cxx", "-lstereoscan_b200", f"-Wl,-rpath,{LIB_DIR}",
                   f"-Wl,-rpath,{CUDA_LIB}"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"C++ test build failed:\n{r.stdout}\n{r.stderr}")
            if verbose:
                print(f"built {exe}")
    # source-compatibility probe: the reference's unmodified reference.cpp
    # against this repository's headers (only where /root/reference exists;
    # the binary travels to the GPU box with the snapshot)
    ref_src = "/root/reference/proj/src/stereo/reference.cpp"
    ref_inc = "/root/reference/proj/include"
    src = os.path.join(ROOT, "tests", "cpp", "ref_compat.cpp")
    exe = os.path.join(out_dir, "ref_compat")
    if os.path.exists(ref_src) and _newer(exe, [src, ref_src, LIB, LIB_CXX] + _deps()):
        cmd = ["g++", "-std=c++20", "-O1", f"-I{INC}", f"-idirafter{ref_inc}", src, ref_src,
               "-o", exe, f"-L{LIB_DIR}", "-lstereoscan_b200_cxx", "-lstereoscan_b200",
               f"-Wl,-rpath,{LIB_DIR}", f"-Wl,-rpath,{CUDA_LIB}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference.cpp against include/ failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {exe}")


if __name__ == "__main__":
    build()
