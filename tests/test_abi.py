"""CPU-side checks of the drop-in boundary (no GPU needed).

* the in-tree library builds for sm_100a and exports every symbol the public
  header include/ss_stereo.h declares;
* the product never imports the oracle and has no CPU fallback: on a machine
  without a CUDA device every compute entry point fails loudly (SS_ENODEV);
* host-side helpers of the boundary (defaults, validation messages, support
  constants) match the reference.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "ss_stereo.h")
LIB = os.path.join(ROOT, "paper_2007_12623_b200", "lib", "libstereoscan_b200.so")


@pytest.fixture(scope="module")
def built():
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    return LIB


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for s in ["ss_compute_disparity", "ss_cleanup_pass", "ss_refine_disparities",
              "ss_disparity_to_cloud", "ss_remove_outliers", "ss_fill_holes", "ss_to_gray",
              "ss_params_validate", "ss_stereo_batch", "ss_ctx_create"]:
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ss_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(built)
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", built],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2007_12623_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ss_oracle" not in txt and "libss_ref" not in txt, f


@pytest.mark.skipif(has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback(built):
    import paper_2007_12623_b200 as ss
    L = np.zeros((32, 32), np.uint8)
    with pytest.raises(ss.StereoError) as e:
        ss.compute_disparity(L, L, ss.StereoParams(d_min=0, d_max=8))
    assert e.value.code == 5 and "no CUDA device" in str(e.value)
    with pytest.raises(ss.StereoError):
        ss.StereoContext(0, 64, 64, 1, ss.StereoParams(d_min=0, d_max=8))


def test_host_helpers_match_reference(built, orc):
    import paper_2007_12623_b200 as ss
    for r in (1, 5, 20, 33):
        assert ss.disc_neighbor_count(r) == orc.disc_neighbor_count(r)
        assert ss.disc_fill_min_support(r) == orc.disc_fill_min_support(r)
    ss.StereoParams().validate()
    for kw, msg in [(dict(window=4), "stereo: window must be odd and >= 3"),
                    (dict(d_min=5, d_max=5), "stereo: d_min must be < d_max"),
                    (dict(fill_radius_disc=0), "stereo: radii must be > 0"),
                    (dict(alpha=-0.1), "stereo: alpha must be in [0,1]"),
                    (dict(cleanup_iterations=-2), "stereo: cleanup_iterations must be >= 0"),
                    (dict(refine_iterations=-1), "stereo: refine_iterations must be >= 0")]:
        with pytest.raises(ss.StereoError) as e:
            ss.StereoParams(**kw).validate()
        assert str(e.value) == msg
    with pytest.raises(ss.StereoError) as e:
        ss.StereoRig(fx=1, fy=1, cx=5, cy=5, width=10, height=10, baseline_mm=0).validate()
    assert str(e.value) == "rig: baseline_mm must be > 0"
    with pytest.raises(ss.StereoError) as e:
        ss.StereoRig(fx=1, fy=1, cx=50, cy=5, width=10, height=10, baseline_mm=1).validate()
    assert str(e.value) == "intrinsics: cx out of image bounds"
