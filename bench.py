#!/usr/bin/env python
"""Benchmark: stereo pairs/s of the full per-frame stereo chain on B200.

Metric (BASELINE.json): stereo pairs/sec at 960x540 D=64 (1/2/4/8 B200),
ms/pair, fraction of the roofline. Every step runs the whole run_stereo_only
chain on every frame: luma -> ZNCC WTA -> 3 rounds of
outlier removal + hole filling -> 10 refinement iterations -> oriented point
cloud (points, normals, colours). Frames shard across ranks with no collective;
NCCL carries only the barrier and the max-over-ranks time.

Workloads (--workload; BASELINE.json configs):
  c4  (default, configs[3]) 256 synthetic textured 960x540 pairs per GPU per
      step, D=64 (d 0..63); weak scaling.
  c2  (configs[1]) the same with the low-texture recipe.
  c3  (configs[2]) 32 textured 1920x1080 pairs per GPU per step, D=128.
  c5  (configs[4]) a 1024-pair 1920x1080 D=128 synthetic video stream split
      into contiguous frame blocks across the GPUs (strong scaling); e2e
      streams it through the host API into a per-thread host ring (the
      streaming contract of SPEC.md:600: a frame's outputs are consumed before
      their slot is reused).

Keys:
  value     device-resident pairs/s: inputs in HBM, results written to device
            buffers; CUDA events on the context streams, max over ranks.
  e2e       the same through the public host API (ss_stereo_batch): pinned
            host RGB in, H2D + chain + D2H of disparity/validity/cloud inside
            the timed region, in the compact transfer format (points f32,
            normals octahedral snorm16, cloud arrays trimmed to n_points);
            e2e.full_format is the same with the reference's full layout.
  roofline  the dominant kernel group (largest device-time share, measured
            live with CUDA events on the launching stream): algorithmic
            lane-ops per launch (SURVEY.md §8d census) / its
            average launch time vs the ALU issue peak 148 SM x 128 lanes x
            sm_max_mhz; `stages` holds every kernel group's fraction.
  parity    the step's own outputs against SHA-256 digests of the reference's
            outputs for the same seeded frames (tests/golden/digests.json,
            made from oracle/_ref by tests/golden/make_digests.py), and, in
            the cpu_baseline leg, whole arrays against the reference run here.
            Any mismatch fails the run (exit status 1).
  cpu_baseline  the reference itself (oracle/_ref) on the host cores, bounded
            sample of the same workload's frames.

`--impl reference` runs only the reference CPU path (rank 0) on the same
metric and config. `--gpus N` without a torchrun environment re-launches
itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c4": dict(kind="textured", W=960, H=540, D=64, frames=256, batch=16, streams=4, unique=32,
               seed_base=0, scaling="weak", ref_pairs=5,
               desc="C4 (BASELINE.json configs[3]): 256 synthetic textured 960x540 stereo pairs "
                    "per GPU per step, D=64 (d 0..63), full chain luma+WTA+cleanup+refine+"
                    "cloud(normals)"),
    "c2": dict(kind="lowtex", W=960, H=540, D=64, frames=256, batch=16, streams=4, unique=32,
               seed_base=0, scaling="weak", ref_pairs=5,
               desc="C2 (BASELINE.json configs[1]): 256 synthetic low-texture 960x540 pairs per "
                    "GPU per step, D=64, full chain incl. normals"),
    "c3": dict(kind="textured", W=1920, H=1080, D=128, frames=32, batch=4, streams=4, unique=8,
               seed_base=100, scaling="weak", ref_pairs=2,
               desc="C3 (BASELINE.json configs[2]): 32 synthetic textured 1920x1080 stereo pairs "
                    "per GPU per step, D=128 (d 0..127), full chain incl. normals"),
    "c5": dict(kind="video", W=1920, H=1080, D=128, frames=1024, batch=4, streams=4, unique=32,
               seed_base=0, scaling="strong", ref_pairs=2,
               desc="C5 (BASELINE.json configs[4]): 1024-pair 1920x1080 D=128 synthetic video "
                    "stream (32 distinct drifting frames, tiled) split into contiguous frame "
                    "blocks across the GPUs, full chain incl. normals, clouds gathered to host"),
}
# SURVEY.md §8d census, 32-bit lane-ops per pair (whole chain).
CENSUS_TOTAL = {"c4": 2.16e9, "c2": 2.25e9, "c3": 10.6e9, "c5": 10.6e9}
# measured disc-fill list sizes summed over the 3 rounds (C3 scaled by area)
I_DISC = {"c4": 29.4e3, "c2": 54.0e3, "c3": 117.6e3, "c5": 117.6e3}
DIGEST_PATH = os.path.join(ROOT, "tests", "golden", "digests.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--frames", type=int, default=None, help="pairs per rank per step (c5: total)")
    ap.add_argument("--batch", type=int, default=None, help="frames per device launch")
    ap.add_argument("--streams", type=int, default=None,
                    help="concurrent contexts (one CUDA stream each) sharing the frames")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="steps in the e2e timed region (default: --steps, at least 3; "
                         "c5 at most 5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extensions", action="store_true",
                    help="skip the LR-check / feature / fusion side measurements")
    ap.add_argument("--cpu-pairs", type=int, default=2)
    ap.add_argument("--cpu-configs", action="store_true",
                    help="also time the reference CPU chain on C1/C2/C3 (median of 3; minutes)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/sharding logic only (gloo, no GPU work): for CPU tests")
    a = ap.parse_args()
    wl = WORKLOADS[a.workload]
    a.frames = a.frames or wl["frames"]
    a.batch = a.batch or wl["batch"]
    a.streams = a.streams or wl["streams"]
    if a.e2e_steps is None:  # the same K steps as the device-resident number
        a.e2e_steps = max(3, a.steps if wl["scaling"] == "weak" else min(a.steps, 5))
    return a


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def self_launch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run, one rank
    per GPU (the driver's own launch, so the measured path is the same)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        return
    if args.gpus <= 1:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, p in zip(names, parts[2:]):
                if p.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- frames

def frame_seed(wl_name, rank, world, i, frames):
    """(seed, video frame) of local frame i of `rank` (the tiling is by seed, so
    the digest table names the first frames of rank 0 directly)."""
    wl = WORKLOADS[wl_name]
    u = wl["unique"]
    if wl["scaling"] == "strong":
        from paper_2007_12623_b200.shard import frame_range
        g = frame_range(frames, rank, world)[0] + i
        return g % u, g % u
    return wl["seed_base"] + rank * frames + (i % u), 0


def local_frames(args, rank, world):
    if WORKLOADS[args.workload]["scaling"] == "strong":
        from paper_2007_12623_b200.shard import frame_range
        a, b = frame_range(args.frames, rank, world)
        return b - a
    return args.frames


def make_unique(args, rank, world, count):
    """The distinct frames this rank needs (RGB), in local order modulo `unique`."""
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    wl = WORKLOADS[args.workload]
    u = max(1, min(wl["unique"], count))
    Ls, Rs = [], []
    for i in range(u):
        seed, fr = frame_seed(args.workload, rank, world, i, args.frames)
        L, R, _ = stereo_pair(wl["kind"], wl["W"], wl["H"], wl["D"], seed=seed, frame=fr)
        Ls.append(as_rgb(L))
        Rs.append(as_rgb(R))
    return np.stack(Ls), np.stack(Rs)


def config_dict(args, world):
    wl = WORKLOADS[args.workload]
    return {"workload": wl["desc"], "width": wl["W"], "height": wl["H"], "disparities": wl["D"],
            "cache": "inputs > L2: every frame of a step is read from its own HBM copy (c4/c2/c3: "
                     "distinct per-frame buffers, >= 398 MB per GPU; c5: 32 distinct 12.4 MB frames "
                     "in rotation), no flush",
            "parallelism": f"frame-shard x{world}, no collective"}


# ---------------------------------------------------------------- digests

def map_digest(d, v):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d, np.float32).tobytes())
    h.update(np.ascontiguousarray(v, np.uint8).tobytes())
    return h.hexdigest()


def sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dt).tobytes()).hexdigest()


def digest_keys(args):
    dig = json.load(open(DIGEST_PATH)) if os.path.exists(DIGEST_PATH) else {}
    pre = {"c4": "bench_c4_", "c2": "bench_c2_", "c3": "bench_c3_",
           "c5": "bench_c5_"}.get(args.workload)
    if pre is None:
        return dig, []
    keys = sorted(k for k in dig if k.startswith(pre))
    return dig, keys


def check_frames(get_frame, keys, dig, cloud=True):
    """get_frame(i) -> dict of host arrays for local frame i; returns mismatching keys."""
    bad = []
    for i, k in enumerate(keys):
        e, f = dig[k], get_frame(i)
        ok = map_digest(f["disparity"], f["valid"]) == e["refine"]
        if cloud and ok:
            n = int(f["n_points"])
            ok = (n == e["n_points"] and sha(f["index"], np.int32) == e["cloud_index"]
                  and sha(f["points"][:n], np.float32) == e["cloud_points_f32"])
        if not ok:
            bad.append(k)
    return bad


# ---------------------------------------------------------------- reference CPU path

def reference_chain(pairs, wl, want_outputs=False):
    """The reference's own CPU path (oracle/_ref) on host RGB pairs; cloud
    stage from the restatement (the reference's needs Eigen, absent). Returns
    (seconds, kind, outputs)."""
    from oracle.oracle import Oracle
    from paper_2007_12623_b200.synth import default_rig, params_for
    kind = "reference" if Oracle.available("ref") else "port"
    ref = Oracle("ref" if kind == "reference" else "orc")
    orc = Oracle("orc")
    p = params_for(wl["D"])
    rig = default_rig(wl["W"], wl["H"])
    outs = []
    t0 = time.perf_counter()
    for L, R in pairs:
        lg, rg = ref.to_gray(L), ref.to_gray(R)
        d, v = ref.compute_disparity(lg, rg, p)
        d, v = ref.cleanup_pass(d, v, p)
        d, v = ref.refine_disparities(d, v, lg, rg, p)
        cl = orc.disparity_to_cloud(d, v, L, rig)
        if want_outputs:
            outs.append((d, v, cl))
    return time.perf_counter() - t0, kind, outs


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def omp_threads(n):
    """Set the OpenMP team size of this process (the reference library's)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
        return True
    except OSError:
        return False


def workload_pairs(args, n):
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    wl = WORKLOADS[args.workload]
    out = []
    for i in range(n):
        seed, fr = frame_seed(args.workload, 0, 1, i, args.frames)
        L, R, _ = stereo_pair(wl["kind"], wl["W"], wl["H"], wl["D"], seed=seed, frame=fr)
        out.append((as_rgb(L), as_rgb(R)))
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    k = wl["ref_pairs"]
    pairs = workload_pairs(args, k)
    times = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        t, kind, _ = reference_chain(pairs, wl)
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = k * len(times) / total
    cores = os.cpu_count()
    line = {
        "metric": "stereo pairs/sec", "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / len(times), "pairs_per_step": k,
        "ms_per_pair": 1000.0 * total / (k * len(times)),
        "higher_is_better": True, "scaling": wl["scaling"],
        "vs_baseline": None, "dtype": "u8/int64/f64", "data": "synthetic",
        "config": config_dict(args, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{k} pairs of the workload's first frames per step through "
                                   "oracle/_ref (unmodified reference matcher/cleanup/smoothing, "
                                   "OpenMP on all cores) + restated cloud (Eigen absent); the "
                                   "reference API is per pair"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_side_by_side(runs=3):
    """SURVEY.md §8d CPU side-by-side: the reference chain (oracle/_ref) on one
    pair of each of C1, C2 and C3, median of `runs`, all host cores; C1 also
    on one thread. Seconds of host time: opt-in (--cpu-configs)."""
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    out = {"cores": os.cpu_count(), "cpu_model": cpu_model(), "runs": runs}
    for key, kind, Wc, Hc, Dc in (("C1", "textured", 960, 540, 64), ("C2", "lowtex", 960, 540, 64),
                                  ("C3", "textured", 1920, 1080, 128)):
        L, R, _ = stereo_pair(kind, Wc, Hc, Dc, seed=1234)
        wl = dict(W=Wc, H=Hc, D=Dc)
        ts = [reference_chain([(as_rgb(L), as_rgb(R))], wl)[0] for _ in range(runs)]
        out[key] = {"pairs_per_s": 1.0 / statistics.median(ts), "median_s": statistics.median(ts)}
    return out


# ---------------------------------------------------------------- roofline

def roofline_report(args, stages, frames_timed, n_sm, sm_max, hbm_peak, iters=10):
    """Per kernel group: census lane-ops per
    launch over the live average launch time (CUDA events on the launching
    stream, one context, no concurrency)."""
    wl = WORKLOADS[args.workload]
    N, D = wl["W"] * wl["H"], wl["D"]
    alu_peak = n_sm * 128 * sm_max * 1e6
    census = {  # lane-ops per frame
        "wta_sweep": ("k_wta11: chessboard ZNCC over [d_min, d_max] + WTA", 15.0 * N * D),
        "refine_repick": ("k_d_gather + k_repick_list (iteration 0: k_d_repick): b-disc "
                          "gather 62N + smoothing 3N + re-pick 60N per iteration (re-picks "
                          "certified unchanged are skipped, their census still counted)",
                          125.0 * N * iters),
        "cleanup_disc": ("k_row_count/k_disc_select/k_disc_sum: I_disc x (82 + 3 x 1256)",
                         I_DISC[args.workload] * (82 + 3 * 1256)),
        "cleanup_radial": ("k_fill_radial_list: 144N", 144.0 * N),
        "cleanup_outliers": ("k_edge_words + k_outlier_words: 72N", 72.0 * N),
        "cloud_normals": ("k_cloud_normals: 7x7 moments + 3x3 eigen, 600N", 600.0 * N),
    }
    hbm = {"refine_scan": ("k_scan_b / k_scan_bt: row prefix scans, 29 B/px per iteration",
                           29.0 * N * iters)}
    out = {}
    for name, (what, ops) in census.items():
        ms, launches = stages.get(name, (0.0, 0))
        if ms <= 0 or launches <= 0:
            continue
        per_launch = ops * frames_timed / launches
        t = ms / launches / 1e3
        out[name] = {"kernel": what, "bound": "alu", "achieved": per_launch / t / 1e12,
                     "peak": alu_peak / 1e12, "unit": "Tlane-op/s",
                     "frac": per_launch / t / alu_peak, "ops_per_launch": per_launch,
                     "avg_launch_ms": t * 1e3, "launches": launches,
                     "share_of_chain": None}
    for name, (what, nbytes) in hbm.items():
        ms, launches = stages.get(name, (0.0, 0))
        if ms <= 0 or launches <= 0:
            continue
        per_launch = nbytes * frames_timed / launches
        t = ms / launches / 1e3
        out[name] = {"kernel": what, "bound": "hbm", "achieved": per_launch / t / 1e9,
                     "peak": hbm_peak, "unit": "GB/s", "frac": per_launch / t / 1e9 / hbm_peak,
                     "bytes_per_launch": per_launch, "avg_launch_ms": t * 1e3,
                     "launches": launches, "share_of_chain": None}
    chain_ms = sum(stages[k][0] for k in ("luma", "stats", "wta_sweep", "wta_resolve", "cleanup",
                                          "refine", "cloud"))
    for name, r in out.items():
        r["share_of_chain"] = stages[name][0] / chain_ms if chain_ms else None
    # whole-stage view (census per pair over the stage's per-pair time)
    stage_census = {"wta_sweep": 15.0 * N * D,
                    "cleanup": 216.0 * N + I_DISC[args.workload] * (82 + 3 * 1256),
                    "refine": 1910.0 * N, "cloud": 700.0 * N,
                    "luma+stats": 36.0 * N}
    per_stage = {}
    for name, ops in stage_census.items():
        ms = (stages["luma"][0] + stages["stats"][0]) if name == "luma+stats" else stages[name][0]
        if ms > 0:
            t = ms / frames_timed / 1e3
            per_stage[name] = {"us_per_pair": t * 1e6, "frac": ops / t / alu_peak}
    return out, per_stage, alu_peak


# ---------------------------------------------------------------- our arm

def run_dry(args):
    """Launcher / sharding check without a GPU (tests/test_bench_contract.py)."""
    import torch.distributed as dist
    from paper_2007_12623_b200.shard import frame_range, max_over_ranks
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    n = local_frames(args, rank, world)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_flag": args.gpus,
                          "frames_rank0": n, "max_over_ranks": t,
                          "block0": frame_range(args.frames, 0, world)
                          if WORKLOADS[args.workload]["scaling"] == "strong" else None}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.shard import max_over_ranks
    from paper_2007_12623_b200.synth import default_rig, params_for

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = WORKLOADS[args.workload]
    W, H, D = wl["W"], wl["H"], wl["D"]
    N = W * H
    B, S = args.batch, max(1, args.streams)
    F = local_frames(args, rank, world)
    strong = wl["scaling"] == "strong"
    Lu_np, Ru_np = make_unique(args, rank, world, F)
    u = len(Lu_np)
    assert u % B == 0 or F <= u, "unique frames must tile into whole launches"
    # HBM-resident inputs. c4/c2/c3: one distinct copy per frame of the step
    # (> L2); c5: the 32 distinct frames in rotation.
    Lu = torch.from_numpy(Lu_np).to(dev)
    Ru = torch.from_numpy(Ru_np).to(dev)
    if strong:
        Ld, Rd = Lu, Ru
        in_index = [i % u for i in range(F)]
    else:
        reps = (F + u - 1) // u
        Ld = Lu.repeat(reps, 1, 1, 1)[:F].contiguous()
        Rd = Ru.repeat(reps, 1, 1, 1)[:F].contiguous()
        in_index = list(range(F))
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    # device outputs: all frames of the step (weak); a ring of 2 launches per
    # context (strong: the stream's consumer has drained a slot before reuse)
    n_out = F if not strong else min(F, 2 * S * B)
    od = ss.StereoContext.alloc_outputs(n_out, H, W, flags,
                                        alloc=lambda s, dt: torch.empty(
                                            s, dtype=torch.from_numpy(np.empty(0, dt)).dtype, device=dev))
    p = params_for(D)
    ctxs = [ss.StereoContext(local, W, H, B, ss.StereoParams(**p),
                             ss.StereoRig(**default_rig(W, H))) for _ in range(S)]
    ctx = ctxs[0]
    streams = [torch.cuda.ExternalStream(c.stream, device=dev) for c in ctxs]
    stream = streams[0]
    chunks = [(f0, min(B, F - f0)) for f0 in range(0, F, B)]

    def step_device(cs=ctxs):
        for i, (f0, m) in enumerate(chunks):
            o0 = f0 % n_out
            d_out = {k: t[o0:o0 + m].data_ptr() for k, t in od.items()}
            j = in_index[f0]
            cs[i % len(cs)].run_device(m, W, H, Ld[j].data_ptr(), Rd[j].data_ptr(), flags,
                                       d_out=d_out)

    def barrier():
        torch.cuda.synchronize(dev)
        for c in ctxs:
            c.sync()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step_device()
    barrier()
    for c in ctxs:
        c.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for st in streams[1:]:
            st.wait_event(e0)
        for _ in range(args.steps):
            step_device()
        for st in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)
        e1.record(stream)
        e1.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    stats = {k: sum(c.stats()[k] for c in ctxs) for k in ctxs[0].stats()}

    # ---- parity of the timed step's own outputs (rank 0 holds the digest frames)
    dig, keys = digest_keys(args)
    parity = None
    if rank == 0 and keys:
        keys = keys[:min(len(keys), F)]
        if strong:  # the ring was overwritten: re-run the stream's first launch
            ctx.run_device(B, W, H, Ld[0].data_ptr(), Rd[0].data_ptr(), flags,
                           d_out={k: t[0:B].data_ptr() for k, t in od.items()})
            ctx.sync()
        torch.cuda.synchronize(dev)
        hk = {k: t[:len(keys)].cpu().numpy() for k, t in od.items()}
        bad = check_frames(lambda i: {k: v[i] for k, v in hk.items()}, keys, dig)
        parity = {"reference": "SHA-256 of oracle/_ref outputs (tests/golden/digests.json)",
                  "device_frames_checked": len(keys), "device_frames_mismatched": bad}

    # ---- per-kernel-group device times on one context (no concurrency)
    ctx.enable_timing(True)
    step_device([ctx])
    barrier()
    stages = ctx.stage_times()
    ctx.enable_timing(False)
    ms_max = max_over_ranks(ms, device=dev)
    pairs = (args.frames if strong else world * F) * args.steps
    value = pairs / (ms_max / 1000.0)

    # ---- e2e through the public host API (pinned host buffers) ----
    # headline: the compact transfer format (points f32 and colours exact,
    # normals octahedral snorm16 within 1e-4 rad, cloud arrays trimmed to
    # n_points); also measured: the full reference-format transfer
    compact = flags & ~ss.SS_OUT_NORMALS | ss.SS_OUT_NORMALS_OCT | ss.SS_OUT_TRIM
    e2e_value, h2d, d2h, e2e_extra = None, 0, 0, {}
    if args.e2e_steps > 0:
        Lh = ss.pinned_empty(tuple(Ld.shape), np.uint8)
        Rh = ss.pinned_empty(tuple(Rd.shape), np.uint8)
        Lh[...] = Ld.cpu().numpy()
        Rh[...] = Rd.cpu().numpy()

        def d2h_bytes(fl, npts):
            per_px = 4 + 1 + 4  # disparity, valid, index
            per_pt = 12 + 3 + (4 if fl & ss.SS_OUT_NORMALS_OCT else 12)
            pts = int(np.sum(npts)) if fl & ss.SS_OUT_TRIM else len(npts) * N
            return len(npts) * (N * per_px + 4) + pts * per_pt

        # one set of pinned host outputs serves both formats (the compact one
        # adds only the octahedral normals): ~4.8 GB per rank at C4, not 2x
        pool = {}

        def host_outputs(n, fl):
            want = ss.StereoContext.alloc_outputs(n, H, W, fl, alloc=lambda s_, dt: (s_, dt))
            out = {}
            for k, (shape, dt) in want.items():
                if k not in pool or pool[k].shape != shape:
                    pool[k] = ss.pinned_empty(shape, dt)
                out[k] = pool[k]
            return out

        def measure_e2e(fl):
            consumed = [0] * S
            if strong:
                # per-thread host ring of 2 launches; each chunk is consumed
                # (its point count read) before the ring slot is reused
                ho = [ss.StereoContext.alloc_outputs(2 * B, H, W, fl,
                                                     alloc=lambda s_, dt: ss.pinned_empty(s_, dt))
                      for _ in range(S)]  # a ring of 2 launches per thread: small
                nbytes = [0] * S

                def part(k, steps):
                    for _ in range(steps):
                        for ci in range(k, len(chunks), S):
                            f0, m = chunks[ci]
                            j = in_index[f0]
                            slot = (ci // S) % 2
                            o = {kk: v[slot * B:slot * B + m] for kk, v in ho[k].items()}
                            ctxs[k].run(Lh[j:j + m], Rh[j:j + m], fl, out=o)
                            consumed[k] += int(o["n_points"].sum())
                            nbytes[k] += d2h_bytes(fl, o["n_points"])
                outs = None
            else:
                outs = host_outputs(F, fl)
                cuts = [F * i // S for i in range(S + 1)]

                def part(k, steps):
                    a, b = cuts[k], cuts[k + 1]
                    for _ in range(steps):
                        ctxs[k].run(Lh[a:b], Rh[a:b], fl, out={kk: v[a:b] for kk, v in outs.items()})

            def run_all(steps):
                th = [threading.Thread(target=part, args=(k, steps)) for k in range(S)]
                for t in th:
                    t.start()
                for t in th:
                    t.join()

            run_all(1)  # warm the host path: every pipeline slot allocated before timing
            barrier()
            if strong:
                consumed[:] = [0] * S
                nbytes[:] = [0] * S
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            run_all(args.e2e_steps)
            t1.record(stream)
            t1.synchronize()
            barrier()
            ems = max_over_ranks(t0.elapsed_time(t1), device=dev)
            val = (args.frames if strong else world * F) * args.e2e_steps / (ems / 1000.0)
            db = (sum(nbytes) / args.e2e_steps) if strong else d2h_bytes(fl, outs["n_points"])
            ext = {"d2h_bytes_per_pair": db / F, "d2h_gbs_per_gpu": db * args.e2e_steps /
                   (ems / 1000.0) / 1e9}
            if strong:
                ext["host_ring_frames_per_thread"] = 2 * B
                ext["points_consumed_per_step"] = int(sum(consumed)) // args.e2e_steps
            return val, db, ext, outs

        e2e_value, d2h, e2e_extra, ho_c = measure_e2e(compact)
        if parity is not None and not strong:  # checked before the buffers are reused
            bad_c = check_frames(lambda i: {k: v[i] for k, v in ho_c.items()}, keys, dig)
        h2d = 2 * F * N * 3
        e2e_extra["format"] = ("compact (SS_OUT_NORMALS_OCT | SS_OUT_TRIM): disparity f32, valid, "
                               "index, n_points, points f32 + colours for n_points entries, "
                               "normals octahedral snorm16 (<= 1e-4 rad)")
        full_val, full_db, _, ho_f = measure_e2e(flags)
        e2e_extra["full_format"] = {"value": full_val, "unit": "pairs/s",
                                    "d2h_bytes_per_pair": full_db / F,
                                    "format": "reference outputs at full per-frame capacity: "
                                              "normals f32x3, untrimmed cloud arrays"}
        if parity is not None and not strong:
            bad = bad_c + check_frames(lambda i: {k: v[i] for k, v in ho_f.items()}, keys, dig)
            parity["e2e_frames_checked"] = 2 * len(keys)
            parity["e2e_frames_mismatched"] = bad
        del ho_c, ho_f
        pool.clear()

    if world > 1:
        dist.barrier()
    if rank != 0:
        for c in ctxs:
            c.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    hbm_peak = float(peaks.get("hbm_gbs", 6446.9))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    groups, per_stage, alu_peak = roofline_report(args, stages, F, n_sm, sm_max, hbm_peak,
                                                  iters=p["refine_iterations"])
    top = max(groups, key=lambda k: groups[k]["share_of_chain"] or 0.0)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get(top, {})
        if t.get("frames_per_launch") == B and t.get("workload") == args.workload:
            traffic = t.get("dram_bytes_per_launch")
    # Binding-pipe view (measured pipe peaks, profiles/r2/pipe_rates.json): the
    # group's launch time if its dominant kernel's busiest pipe (ncu) ran at
    # 100%, over the live launch time. The census peak above counts every op
    # at 128 lanes/clock; FP64, dp4a and IMAD issue at 64 and shared memory
    # moves 128 B/clock, so the census fraction understates how close a kernel is.
    ppath = os.path.join(ROOT, "profiles", "pipe_roofline.json")
    if os.path.exists(ppath):
        for name, pr in json.load(open(ppath))["groups"].items():
            g = groups.get(name)
            if g and pr.get("frames_per_launch") == B and pr.get("workload") == args.workload:
                g["pipe_roofline"] = {
                    "kernel": pr["kernel"], "binding_pipe": pr["binding_pipe"],
                    "roof_ms_per_launch": pr["roof_ms_per_launch"],
                    "frac": pr["roof_ms_per_launch"] / g["avg_launch_ms"],
                    "source": "profiles/pipe_roofline.json (ncu --set full, one launch)"}
    roofline = dict(groups[top])
    roofline.update({
        "group": top, "traffic": traffic,
        "traffic_unit": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                        "(profiles/roofline_traffic.json)",
        "peak_source": f"{n_sm} SM x 128 lanes x sm_max_mhz {sm_max:.0f} (MEASURED_PEAKS.json); "
                       "ALU issue, not a bf16/HBM figure: the path is integer/FP64 ALU work",
        "stages": per_stage, "kernel_groups": groups,
        "pipeline_census_frac": CENSUS_TOTAL[args.workload] * value / world / alu_peak,
        "hbm_frac_pipeline": (21.8e6 if N < 1e6 else 87.1e6) * value / world / (hbm_peak * 1e9),
    })

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        npairs = min(args.cpu_pairs, F)
        pairs_cpu = workload_pairs(args, npairs)
        tcpu, kind, routs = reference_chain(pairs_cpu, wl, want_outputs=True)
        cpu = {"value": npairs / tcpu, "unit": "pairs/s", "cores": os.cpu_count(),
               "kind": kind, "cpu_model": cpu_model(),
               "sample": f"the workload's first {npairs} pairs through oracle/_ref (unmodified "
                         "reference, OpenMP all cores) + restated cloud"}
        # whole-array comparison of those frames with this run's device outputs
        if not strong or npairs <= B:
            if strong:
                ctx.run_device(B, W, H, Ld[0].data_ptr(), Rd[0].data_ptr(), flags,
                               d_out={k: t[0:B].data_ptr() for k, t in od.items()})
                ctx.sync()
            torch.cuda.synchronize(dev)
            mism = 0
            for i, (d, v, cl) in enumerate(routs):
                gd = od["disparity"][i].cpu().numpy()
                gv = od["valid"][i].cpu().numpy()
                mism += int((gv != v).sum()) + int((gd.view(np.uint32) != d.view(np.uint32)).sum())
            if parity is None:
                parity = {}
            parity["live_reference_frames"] = npairs
            parity["live_reference_mismatched_px"] = mism
        if omp_threads(1) and args.workload in ("c4", "c2"):  # also one thread
            t1, _, _ = reference_chain(pairs_cpu[:1], wl)
            cpu["single_thread_value"] = 1.0 / t1
            omp_threads(os.cpu_count())
    if cpu is not None and args.cpu_configs:
        cpu["side_by_side"] = cpu_side_by_side()
    ok = True
    if parity is not None:
        ok = (not parity.get("device_frames_mismatched") and not parity.get("e2e_frames_mismatched")
              and not parity.get("live_reference_mismatched_px"))
        parity["ok"] = ok
    ext = None
    if not (args.no_extensions or world > 1 or args.workload != "c4"):
        ext = extensions(ss, ctxs, step_device, barrier, stream, F, Lu_np[0], Ru_np[0], od, W, H)
    line = {
        "metric": "stereo pairs/sec", "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": wl["scaling"],
        "vs_baseline": None, "dtype": "u8/int32/f32-filter/f64", "data": "synthetic",
        "config": config_dict(args, world),
        "workload": args.workload, "pairs_per_step_per_gpu": F, "frames_per_launch": B,
        "streams_per_gpu": S,
        "ms_per_pair": ms_max / args.steps / (pairs / args.steps / world),
        "e2e": dict({"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h, "steps": args.e2e_steps}, **e2e_extra),
        "gpu_launches": int(stats["kernel_launches"]),
        "graph_launches": int(stats.get("graph_launches", 0)),
        "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
        "clocks": clk.summary(),
        "stage_ms_per_pair": {k: v[0] / F for k, v in stages.items()},
        "exact_resolves": {"wta_pixels": stats["wta_resolved"],
                           "refine_repicks": stats["refine_resolved"],
                           "disc_fill_pixels": stats.get("disc_fill_pixels"),
                           "refine_scored": stats.get("refine_scored"),
                           "frames": stats["frames"]},
        "extensions": ext,
    }
    print(json.dumps(line), flush=True)
    for c in ctxs:
        c.close()
    if world > 1:
        dist.destroy_process_group()
    if not ok:
        print("bench.py: outputs differ from the reference digests", file=sys.stderr)
        sys.exit(1)


def extensions(ss, ctxs, step_device, barrier, stream, F, L0, R0, od, W, H):
    """Side measurements of the SURVEY §8f rows (not the headline metric):
    the chain with the opt-in LR check (device pairs/s, same workload), fusion
    of the step's device-resident clouds, and the feature front end on one C1
    frame pair through the per-stage C-ABI (host buffers, transfers included)
    beside the reference's CPU code."""
    import torch
    out = {}
    for c in ctxs:
        c.set_lr_check(True, 1)
    step_device()  # warm: the right-view buffers are allocated on first use
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for st in [torch.cuda.ExternalStream(c.stream) for c in ctxs][1:]:
        st.wait_event(a)
    step_device()
    for c in ctxs[1:]:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(c.stream))
        stream.wait_event(ev)
    b.record(stream)
    b.synchronize()
    out["lr_check_chain"] = {"value": F / (a.elapsed_time(b) / 1000.0), "unit": "pairs/s",
                             "note": "full chain + right-view sweep + LR check, 1 step"}
    for c in ctxs:
        c.set_lr_check(False)
    barrier()
    from paper_2007_12623_b200.synth import default_rig
    rig = default_rig(W, H)
    model = ss.fusion.SurfelModel(torch.cuda.current_device())
    nf = min(F, 32)
    poses = []
    for f in range(nf):
        a_ = 1e-4 * f
        poses.append(np.array([[np.cos(a_), 0, np.sin(a_), 1.0 * f], [0, 1, 0, 0],
                               [-np.sin(a_), 0, np.cos(a_), 0]]))

    def fuse_all(m):
        for f in range(nf):
            m.fuse_device(od["index"][f].data_ptr(), od["points"][f].data_ptr(),
                          od["normals"][f].data_ptr(), od["colors"][f].data_ptr(), poses[f], rig)

    fuse_all(model)  # warm (allocations)
    model.close()
    model = ss.fusion.SurfelModel(torch.cuda.current_device())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fuse_all(model)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["fusion"] = {"frames_per_s": nf / dt, "frames": nf, "surfels": len(model),
                     "note": "fuse_device of C1 clouds (~0.5 M points each) into one model; "
                             "host wall clock around synchronous calls"}
    model.close()
    gl = ss.to_gray(L0)
    gr = ss.to_gray(R0)

    def feat_gpu():
        fl = ss.features.describe(gl, ss.features.detect_corners(gl, 2000, 20))
        fr = ss.features.describe(gr, ss.features.detect_corners(gr, 2000, 20))
        return ss.features.match_features(*fl, *fr, 64)

    feat_gpu()
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        m = feat_gpu()
        t.append(time.perf_counter() - t0)
    out["features_pair"] = {"gpu_ms": 1000 * statistics.median(t), "matches": int(len(m["index_a"])),
                            "what": "detect_corners(2000, thr 20) + describe on both C1 views + "
                                    "match_features(64), per-stage C-ABI incl. H2D/D2H"}
    try:
        from oracle.oracle import Oracle
        if Oracle.available("ref"):
            ref = Oracle("ref")
            t = []
            for _ in range(3):
                t0 = time.perf_counter()
                cl, cr = ref.detect_corners(gl, 2000, 20), ref.detect_corners(gr, 2000, 20)
                ref.match_features(*ref.describe(gl, cl), *ref.describe(gr, cr), 64)
                t.append(time.perf_counter() - t0)
            out["features_pair"]["cpu_reference_ms"] = 1000 * statistics.median(t)
            out["features_pair"]["cpu_cores"] = os.cpu_count()
    except Exception as e:  # the CPU side is informational
        out["features_pair"]["cpu_reference_error"] = str(e)[:200]
    return out


def main():
    args = parse()
    self_launch(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
