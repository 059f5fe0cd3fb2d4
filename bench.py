#!/usr/bin/env python
"""Benchmark: stereo pairs/s of the full per-frame stereo chain on B200.

Metric (BASELINE.json): stereo pairs/sec at 960x540 D=64, 1/2/4/8 B200.
Workload (BASELINE.json configs[3], "C4"): every rank processes a batch of
256 synthetic textured 960x540 pairs per step, d in [0, 63], the whole
run_stereo_only chain: luma -> ZNCC WTA -> 3 rounds of
outlier removal + hole filling -> 10 refinement iterations -> oriented point
cloud (points, normals, colours). Frames shard across ranks with no collective
(weak scaling); NCCL only carries the barrier and the max-over-ranks time.

  value  device-resident throughput: inputs already in HBM, results written to
         device output tensors; CUDA events on the ctx stream, max over ranks.
  e2e    the same through the public host API (ss_stereo_batch): pinned host
         RGB in, H2D + chain + D2H of disparity/validity/cloud inside the timed
         region.
  roofline  dominant kernel = the ZNCC cost sweep (k_wta11): algorithmic
         lane-ops per launch (SURVEY.md §8d census: 12 N (D+10) + 3 N D per
         frame) / its CUDA-event duration vs the ALU issue peak
         (148 SM x 128 lanes x sm_max_mhz).
  cpu_baseline  the reference itself (oracle/_ref, compiled from
         /root/reference by oracle/Makefile) on the host cores, bounded sample.

`--impl reference` runs only that reference CPU path (rank 0) on the same
metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H, D = 960, 540, 64
CENSUS = {"textured": 2.16e9, "lowtex": 2.25e9, "fhd": 10.6e9}  # lane-ops/pair, BASELINE.md


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=256, help="pairs per rank per step")
    ap.add_argument("--batch", type=int, default=16, help="frames per device launch")
    ap.add_argument("--unique", type=int, default=32, help="distinct seeded frames (tiled)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=4,
                    help="concurrent contexts (one CUDA stream each) sharing the frames")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extensions", action="store_true",
                    help="skip the LR-check / feature side measurements")
    ap.add_argument("--cpu-pairs", type=int, default=2)
    ap.add_argument("--cpu-configs", action="store_true",
                    help="also time the reference CPU chain on C1/C2/C3 (median of 3; minutes)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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


def make_frames(rank, world, frames, unique):
    from paper_2007_12623_b200.shard import frame_range
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    start, _ = frame_range(world * frames, rank, world)  # this rank's block of the global batch
    u = max(1, min(unique, frames))
    Ls, Rs = [], []
    for i in range(u):
        L, R, _ = stereo_pair("textured", W, H, D, seed=start + i)
        Ls.append(as_rgb(L))
        Rs.append(as_rgb(R))
    Ls, Rs = np.stack(Ls), np.stack(Rs)
    reps = (frames + u - 1) // u
    return np.tile(Ls, (reps, 1, 1, 1))[:frames], np.tile(Rs, (reps, 1, 1, 1))[:frames]


def reference_chain(pairs, Wc=None, Hc=None, Dc=None):
    """The reference's own CPU path (oracle/_ref) on host pairs; cloud stage from
    the restatement (the reference's needs Eigen, absent). Returns seconds."""
    Wc, Hc, Dc = Wc or W, Hc or H, Dc or D
    from oracle.oracle import Oracle
    from paper_2007_12623_b200.synth import default_rig, params_for
    kind = "reference" if Oracle.available("ref") else "port"
    ref = Oracle("ref" if kind == "reference" else "orc")
    orc = Oracle("orc")
    p = params_for(Dc)
    rig = default_rig(Wc, Hc)
    t0 = time.perf_counter()
    for L, R in pairs:
        lg, rg = ref.to_gray(L), ref.to_gray(R)
        d, v = ref.compute_disparity(lg, rg, p)
        d, v = ref.cleanup_pass(d, v, p)
        d, v = ref.refine_disparities(d, v, lg, rg, p)
        orc.disparity_to_cloud(d, v, L, rig)
    return time.perf_counter() - t0, kind


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


def cpu_pairs(n):
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    out = []
    for i in range(n):
        L, R, _ = stereo_pair("textured", W, H, D, seed=i)
        out.append((as_rgb(L), as_rgb(R)))
    return out


def config_dict(args, world):
    return {"workload": "C4: 256 synthetic textured 960x540 stereo pairs per rank per step, "
                        "D=64 (d 0..63), full chain luma+WTA+cleanup+refine+cloud(normals)",
            "width": W, "height": H, "disparities": D, "pairs_per_step_per_gpu": args.frames,
            "frames_per_launch": args.batch, "unique_seeded_frames": min(args.unique, args.frames),
            "cache": "inputs > L2 (per-step input 796 MB RGB per GPU, not flushed: each frame is "
                     "read once per step)",
            "parallelism": f"frame-shard x{world}, no collective",
            "streams_per_gpu": args.streams}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    pairs = cpu_pairs(1)
    times = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        t, kind = reference_chain(pairs)
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = len(times) / total
    cores = os.cpu_count()
    line = {
        "metric": "stereo pairs/sec at 960x540 D=64", "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/int64/f64", "data": "synthetic",
        "config": config_dict(args, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": kind,
                         "sample": "1 C1 pair per step through oracle/_ref (unmodified reference "
                                   "matcher/cleanup/smoothing, OpenMP all cores) + restated cloud"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def geometry_throughput(ss, kind, Wf, Hf, Df, nf, Bf, nctx):
    """Device-resident pairs/s of the full chain (incl. normals) for one
    synthetic geometry: nf pairs (6 seeded, tiled) in HBM, batches of Bf
    spread over nctx contexts; host wall clock around synchronous batches."""
    import torch
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    uniq = [stereo_pair(kind, Wf, Hf, Df, seed=100 + i)[:2] for i in range(6)]
    Lf = torch.from_numpy(np.stack([as_rgb(uniq[i % 6][0]) for i in range(nf)])).cuda()
    Rf = torch.from_numpy(np.stack([as_rgb(uniq[i % 6][1]) for i in range(nf)])).cuda()
    pf = ss.StereoParams(**params_for(Df))
    rf = ss.StereoRig(**default_rig(Wf, Hf))
    cf = [ss.StereoContext(torch.cuda.current_device(), Wf, Hf, Bf, pf, rf) for _ in range(nctx)]
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS

    def run():
        for i, f0 in enumerate(range(0, nf, Bf)):
            cf[i % nctx].run_device(Bf, Wf, Hf, Lf[f0].data_ptr(), Rf[f0].data_ptr(), flags)
        for c in cf:
            c.sync()

    run()  # warm (allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for c in cf:
        c.close()
    return {"value": nf / dt, "unit": "pairs/s", "ms_per_pair": 1000 * dt / nf,
            "workload": f"{nf} synthetic {kind} {Wf}x{Hf} pairs, D={Df} (d 0..{Df - 1}), "
                        f"full chain incl. normals, {nctx} contexts, inputs in HBM",
            "timing": "host wall clock around synchronous batches"}


def cpu_side_by_side(runs=3):
    """SURVEY.md §8d CPU side-by-side: the reference chain (oracle/_ref) on one
    pair of each of C1, C2 and C3, median of `runs`, all host cores; C1 also
    on one thread. Seconds of host time: opt-in (--cpu-configs)."""
    from paper_2007_12623_b200.synth import as_rgb, stereo_pair
    out = {"cores": os.cpu_count(), "cpu_model": cpu_model(), "runs": runs}
    for key, kind, Wc, Hc, Dc in (("C1", "textured", 960, 540, 64), ("C2", "lowtex", 960, 540, 64),
                                  ("C3", "textured", 1920, 1080, 128)):
        L, R, _ = stereo_pair(kind, Wc, Hc, Dc, seed=1234)
        pair = [(as_rgb(L), as_rgb(R))]
        ts = [reference_chain(pair, Wc, Hc, Dc)[0] for _ in range(runs)]
        out[key] = {"pairs_per_s": 1.0 / statistics.median(ts), "median_s": statistics.median(ts)}
    L, R, _ = stereo_pair("textured", 960, 540, 64, seed=1234)
    omp_threads(1)
    ts = [reference_chain([(as_rgb(L), as_rgb(R))])[0] for _ in range(runs)]
    omp_threads(os.cpu_count())
    out["C1"]["pairs_per_s_1thread"] = 1.0 / statistics.median(ts)
    return out


def extensions(ss, ctxs, step_device, barrier, stream, F, Lh_first, Rh_first, od=None):
    """Side measurements of the SURVEY §8f rows (not the headline metric):
    the chain with the opt-in LR check (device pairs/s, same workload), and
    the feature front end on one C1 frame pair through the per-stage C-ABI
    (host buffers, transfers included) beside the reference's CPU code."""
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
    if od is not None:
        # fusion of the step's device-resident clouds into one surfel model
        # (a slow pan: 1 mm and 0.1 mrad per frame), device events around it
        from paper_2007_12623_b200.synth import default_rig
        rig = default_rig(W, H)
        model = ss.fusion.SurfelModel(torch.cuda.current_device())
        nf = min(F, 32)
        poses = []
        for f in range(nf):
            a_ = 1e-4 * f
            poses.append(np.array([[np.cos(a_), 0, np.sin(a_), 1.0 * f], [0, 1, 0, 0],
                                   [-np.sin(a_), 0, np.cos(a_), 0]]))
        N = W * H

        def fuse_all(m):
            for f in range(nf):
                m.fuse_device(od["index"][f].data_ptr(), od["points"][f].data_ptr(),
                              od["normals"][f].data_ptr(), od["colors"][f].data_ptr(),
                              poses[f], rig)

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
    # C3 / C5 geometry (BASELINE.json configs[2], [4]): 1920x1080, D = 128; and
    # C2 (960x540 low-texture, D = 64): device-resident throughput over
    # synthetic pairs (6 seeded, tiled)
    for key, kind, Wf, Hf, Df, nf, Bf, nctx in (("fhd_d128", "textured", 1920, 1080, 128, 48, 8, 2),
                                                ("lowtex_c2", "lowtex", 960, 540, 64, 128, 16, 4)):
        try:
            out[key] = geometry_throughput(ss, kind, Wf, Hf, Df, nf, Bf, nctx)
        except Exception as e:  # informational side measurement
            out[key] = {"error": str(e)[:200]}
    gl = ss.to_gray(Lh_first)
    gr = ss.to_gray(Rh_first)

    def feat_gpu():
        fl = ss.features.describe(gl, ss.features.detect_corners(gl, 2000, 20))
        fr = ss.features.describe(gr, ss.features.detect_corners(gr, 2000, 20))
        return ss.features.match_features(*fl, *fr, 64)

    def feat_cpu(ref):
        cl = ref.detect_corners(gl, 2000, 20)
        cr = ref.detect_corners(gr, 2000, 20)
        fl, fr = ref.describe(gl, cl), ref.describe(gr, cr)
        return ref.match_features(*fl, *fr, 64)

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
                feat_cpu(ref)
                t.append(time.perf_counter() - t0)
            out["features_pair"]["cpu_reference_ms"] = 1000 * statistics.median(t)
            out["features_pair"]["cpu_cores"] = os.cpu_count()
    except Exception as e:  # the CPU side is informational
        out["features_pair"]["cpu_reference_error"] = str(e)[:200]
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.synth import default_rig, params_for

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    F, B = args.frames, args.batch
    N = W * H
    Lh_np, Rh_np = make_frames(rank, world, F, args.unique)
    # pinned host inputs (e2e) and HBM-resident copies (device value)
    Lh = torch.from_numpy(Lh_np).pin_memory()
    Rh = torch.from_numpy(Rh_np).pin_memory()
    Ld, Rd = Lh.to(dev), Rh.to(dev)
    del Lh_np, Rh_np
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    od = {"disparity": torch.empty((F, H, W), dtype=torch.float32, device=dev),
          "valid": torch.empty((F, H, W), dtype=torch.uint8, device=dev),
          "index": torch.empty((F, H, W), dtype=torch.int32, device=dev),
          "points": torch.empty((F, N, 3), dtype=torch.float32, device=dev),
          "normals": torch.empty((F, N, 3), dtype=torch.float32, device=dev),
          "colors": torch.empty((F, N, 3), dtype=torch.uint8, device=dev),
          "n_points": torch.empty((F,), dtype=torch.int32, device=dev)}
    p = params_for(D)
    # S contexts, one CUDA stream each: 16-frame chunks go round-robin, so one
    # chunk's latency-bound phases (serial FP64 scans, small exact-resolve
    # grids, launch tails) overlap another's wide kernels.
    S = max(1, args.streams)
    ctxs = [ss.StereoContext(local, W, H, B, ss.StereoParams(**p), ss.StereoRig(**default_rig(W, H)))
            for _ in range(S)]
    ctx = ctxs[0]
    streams = [torch.cuda.ExternalStream(c.stream, device=dev) for c in ctxs]
    stream = streams[0]

    def step_device(cs=ctxs):
        for i, f0 in enumerate(range(0, F, B)):
            m = min(B, F - f0)
            d_out = {k: t[f0:f0 + m].data_ptr() for k, t in od.items()}
            cs[i % len(cs)].run_device(m, W, H, Ld[f0].data_ptr(), Rd[f0].data_ptr(), flags,
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
    # Per-stage device times (and the sweep's roofline) from one extra,
    # untimed-for-value step on a single context: kernels of concurrent
    # streams would inflate each other's event brackets.
    ctx.enable_timing(True)
    step_device([ctx])
    barrier()
    stages = ctx.stage_times()
    ctx.enable_timing(False)
    from paper_2007_12623_b200.shard import max_over_ranks
    ms_max = max_over_ranks(ms, device=dev)
    pairs = world * F * args.steps
    value = pairs / (ms_max / 1000.0)

    # ---- e2e through the public host API (pinned host buffers) ----
    e2e_value, h2d, d2h = None, 0, 0
    if args.e2e_steps > 0:
        ho = ss.StereoContext.alloc_outputs(F, H, W, flags,
                                            alloc=lambda s, dt: ss.pinned_empty(s, dt))
        # the S contexts take contiguous frame ranges, one host thread each
        # (ss_stereo_batch is synchronous; ctypes releases the GIL)
        cuts = [F * i // S for i in range(S + 1)]
        Lnp, Rnp = Lh.numpy(), Rh.numpy()

        def e2e_part(i, steps):
            a, b = cuts[i], cuts[i + 1]
            for _ in range(steps):
                ctxs[i].run(Lnp[a:b], Rnp[a:b], flags, out={k: v[a:b] for k, v in ho.items()})

        def e2e_all(steps):
            th = [threading.Thread(target=e2e_part, args=(i, steps)) for i in range(S)]
            for t in th:
                t.start()
            for t in th:
                t.join()

        e2e_all(1)  # warm the host path: every pipeline slot allocated before timing
        barrier()
        f0e, f1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0e.record(stream)
        e2e_all(args.e2e_steps)
        f1e.record(stream)
        f1e.synchronize()
        barrier()
        ems = max_over_ranks(f0e.elapsed_time(f1e), device=dev)
        e2e_value = world * F * args.e2e_steps / (ems / 1000.0)
        h2d = 2 * F * N * 3
        # cloud arrays leave at full per-frame capacity (ss_stereo_batch pipeline)
        d2h = F * N * (4 + 1 + 4) + 4 * F + F * N * (12 + 12 + 3)

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
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = n_sm * 128 * sm_max * 1e6  # lane-ops/s
    wta_ms, wta_launches = stages["wta_sweep"]
    per_frame_ops = N * (12 * (D + 10) + 3 * D)
    launches = max(wta_launches, 1)
    frames_timed = F  # the single-context stage-timing step
    ops_per_launch = per_frame_ops * frames_timed / launches
    achieved = ops_per_launch / (wta_ms / launches / 1000.0) if wta_ms > 0 else 0.0
    hbm_peak = float(peaks.get("hbm_gbs", 6446.9))
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get("k_wta11", {})
        if t.get("frames_per_launch") == B:
            traffic = t.get("dram_bytes_per_launch")
    roofline = {
        "bound": "alu", "kernel": "k_wta11 (ZNCC cost sweep + WTA)",
        "achieved": achieved / 1e12, "peak": alu_peak / 1e12, "unit": "Tlane-op/s",
        "frac": achieved / alu_peak if alu_peak else None, "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch (ncu, profiles/roofline_traffic.json)",
        "peak_source": f"{n_sm} SM x 128 lanes x sm_max_mhz {sm_max:.0f} (MEASURED_PEAKS.json); "
                       "ALU issue, not a bf16/HBM figure: the path is integer/FP64 ALU work",
        "ops_per_launch": ops_per_launch, "avg_launch_ms": wta_ms / launches,
        "hbm_view": ({"achieved_gbs": traffic / (wta_ms / launches / 1000.0) / 1e9,
                      "peak_gbs": hbm_peak,
                      "frac": traffic / (wta_ms / launches / 1000.0) / 1e9 / hbm_peak,
                      "note": "ncu DRAM bytes per launch over the live launch time: the "
                              "sweep is not HBM-bound"}
                     if traffic and wta_ms > 0 else None),
        "pipeline_census_frac": CENSUS["textured"] * value / world / alu_peak,
        "hbm_frac_pipeline": 21.8e6 * value / world / (hbm_peak * 1e9),
    }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        pairs_cpu = cpu_pairs(args.cpu_pairs)
        tcpu, kind = reference_chain(pairs_cpu)
        cpu = {"value": len(pairs_cpu) / tcpu, "unit": "pairs/s", "cores": os.cpu_count(),
               "kind": kind, "cpu_model": cpu_model(),
               "sample": f"{len(pairs_cpu)} C1 pairs (960x540 D=64) through oracle/_ref "
                         "(unmodified reference, OpenMP all cores) + restated cloud"}
        if omp_threads(1):  # also one thread
            t1, _ = reference_chain(pairs_cpu[:1])
            cpu["single_thread_value"] = 1.0 / t1
            omp_threads(os.cpu_count())
    if cpu is not None and args.cpu_configs:
        cpu["side_by_side"] = cpu_side_by_side()
    stage_ms_per_pair = {k: v[0] / frames_timed for k, v in stages.items()}
    ext = None if (args.no_extensions or world > 1) else extensions(ss, ctxs, step_device, barrier, stream, F,
                                                     Lh_first=Lh[0].numpy(), Rh_first=Rh[0].numpy(),
                                                     od=od)
    line = {
        "metric": "stereo pairs/sec at 960x540 D=64", "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/int32/f32-filter/f64", "data": "synthetic",
        "config": config_dict(args, world),
        "ms_per_pair": ms_max / args.steps / F,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(stats["kernel_launches"]),
        "roofline": roofline, "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "stage_ms_per_pair": stage_ms_per_pair,
        "exact_resolves": {"wta_pixels": stats["wta_resolved"],
                           "refine_repicks": stats["refine_resolved"],
                           "frames": stats["frames"]},
        "extensions": ext,
    }
    print(json.dumps(line), flush=True)
    for c in ctxs:
        c.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
