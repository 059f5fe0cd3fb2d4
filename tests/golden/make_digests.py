"""SHA-256 digests of the REAL reference's outputs at full size.

The full-size configurations (C1/C2/C3 and the bench's own frames) are too
large to commit as fixtures, so this script commits their digests instead:
``tests/golden/digests.json``. For every case it runs the unmodified reference
sources (``oracle/_ref/libss_ref.so``: ``compute_disparity`` ->
``cleanup_pass`` -> ``refine_disparities``, matcher.cpp:166-211,
cleanup.cpp:111-123, smoothing.cpp:68-159) on the seeded synthetic pair and
records sha256(disparity f32 bytes || valid u8 bytes) after each stage. The
cloud stage (cloud.cpp:14-94) cannot be built (Eigen is absent), so its
digests come from the C restatement and are labelled ``cloud_source:
restatement``: index map and float32 points (the batch API's output type).

Consumers: ``tests/test_full_size_ref.py`` (GPU outputs and the restatement
against these digests) and ``bench.py`` (its own output frames, after the
timed region). Runs only where /root/reference exists; re-run with
``python tests/golden/make_digests.py``.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair  # noqa: E402

OUT = os.path.join(HERE, "digests.json")

# (key, kind, W, H, D, seed, frame). "C1"/"C2"/"C3" are the SURVEY §8 single-pair
# configs; "bench_*" are the first frames each bench.py workload processes.
CASES = [
    ("C1", "textured", 960, 540, 64, 1234, 0),
    ("C2", "lowtex", 960, 540, 64, 1234, 0),
    ("C3", "textured", 1920, 1080, 128, 1234, 0),
    ("bench_c4_0", "textured", 960, 540, 64, 0, 0),
    ("bench_c4_1", "textured", 960, 540, 64, 1, 0),
    ("bench_c4_2", "textured", 960, 540, 64, 2, 0),
    ("bench_c4_3", "textured", 960, 540, 64, 3, 0),
    ("bench_c2_0", "lowtex", 960, 540, 64, 0, 0),
    ("bench_c2_1", "lowtex", 960, 540, 64, 1, 0),
    ("bench_c2_2", "lowtex", 960, 540, 64, 2, 0),
    ("bench_c2_3", "lowtex", 960, 540, 64, 3, 0),
    ("bench_c3_0", "textured", 1920, 1080, 128, 100, 0),
    ("bench_c3_1", "textured", 1920, 1080, 128, 101, 0),
    ("bench_c5_0", "video", 1920, 1080, 128, 0, 0),
    ("bench_c5_1", "video", 1920, 1080, 128, 1, 1),
]


def map_digest(d, v):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d, np.float32).tobytes())
    h.update(np.ascontiguousarray(v, np.uint8).tobytes())
    return h.hexdigest()


def cloud_digests(index, points_f32):
    return (hashlib.sha256(np.ascontiguousarray(index, np.int32).tobytes()).hexdigest(),
            hashlib.sha256(np.ascontiguousarray(points_f32, np.float32).tobytes()).hexdigest())


def case_inputs(kind, W, H, D, seed, frame):
    L, R, _ = stereo_pair(kind, W, H, D, seed=seed, frame=frame)
    return L, R


def main(only=None):
    ref = Oracle("ref")
    orc = Oracle("orc")
    out = json.load(open(OUT)) if os.path.exists(OUT) and only else {}
    for key, kind, W, H, D, seed, frame in CASES:
        if only and key not in only:
            continue
        t0 = time.time()
        L, R = case_inputs(kind, W, H, D, seed, frame)
        p = params_for(D)
        lg, rg = ref.to_gray(as_rgb(L)), ref.to_gray(as_rgb(R))
        assert np.array_equal(lg, L) and np.array_equal(rg, R)
        d, v = ref.compute_disparity(lg, rg, p)
        e = {"kind": kind, "width": W, "height": H, "D": D, "seed": seed, "frame": frame,
             "params": p, "wta": map_digest(d, v), "wta_valid_px": int(v.sum())}
        d, v = ref.cleanup_pass(d, v, p)
        e.update(clean=map_digest(d, v), clean_valid_px=int(v.sum()))
        d, v = ref.refine_disparities(d, v, lg, rg, p)
        e.update(refine=map_digest(d, v), refine_valid_px=int(v.sum()))
        cl = orc.disparity_to_cloud(d, v, as_rgb(L), default_rig(W, H))
        ih, ph = cloud_digests(cl.index, cl.points.astype(np.float32))
        e.update(cloud_source="restatement (cloud.cpp needs Eigen)", n_points=len(cl.points),
                 cloud_index=ih, cloud_points_f32=ph, rig=default_rig(W, H))
        out[key] = e
        print(f"{key}: {time.time() - t0:.1f}s valid {e['refine_valid_px']} points {e['n_points']}",
              flush=True)
    out["_generator"] = ("tests/golden/make_digests.py: oracle/_ref (unmodified reference "
                         "matcher/cleanup/smoothing, -O3 -fopenmp -ffp-contract=off); cloud from "
                         "oracle/ss_oracle.c")
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
