"""Generate the golden vectors in tests/golden/ from the REAL reference.

Runs the unmodified reference sources (oracle/_ref/libss_ref.so, built by
``make -C oracle`` from /root/reference) on small seeded inputs and stores the
inputs and every stage output as compressed .npz fixtures. The fixtures are
committed; this script only runs where /root/reference exists (not on the GPU
box). Re-run with ``python tests/golden/make_golden.py``.

Cases (SPEC.md examples / SURVEY.md §4 pins):
  tex_d16      96x64 textured pair, d in [0,15]: WTA, cleanup, refine (+trace)
  low_d16      96x64 low-texture pair with stripes: same stages
  tex_default  128x72 textured, reference default params d in [-20,80]
  win7/win13   80x56 textured, window 7 / 13 (generic-window path)
  shift7       160x64 texture shifted by 7 px
  uniform      64x48 uniform gray pair
  spikes       48x48 smooth field with 20% spikes: remove_outliers r=3..10,
               fill_holes radial/disc, cleanup_pass
  stripes      96x64 field with invalid stripes holding stale values
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2007_12623_b200.synth import params_for, stereo_pair  # noqa: E402

PARAM_KEYS = ["window", "d_min", "d_max", "neighbor_jump_threshold", "outlier_radius_start",
              "outlier_radius_step", "cleanup_iterations", "fill_radius_radial",
              "fill_radius_disc", "smoothing_radius", "alpha", "eta_smooth",
              "refine_iterations", "min_zncc"]


def pvec(p):
    return np.array([p[k] for k in PARAM_KEYS], np.float64)


def chain(ref, name, L, R, p, trace=False):
    out = dict(left=L, right=R, params=pvec(p))
    d, v = ref.compute_disparity(L, R, p)
    out.update(wta_disp=d, wta_valid=v)
    cd, cv = ref.cleanup_pass(d, v, p)
    out.update(clean_disp=cd, clean_valid=cv)
    if trace:
        rd, rv, td, ts = ref.refine_disparities(cd, cv, L, R, p, trace=True)
        out.update(trace_discrete=td, trace_smooth=ts)
    else:
        rd, rv = ref.refine_disparities(cd, cv, L, R, p)
    out.update(refine_disp=rd, refine_valid=rv)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: wta valid {v.mean():.3f} clean valid {cv.mean():.3f}")


def main():
    ref = Oracle("ref")
    L, R, _ = stereo_pair("textured", 96, 64, 16, seed=11)
    chain(ref, "tex_d16", L, R, params_for(16))
    L, R, _ = stereo_pair("lowtex", 96, 64, 16, seed=12)
    chain(ref, "low_d16", L, R, params_for(16))
    L, R, _ = stereo_pair("textured", 48, 40, 8, seed=13)
    chain(ref, "tex_trace", L, R, params_for(8, refine_iterations=4), trace=True)
    # Reference defaults: d in [-20, 80]; shift the right view so some true
    # disparities are negative.
    L, R, _ = stereo_pair("textured", 128, 72, 24, seed=14)
    R = np.roll(R, 12, axis=1)
    chain(ref, "tex_default", L, R, params_for(1, d_min=-20, d_max=80))
    L, R, _ = stereo_pair("textured", 80, 56, 12, seed=15)
    chain(ref, "win7", L, R, params_for(12, window=7))
    chain(ref, "win13", L, R, params_for(12, window=13))

    rng = np.random.default_rng(16)
    tex = rng.integers(0, 256, (64, 170), dtype=np.uint8)
    L = tex[:, 0:160].copy()
    R = tex[:, 7:167].copy()  # R(u - 7) == L(u): disparity +7
    d, v = ref.compute_disparity(L, R, params_for(16))
    np.savez_compressed(os.path.join(HERE, "shift7.npz"), left=L, right=R,
                        params=pvec(params_for(16)), wta_disp=d, wta_valid=v)

    U = np.full((48, 64), 77, np.uint8)
    d, v = ref.compute_disparity(U, U, params_for(16))
    np.savez_compressed(os.path.join(HERE, "uniform.npz"), left=U, right=U,
                        params=pvec(params_for(16)), wta_disp=d, wta_valid=v)

    # 48x48 smooth field with 20% spikes and some invalid pixels.
    yy, xx = np.mgrid[0:48, 0:48]
    field = (20.0 + 0.15 * xx + 0.05 * yy).astype(np.float32)
    spikes = rng.random((48, 48)) < 0.2
    field = np.where(spikes, field + rng.uniform(3, 15, (48, 48)).astype(np.float32), field)
    valid = (rng.random((48, 48)) > 0.05).astype(np.uint8)
    out = dict(disp=field.astype(np.float32), valid=valid)
    for r in (3, 5, 10):
        od, ov = ref.remove_outliers(field, valid, r, 2.5)
        nd, nv = ref.remove_outliers(field, valid, r, 2.5, naive=True)
        assert np.array_equal(od, nd) and np.array_equal(ov, nv)
        out[f"ro{r}_disp"], out[f"ro{r}_valid"] = od, ov
    od, ov = ref.remove_outliers(field, valid, 5, 2.5)
    rd, rv = ref.fill_holes(od, ov, 0, 50, 4)
    dd, dvv = ref.fill_holes(od, ov, 1, 20, ref.disc_fill_min_support(20))
    out.update(radial_disp=rd, radial_valid=rv, disc_disp=dd, disc_valid=dvv)
    p = params_for(16)
    cd, cv = ref.cleanup_pass(field, valid, p)
    out.update(clean_disp=cd, clean_valid=cv, params=pvec(p))
    np.savez_compressed(os.path.join(HERE, "spikes.npz"), **out)

    # Stale values: invalid stripes whose disparity keeps an old number.
    L, R, _ = stereo_pair("lowtex", 96, 64, 16, seed=17)
    d, v = ref.compute_disparity(L, R, params_for(16))
    v = v.copy()
    v[:, 40:46] = 0
    d = d.copy()
    d[:, 40:46] = 99.0  # stale values under an invalid mask
    cd, cv = ref.cleanup_pass(d, v, params_for(16))
    rd, rv = ref.refine_disparities(cd, cv, L, R, params_for(16))
    np.savez_compressed(os.path.join(HERE, "stripes.npz"), left=L, right=R,
                        params=pvec(params_for(16)), in_disp=d, in_valid=v, clean_disp=cd,
                        clean_valid=cv, refine_disp=rd, refine_valid=rv)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
