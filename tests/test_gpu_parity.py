"""GPU parity: the sm_100a path vs the reference (golden vectors) and the oracle.

Bar (BASELINE.json north_star):
  * WTA disparity/valid: bit-exact. Near-tie / near-threshold pixels are
    resolved in exact FP64 on the device, so no exception is needed; their
    count is reported (ctx stats) and checked to be small.
  * cleanup: bit-exact including stale values under invalid pixels.
  * refine (exact FP64 state): bit-exact disparity and RefineTrace.
  * cloud: index/colors/pixels identical, points bit-exact (same FP64 ops),
    normals within 1e-3 rad where the oracle's eigen gap >= 1e-3.
All calls go through the C-ABI (ctypes) into libstereoscan_b200.so.
"""
import math

import numpy as np
import pytest

from conftest import GOLDEN_CHAINS, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    if ss.device_count() < 1:
        pytest.fail("no CUDA device visible to the GPU parity tests")
    return ss


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64, 1: np.uint8}[a.dtype.itemsize])


def assert_map_equal(got, want, what):
    gd, gv = got
    wd, wv = want
    nv = int((gv != wv).sum())
    nd = int((bits(gd) != bits(wd)).sum())
    assert nv == 0 and nd == 0, f"{what}: {nv} validity and {nd} disparity mismatches"


# ---------- golden vectors (generated from the real reference) ----------

@pytest.mark.parametrize("name", GOLDEN_CHAINS)
def test_golden_chain_stage_isolated(ss, name):
    g = load_golden(name)
    p = g["params"]
    assert_map_equal(ss.compute_disparity(g["left"], g["right"], p),
                     (g["wta_disp"], g["wta_valid"]), f"{name} WTA")
    assert_map_equal(ss.cleanup_pass(g["wta_disp"], g["wta_valid"], p),
                     (g["clean_disp"], g["clean_valid"]), f"{name} cleanup")
    if "trace_discrete" in g:
        rd, rv, td, ts = ss.refine_disparities(g["clean_disp"], g["clean_valid"], g["left"],
                                               g["right"], p, trace=True)
        assert np.array_equal(td, g["trace_discrete"]), f"{name} trace o"
        assert np.array_equal(bits(ts), bits(g["trace_smooth"])), f"{name} trace d"
    else:
        rd, rv = ss.refine_disparities(g["clean_disp"], g["clean_valid"], g["left"], g["right"], p)
    assert_map_equal((rd, rv), (g["refine_disp"], g["refine_valid"]), f"{name} refine")


def test_golden_kats(ss):
    g = load_golden("shift7")
    d, v = ss.compute_disparity(g["left"], g["right"], g["params"])
    assert_map_equal((d, v), (g["wta_disp"], g["wta_valid"]), "shift7")
    assert v.sum() > 0 and np.all(d[v == 1] == 7.0)
    g = load_golden("uniform")
    d, v = ss.compute_disparity(g["left"], g["right"], g["params"])
    assert v.sum() == 0


def test_golden_cleanup_parts(ss):
    g = load_golden("spikes")
    for r in (3, 5, 10):
        assert_map_equal(ss.remove_outliers(g["disp"], g["valid"], r, 2.5),
                         (g[f"ro{r}_disp"], g[f"ro{r}_valid"]), f"remove_outliers r={r}")
    od, ov = ss.remove_outliers(g["disp"], g["valid"], 5, 2.5)
    assert_map_equal(ss.fill_holes(od, ov, "radial", 50, 4),
                     (g["radial_disp"], g["radial_valid"]), "radial fill")
    assert_map_equal(ss.fill_holes(od, ov, "disc", 20, ss.disc_fill_min_support(20)),
                     (g["disc_disp"], g["disc_valid"]), "disc fill")
    assert_map_equal(ss.cleanup_pass(g["disp"], g["valid"], g["params"]),
                     (g["clean_disp"], g["clean_valid"]), "cleanup")


def test_golden_stale_values(ss):
    g = load_golden("stripes")
    cd, cv = ss.cleanup_pass(g["in_disp"], g["in_valid"], g["params"])
    assert_map_equal((cd, cv), (g["clean_disp"], g["clean_valid"]), "stripes cleanup")
    assert_map_equal(ss.refine_disparities(cd, cv, g["left"], g["right"], g["params"]),
                     (g["refine_disp"], g["refine_valid"]), "stripes refine")


# ---------- oracle equivalence on seeded inputs ----------

def test_random_pairs_vs_oracle(ss, orc):
    """100 random 64x64 pairs, exact."""
    from paper_2007_12623_b200.synth import params_for
    rng = np.random.default_rng(2024)
    p = params_for(16)
    for _ in range(100):
        L = rng.integers(0, 256, (64, 64), dtype=np.uint8)
        R = np.roll(L, int(rng.integers(0, 12)), axis=1)
        R = np.clip(R.astype(int) + rng.integers(-2, 3, R.shape), 0, 255).astype(np.uint8)
        assert_map_equal(ss.compute_disparity(L, R, p), orc.compute_disparity(L, R, p), "random")


def test_random_fields_remove_outliers(ss, orc):
    """random fields with 20% spikes vs the 8-ray rule."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        f = (10 + rng.standard_normal((48, 48)).cumsum(1) * 0.3).astype(np.float32)
        sp = rng.random(f.shape) < 0.2
        f[sp] += rng.uniform(-12, 12, sp.sum()).astype(np.float32)
        v = (rng.random(f.shape) > 0.1).astype(np.uint8)
        r = int(rng.integers(1, 15))
        assert_map_equal(ss.remove_outliers(f, v, r, 2.5), orc.remove_outliers(f, v, r, 2.5),
                         "outliers")


def test_remove_outliers_long_rays(ss, orc):
    """Rays longer than one 32-bit word of the edge bitmaps, ragged sizes,
    smooth fields with sparse spikes and holes (every direction must decide)."""
    rng = np.random.default_rng(11)
    for h, w in ((131, 203), (77, 64), (33, 95), (1, 40), (40, 1)):
        base = 20 + np.add.outer(np.arange(h) * 0.05, np.arange(w) * 0.03)
        f = (base + rng.standard_normal((h, w)) * 0.2).astype(np.float32)
        sp = rng.random(f.shape) < 0.01
        f[sp] += rng.uniform(-20, 20, sp.sum()).astype(np.float32)
        v = (rng.random(f.shape) > 0.02).astype(np.uint8)
        for r in (1, 5, 31, 32, 33, 40, 64, 70):
            assert_map_equal(ss.remove_outliers(f, v, r, 2.5), orc.remove_outliers(f, v, r, 2.5),
                             f"outliers {h}x{w} r={r}")


def test_fill_holes_properties(ss, orc):
    """never touches valid pixels; support threshold honoured."""
    rng = np.random.default_rng(9)
    f = rng.uniform(5, 30, (64, 80)).astype(np.float32)
    v = (rng.random(f.shape) > 0.6).astype(np.uint8)
    for mode, radius, sup in (("radial", 50, 4), ("radial", 7, 8), ("disc", 20, 314),
                              ("disc", 6, 30)):
        got = ss.fill_holes(f, v, mode, radius, sup)
        assert_map_equal(got, orc.fill_holes(f, v, 0 if mode == "radial" else 1, radius, sup),
                         f"fill {mode} r={radius}")
        assert np.array_equal(bits(got[0][v == 1]), bits(f[v == 1]))


@pytest.mark.parametrize("kind,W,H,D", [("textured", 960, 540, 64), ("lowtex", 960, 540, 64),
                                        ("textured", 1920, 1080, 128)])
def test_full_size_chain_vs_oracle(ss, orc, kind, W, H, D):
    """C1 / C2 / C3 end to end, stage-isolated and chained, bit-exact."""
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    L, R, _ = stereo_pair(kind, W, H, D, seed=1234)
    p = params_for(D)
    want = orc.compute_disparity(L, R, p)
    got = ss.compute_disparity(L, R, p)
    assert_map_equal(got, want, f"{kind} WTA")
    wc = orc.cleanup_pass(*want, p)
    assert_map_equal(ss.cleanup_pass(*want, p), wc, f"{kind} cleanup")
    wr = orc.refine_disparities(*wc, L, R, p)
    assert_map_equal(ss.refine_disparities(*wc, L, R, p), wr, f"{kind} refine")


def test_refine_trace_full_size(ss, orc):
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    L, R, _ = stereo_pair("lowtex", 480, 270, 32, seed=77)
    p = params_for(32)
    d, v = orc.cleanup_pass(*orc.compute_disparity(L, R, p), p)
    a = orc.refine_disparities(d, v, L, R, p, trace=True)
    b = ss.refine_disparities(d, v, L, R, p, trace=True)
    for x, y, what in zip(a, b, ["disp", "valid", "trace o", "trace d"]):
        assert np.array_equal(bits(x), bits(y)), what
    assert np.all(np.abs(b[2] - b[3])[:, v == 1] <= 5.0)


def test_default_params_negative_disparities(ss, orc):
    from paper_2007_12623_b200.synth import stereo_pair
    L, R, _ = stereo_pair("textured", 320, 200, 24, seed=8)
    R = np.roll(R, 16, axis=1)
    p = dict(d_min=-20, d_max=80)
    want = orc.compute_disparity(L, R, p)
    assert_map_equal(ss.compute_disparity(L, R, p), want, "default WTA")
    wc = orc.cleanup_pass(*want, p)
    assert_map_equal(ss.cleanup_pass(*want, p), wc, "default cleanup")
    assert_map_equal(ss.refine_disparities(*wc, L, R, p), orc.refine_disparities(*wc, L, R, p),
                     "default refine")


@pytest.mark.parametrize("d_min,d_max", [(0, 199), (-40, 199), (0, 255), (3, 9)])
def test_wide_and_narrow_disparity_ranges(ss, orc, d_min, d_max):
    """Sweep geometry at the edges: 13-15 sweep warps (the fast path's limit is
    15 + the merge warp), the generic exact path beyond, and fewer candidates
    than one 16-wide warp block (masked lanes, windows rebuilt)."""
    from paper_2007_12623_b200.synth import stereo_pair
    L, R, _ = stereo_pair("textured", 400, 96, 48, seed=12)
    R = np.roll(R, 30, axis=1)
    p = dict(d_min=d_min, d_max=d_max)
    want = orc.compute_disparity(L, R, p)
    assert_map_equal(ss.compute_disparity(L, R, p), want, f"WTA {d_min}..{d_max}")
    wc = orc.cleanup_pass(*want, p)
    assert_map_equal(ss.refine_disparities(*wc, L, R, p), orc.refine_disparities(*wc, L, R, p),
                     f"refine {d_min}..{d_max}")


@pytest.mark.parametrize("window", [3, 7, 9, 13])
def test_other_windows(ss, orc, window):
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    L, R, _ = stereo_pair("textured", 120, 80, 16, seed=window)
    p = params_for(16, window=window)
    want = orc.compute_disparity(L, R, p)
    assert_map_equal(ss.compute_disparity(L, R, p), want, f"w{window} WTA")
    wc = orc.cleanup_pass(*want, p)
    assert_map_equal(ss.refine_disparities(*wc, L, R, p), orc.refine_disparities(*wc, L, R, p),
                     f"w{window} refine")


def test_edge_shapes(ss, orc):
    from paper_2007_12623_b200.synth import params_for
    p = params_for(8)
    rng = np.random.default_rng(3)
    for (h, w) in [(1, 1), (5, 40), (11, 11), (12, 13), (40, 9), (23, 57)]:
        L = rng.integers(0, 256, (h, w), dtype=np.uint8)
        R = rng.integers(0, 256, (h, w), dtype=np.uint8)
        want = orc.compute_disparity(L, R, p)
        assert_map_equal(ss.compute_disparity(L, R, p), want, f"{h}x{w} WTA")
        wc = orc.cleanup_pass(*want, p)
        assert_map_equal(ss.cleanup_pass(*want, p), wc, f"{h}x{w} cleanup")
        assert_map_equal(ss.refine_disparities(*wc, L, R, p), orc.refine_disparities(*wc, L, R, p),
                         f"{h}x{w} refine")
    e = np.zeros((0, 0), np.uint8)
    d, v = ss.compute_disparity(e, e, p)
    assert d.shape == (0, 0)


def test_errors_match_reference(ss):
    L = np.zeros((20, 30), np.uint8)
    R = np.zeros((20, 31), np.uint8)
    with pytest.raises(ss.InvalidArgument) as e:
        ss.compute_disparity(L, R, ss.StereoParams())
    assert str(e.value) == "compute_disparity: image sizes differ"
    with pytest.raises(ss.StereoError) as e:
        ss.compute_disparity(L, L, ss.StereoParams(window=10))
    assert str(e.value) == "stereo: window must be odd and >= 3"


def test_to_gray_exact(ss, orc):
    rng = np.random.default_rng(0)
    rgb = rng.integers(0, 256, (57, 91, 3), dtype=np.uint8)
    assert np.array_equal(ss.to_gray(rgb), orc.to_gray(rgb))
    # every (r, g, b) corner value near .5 rounding boundaries
    grid = np.stack(np.meshgrid(np.arange(0, 256, 3), np.arange(0, 256, 5),
                                np.arange(0, 256, 7), indexing="ij"), -1).reshape(1, -1, 3)
    assert np.array_equal(ss.to_gray(grid.astype(np.uint8)), orc.to_gray(grid.astype(np.uint8)))


def test_cloud_vs_oracle(ss, orc):
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    L, R, _ = stereo_pair("textured", 320, 240, 32, seed=4)
    p = params_for(32)
    d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p), L, R, p)
    rig = default_rig(320, 240)
    rgb = as_rgb(L)
    want = orc.disparity_to_cloud(d, v, rgb, rig)
    got = ss.disparity_to_cloud(d, v, rgb, rig)
    assert np.array_equal(got.index, want.index)
    assert np.array_equal(bits(got.points), bits(want.points))
    assert np.array_equal(got.colors, want.colors) and np.array_equal(got.pixels, want.pixels)
    cosang = np.clip(np.abs(np.sum(got.normals * want.normals, axis=1)), 0, 1)
    ang = np.arccos(cosang)
    ok = want.eigen_gap >= 1e-3
    assert ok.mean() > 0.9
    assert np.all(ang[ok] <= 1e-3), f"max normal angle {ang[ok].max()}"
    # orientation: camera-facing everywhere (cloud.cpp:89)
    assert np.all(np.sum(got.normals * got.points, axis=1) <= 0)


def test_cloud_kats(ss):
    rig = dict(fx=1000.0, fy=1000.0, cx=10.0, cy=8.0, width=21, height=17, baseline_mm=5.0)
    d = np.full((17, 21), 50.0, np.float32)
    v = np.ones((17, 21), np.uint8)
    cl = ss.disparity_to_cloud(d, v, np.zeros((17, 21, 3), np.uint8), rig)
    assert np.allclose(cl.points[cl.index[8, 10]], [0.0, 0.0, 100.0])
    assert np.allclose(cl.normals, [0.0, 0.0, -1.0], atol=1e-3)
    yy, xx = np.mgrid[0:17, 0:21]
    a = 0.3
    z = 100.0 / (1.0 - a * (xx - 10.0) / 1000.0)
    cl = ss.disparity_to_cloud((5000.0 / z).astype(np.float32), v, None, rig)
    n_true = np.array([a, 0.0, -1.0]) / math.sqrt(1 + a * a)
    assert np.all(np.abs(cl.normals @ n_true) > math.cos(math.radians(1.0)))
    with pytest.raises(ss.StereoError) as e:
        ss.disparity_to_cloud(d, v, None, dict(rig, fx=0.0))
    assert str(e.value) == "intrinsics: fx must be > 0"


def test_batch_api_matches_per_stage(ss, orc):
    """Frames are independent: a batch gives the per-frame answers, for any
    batch size (the determinism row of SURVEY.md §8e)."""
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D, n = 256, 160, 32, 5
    p = params_for(D)
    pairs = [stereo_pair("textured" if i % 2 else "lowtex", W, H, D, seed=50 + i)
             for i in range(n)]
    Ls = np.stack([as_rgb(a) for a, _, _ in pairs])
    Rs = np.stack([as_rgb(b) for _, b, _ in pairs])
    rig = default_rig(W, H)
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    outs = []
    for mb in (1, 2, 5):
        ctx = ss.StereoContext(0, W, H, mb, ss.StereoParams(**p), ss.StereoRig(**rig))
        outs.append(ctx.run(Ls, Rs, flags))
        st = ctx.stats()
        assert st["frames"] == n and st["kernel_launches"] > 0
        ctx.close()
    for o in outs[1:]:
        for k in ("disparity", "valid", "index", "n_points"):
            assert np.array_equal(bits(o[k]), bits(outs[0][k])), k
    for i, (L, R, _) in enumerate(pairs):
        d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p),
                                      L, R, p)
        assert_map_equal((outs[0]["disparity"][i], outs[0]["valid"][i]), (d, v), f"frame {i}")
        cl = orc.disparity_to_cloud(d, v, as_rgb(L), rig)
        k = outs[0]["n_points"][i]
        assert k == len(cl.points)
        assert np.array_equal(outs[0]["points"][i][:k], cl.points.astype(np.float32))
        assert np.array_equal(outs[0]["colors"][i][:k], cl.colors)


def _random_params(rng):
    """One seeded draw over every StereoParams field the validator accepts,
    including smoothing radii that take the generic gather (R != 15) and the
    global-memory gather (tile too large for shared memory), eta <= 0,
    min_zncc <= 0 and zero cleanup / refine iterations."""
    d_min = int(rng.integers(-12, 6))
    return dict(window=int(rng.choice([3, 5, 7, 9, 11, 13])), d_min=d_min,
                d_max=d_min + int(rng.integers(3, 41)),
                neighbor_jump_threshold=float(rng.choice([0.5, 1.0, 2.5, 6.0])),
                outlier_radius_start=int(rng.integers(1, 16)),
                outlier_radius_step=int(rng.integers(1, 13)),
                cleanup_iterations=int(rng.integers(0, 5)),
                fill_radius_radial=int(rng.integers(1, 61)),
                fill_radius_disc=int(rng.integers(1, 26)),
                smoothing_radius=int(rng.choice([1, 4, 15, 15, 16, 31, 33, 70, 120])),
                alpha=float(rng.choice([0.0, 0.1, 0.35, 1.0])),
                eta_smooth=float(rng.choice([-0.02, 0.0, 0.01, 0.05])),
                refine_iterations=int(rng.integers(0, 5)),
                min_zncc=float(rng.choice([-0.5, 0.0, 0.3, 0.5, 0.9])))


@pytest.mark.parametrize("seed", range(36))
def test_random_parameter_sets(ss, orc, seed):
    """Every stage bit-exact to the oracle under a random parameter set
    (params.hpp:7-24 fields) and a ragged image size, stage-isolated: WTA,
    cleanup, refine."""
    from paper_2007_12623_b200.synth import stereo_pair
    rng = np.random.default_rng(1000 + seed)
    p = _random_params(rng)
    kind = "lowtex" if seed % 3 == 0 else "textured"
    w, h = [(144, 88), (97, 61), (300, 40), (33, 150)][seed % 4]
    L, R, _ = stereo_pair(kind, w, h, 24, seed=seed)
    R = np.roll(R, -p["d_min"] // 2, axis=1)
    want = orc.compute_disparity(L, R, p)
    assert_map_equal(ss.compute_disparity(L, R, p), want, f"WTA {p}")
    wc = orc.cleanup_pass(*want, p)
    assert_map_equal(ss.cleanup_pass(*want, p), wc, f"cleanup {p}")
    assert_map_equal(ss.refine_disparities(*wc, L, R, p), orc.refine_disparities(*wc, L, R, p),
                     f"refine {p}")


@pytest.mark.parametrize("seed", [3, 7])
def test_batch_api_random_params(ss, orc, seed):
    """The fused batch chain (one context, frames in one launch) under a
    random parameter set equals the oracle's per-stage chain per frame."""
    from paper_2007_12623_b200.synth import as_rgb, default_rig, stereo_pair
    rng = np.random.default_rng(2000 + seed)
    p = _random_params(rng)
    W, H, n = 200, 120, 3
    pairs = [stereo_pair("textured", W, H, 24, seed=seed * 10 + i) for i in range(n)]
    Ls = np.stack([as_rgb(a) for a, _, _ in pairs])
    Rs = np.stack([as_rgb(b) for _, b, _ in pairs])
    ctx = ss.StereoContext(0, W, H, n, ss.StereoParams(**p), ss.StereoRig(**default_rig(W, H)))
    out = ctx.run(Ls, Rs, ss.SS_OUT_DISPARITY)
    ctx.close()
    for i, (L, R, _) in enumerate(pairs):
        d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p),
                                      L, R, p)
        assert_map_equal((out["disparity"][i], out["valid"][i]), (d, v), f"frame {i} {p}")


@pytest.mark.parametrize("seed", range(6))
def test_cloud_random_rigs(ss, orc, seed):
    """Back-projection under random intrinsics / baselines and disparity
    fields with negative, zero and tiny values (cloud.cpp:43-60 skips d <= 0):
    index, points, colours bit-exact; normals within 1e-3 rad where the
    oracle's eigen gap >= 1e-3."""
    from paper_2007_12623_b200.synth import as_rgb, params_for, stereo_pair
    rng = np.random.default_rng(600 + seed)
    W, H = [(200, 120), (97, 61), (64, 150)][seed % 3]
    L, R, _ = stereo_pair("textured", W, H, 24, seed=seed)
    p = params_for(24, d_min=-4)
    d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p), L, R, p)
    d = d.copy()
    d[rng.random(d.shape) < 0.02] = 0.0
    d[rng.random(d.shape) < 0.01] = 1e-6
    rig = dict(fx=float(rng.uniform(200, 3000)), fy=float(rng.uniform(200, 3000)),
               cx=float(rng.uniform(0, W - 1)), cy=float(rng.uniform(0, H - 1)),
               width=W, height=H, baseline_mm=float(rng.uniform(0.5, 120)))
    rgb = as_rgb(L)
    want = orc.disparity_to_cloud(d, v, rgb, rig)
    got = ss.disparity_to_cloud(d, v, rgb, rig)
    assert np.array_equal(got.index, want.index)
    assert np.array_equal(bits(got.points), bits(want.points))
    assert np.array_equal(got.colors, want.colors) and np.array_equal(got.pixels, want.pixels)
    ang = np.arccos(np.clip(np.abs(np.sum(got.normals * want.normals, axis=1)), 0, 1))
    ok = want.eigen_gap >= 1e-3
    assert np.all(ang[ok] <= 1e-3), f"max normal angle {ang[ok].max()}"


def test_stereo_frame_entry(ss, orc):
    """ss_stereo_frame (the fused per-frame entry): the
    oracle's chain for one pair, with and without a rig; a cloud request
    without a rig fails like the batch API."""
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D = 200, 120, 24
    L, R, _ = stereo_pair("textured", W, H, D, seed=31)
    p = params_for(D)
    d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p), L, R, p)
    out = ss.stereo_frame(as_rgb(L), as_rgb(R), ss.StereoParams(**p))
    assert_map_equal((out["disparity"][0], out["valid"][0]), (d, v), "stereo_frame")
    rig = default_rig(W, H)
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    out = ss.stereo_frame(L, R, ss.StereoParams(**p), ss.StereoRig(**rig), flags)
    assert_map_equal((out["disparity"][0], out["valid"][0]), (d, v), "stereo_frame gray")
    cl = orc.disparity_to_cloud(d, v, as_rgb(L), rig)
    k = out["n_points"][0]
    assert k == len(cl.points)
    assert np.array_equal(out["points"][0][:k], cl.points.astype(np.float32))
    with pytest.raises(ss.InvalidArgument):
        ss.stereo_frame(L, R, ss.StereoParams(**p), None, flags)


def test_batch_api_odd_frame_size(ss, orc):
    """Frames of an odd pixel count: every frame after the first starts
    unaligned in the packed RGB / gray buffers (the luma kernel's scalar
    path), ragged column strips in the window statistics and the planes."""
    from paper_2007_12623_b200.synth import as_rgb, params_for, stereo_pair
    W, H, D, n = 97, 61, 16, 3
    p = params_for(D)
    pairs = [stereo_pair("textured", W, H, D, seed=70 + i) for i in range(n)]
    Ls = np.stack([as_rgb(a) for a, _, _ in pairs])
    Rs = np.stack([as_rgb(b) for _, b, _ in pairs])
    ctx = ss.StereoContext(0, W, H, n, ss.StereoParams(**p))
    out = ctx.run(Ls, Rs, ss.SS_OUT_DISPARITY)
    ctx.close()
    for i, (L, R, _) in enumerate(pairs):
        assert np.array_equal(orc.to_gray(as_rgb(L)), L)
        d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p),
                                      L, R, p)
        assert_map_equal((out["disparity"][i], out["valid"][i]), (d, v), f"frame {i}")
