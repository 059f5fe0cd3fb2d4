"""Pins the CPU oracle (the checker) before anything is compared against it.

* restatement (oracle/ss_oracle.c) == golden vectors generated from the real
  reference (tests/golden/*.npz, every stage, fed stage-isolated);
* restatement == compiled reference (oracle/_ref) on random inputs, when the
  reference library is present (this container; it also travels to the box);
* the SPEC.md known-answer tests for the hot path.
"""
import math

import numpy as np
import pytest

from conftest import GOLDEN_CHAINS, load_golden
from paper_2007_12623_b200.synth import params_for, stereo_pair


@pytest.mark.parametrize("name", GOLDEN_CHAINS)
def test_restatement_matches_golden_chain(orc, name):
    g = load_golden(name)
    p = g["params"]
    d, v = orc.compute_disparity(g["left"], g["right"], p)
    assert np.array_equal(v, g["wta_valid"])
    assert np.array_equal(d, g["wta_disp"])
    cd, cv = orc.cleanup_pass(g["wta_disp"], g["wta_valid"], p)
    assert np.array_equal(cv, g["clean_valid"])
    assert np.array_equal(cd.view(np.uint32), g["clean_disp"].view(np.uint32))
    if "trace_discrete" in g:
        rd, rv, td, ts = orc.refine_disparities(g["clean_disp"], g["clean_valid"], g["left"],
                                                g["right"], p, trace=True)
        assert np.array_equal(td, g["trace_discrete"])
        assert np.array_equal(ts.view(np.uint64), g["trace_smooth"].view(np.uint64))
    else:
        rd, rv = orc.refine_disparities(g["clean_disp"], g["clean_valid"], g["left"],
                                        g["right"], p)
    assert np.array_equal(rv, g["refine_valid"])
    assert np.array_equal(rd.view(np.uint32), g["refine_disp"].view(np.uint32))


def test_restatement_golden_kats(orc):
    g = load_golden("shift7")
    d, v = orc.compute_disparity(g["left"], g["right"], g["params"])
    assert np.array_equal(d, g["wta_disp"]) and np.array_equal(v, g["wta_valid"])
    assert v.sum() > 0 and np.all(d[v == 1] == 7.0)
    g = load_golden("uniform")
    d, v = orc.compute_disparity(g["left"], g["right"], g["params"])
    assert v.sum() == 0


def test_restatement_golden_cleanup_parts(orc):
    g = load_golden("spikes")
    for r in (3, 5, 10):
        od, ov = orc.remove_outliers(g["disp"], g["valid"], r, 2.5)
        assert np.array_equal(ov, g[f"ro{r}_valid"]) and np.array_equal(od, g[f"ro{r}_disp"])
    od, ov = orc.remove_outliers(g["disp"], g["valid"], 5, 2.5)
    rd, rv = orc.fill_holes(od, ov, 0, 50, 4)
    assert np.array_equal(rv, g["radial_valid"])
    assert np.array_equal(rd.view(np.uint32), g["radial_disp"].view(np.uint32))
    dd, dv = orc.fill_holes(od, ov, 1, 20, orc.disc_fill_min_support(20))
    assert np.array_equal(dv, g["disc_valid"])
    assert np.array_equal(dd.view(np.uint32), g["disc_disp"].view(np.uint32))
    cd, cv = orc.cleanup_pass(g["disp"], g["valid"], g["params"])
    assert np.array_equal(cv, g["clean_valid"])
    assert np.array_equal(cd.view(np.uint32), g["clean_disp"].view(np.uint32))


def test_restatement_golden_stale_stripes(orc):
    g = load_golden("stripes")
    cd, cv = orc.cleanup_pass(g["in_disp"], g["in_valid"], g["params"])
    assert np.array_equal(cv, g["clean_valid"])
    assert np.array_equal(cd.view(np.uint32), g["clean_disp"].view(np.uint32))
    rd, rv = orc.refine_disparities(cd, cv, g["left"], g["right"], g["params"])
    assert np.array_equal(rd.view(np.uint32), g["refine_disp"].view(np.uint32))


def test_support_constants(orc):
    assert orc.disc_neighbor_count(20) == 1256
    assert orc.disc_fill_min_support(20) == 314


def test_restatement_vs_reference_random_pairs(orc, ref):
    """64x64 random pairs, optimized == naive == restatement."""
    rng = np.random.default_rng(99)
    p = params_for(16)
    for trial in range(20):
        L = rng.integers(0, 256, (64, 64), dtype=np.uint8)
        R = np.roll(L, int(rng.integers(0, 12)), axis=1)
        R = np.clip(R.astype(int) + rng.integers(-3, 4, R.shape), 0, 255).astype(np.uint8)
        a = ref.compute_disparity(L, R, p)
        b = ref.compute_disparity(L, R, p, naive=True)
        c = orc.compute_disparity(L, R, p)
        for x, y in ((a, b), (a, c)):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


def test_restatement_vs_reference_outliers(orc, ref):
    """random fields with 20% spikes vs the 8-ray oracle."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        f = (10 + rng.standard_normal((48, 48)).cumsum(1) * 0.3).astype(np.float32)
        spikes = rng.random(f.shape) < 0.2
        f[spikes] += rng.uniform(-12, 12, spikes.sum()).astype(np.float32)
        v = (rng.random(f.shape) > 0.1).astype(np.uint8)
        r = int(rng.integers(1, 12))
        a = ref.remove_outliers(f, v, r, 2.5, naive=True)
        b = orc.remove_outliers(f, v, r, 2.5)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])


def test_restatement_vs_reference_full_chain(orc, ref):
    L, R, _ = stereo_pair("lowtex", 200, 120, 24, seed=3)
    p = params_for(24)
    a = ref.compute_disparity(L, R, p)
    b = orc.compute_disparity(L, R, p)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    ca = ref.cleanup_pass(*a, p)
    cb = orc.cleanup_pass(*a, p)
    assert np.array_equal(ca[0].view(np.uint32), cb[0].view(np.uint32))
    ra = ref.refine_disparities(*ca, L, R, p, trace=True)
    rb = orc.refine_disparities(*ca, L, R, p, trace=True)
    for x, y in zip(ra, rb):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_zncc_kats(orc):
    """SPEC.md:131-133."""
    rng = np.random.default_rng(1)
    P = rng.integers(20, 120, (11, 11), dtype=np.uint8)
    assert orc.zncc_chessboard(P, P, 5, 5, 5, 5, 11) == pytest.approx(1.0, abs=1e-9)
    A = np.clip(np.rint(1.7 * P.astype(float) + 12), 0, 255).astype(np.uint8)
    assert orc.zncc_chessboard(P, A, 5, 5, 5, 5, 11) == pytest.approx(1.0, abs=1e-2)
    A2 = (2 * P.astype(int) + 12).astype(np.uint8)  # exact affine, no rounding
    assert orc.zncc_chessboard(P, A2, 5, 5, 5, 5, 11) == pytest.approx(1.0, abs=1e-9)
    N = (255 - P.astype(int)).astype(np.uint8)
    assert orc.zncc_chessboard(P, N, 5, 5, 5, 5, 11) == pytest.approx(-1.0, abs=1e-9)
    U = np.full((11, 11), 9, np.uint8)
    assert orc.zncc_chessboard(P, U, 5, 5, 5, 5, 11) is None


def test_params_validate_messages(orc):
    from oracle.oracle import OracleError
    L = np.zeros((16, 16), np.uint8)
    for kw, msg in [(dict(window=4), "stereo: window must be odd and >= 3"),
                    (dict(d_min=5, d_max=5), "stereo: d_min must be < d_max"),
                    (dict(smoothing_radius=0), "stereo: radii must be > 0"),
                    (dict(alpha=1.5), "stereo: alpha must be in [0,1]"),
                    (dict(cleanup_iterations=-1), "stereo: cleanup_iterations must be >= 0"),
                    (dict(refine_iterations=-1), "stereo: refine_iterations must be >= 0")]:
        with pytest.raises(OracleError) as e:
            orc.compute_disparity(L, L, params_for(8, **kw))
        assert str(e.value) == msg and e.value.code == 2


def test_cleanup_and_refine_properties(orc):
    c = np.full((40, 40), 12.0, np.float32)
    v = np.ones((40, 40), np.uint8)
    p = params_for(16)
    d2, v2 = orc.cleanup_pass(c, v, p)
    assert np.array_equal(d2, c) and np.array_equal(v2, v)
    z = np.zeros((40, 40), np.uint8)
    d3, v3 = orc.cleanup_pass(c, z, p)
    assert v3.sum() == 0
    # refine: constant field with consistent images is a fixed point
    rng = np.random.default_rng(5)
    tex = rng.integers(0, 256, (40, 80), dtype=np.uint8)
    L, R = tex[:, 0:40].copy(), tex[:, 12:52].copy()  # disparity +12
    c = np.full((40, 40), 12.0, np.float32)
    m = np.zeros((40, 40), np.uint8)
    m[5:35, 22:35] = 1  # every candidate window fits (u - 17 >= h)
    rd, rv, td, ts = orc.refine_disparities(c, m, L, R, p, trace=True)
    assert np.allclose(rd[m == 1], 12.0, atol=1e-6)
    assert np.all(np.abs(td - ts)[:, m == 1] <= 5.0)


def test_cloud_kats(orc):
    """SPEC.md:185-187."""
    rig = dict(fx=1000.0, fy=1000.0, cx=10.0, cy=8.0, width=21, height=17, baseline_mm=5.0)
    d = np.full((17, 21), 50.0, np.float32)
    v = np.ones((17, 21), np.uint8)
    rgb = np.zeros((17, 21, 3), np.uint8)
    cl = orc.disparity_to_cloud(d, v, rgb, rig)
    i = cl.index[8, 10]
    assert np.allclose(cl.points[i], [0.0, 0.0, 100.0])
    assert np.allclose(cl.normals, [0.0, 0.0, -1.0], atol=1e-3)
    # slanted plane: z = z0 + a x (camera frame) -> disparity = f b / z(u)
    yy, xx = np.mgrid[0:17, 0:21]
    xs = (xx - 10.0) / 1000.0  # x/z
    a, z0 = 0.3, 100.0
    z = z0 / (1.0 - a * xs)  # points with x = z*xs lie on z = z0 + a x
    d = (1000.0 * 5.0 / z).astype(np.float32)
    cl = orc.disparity_to_cloud(d, v, rgb, rig)
    n_true = np.array([a, 0.0, -1.0]) / math.sqrt(1 + a * a)
    cosang = np.abs(cl.normals @ n_true)
    assert np.all(cosang > math.cos(math.radians(1.0)))
