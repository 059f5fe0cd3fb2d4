"""Certified re-picks: after iteration 0 only the pixels whose
smoothed d left their pick's certificate interval are re-scored. The skip
must never change a pick (smoothing.cpp:114-146): every RefineTrace row stays
bit-exact to the reference's restatement under the parameters that shape the
certificates (eta's sign and size, alpha, the candidate-range clamps), and
the skip must actually happen (a small fraction of the pixels re-scored).
"""
import numpy as np
import pytest

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


@pytest.mark.parametrize("kind,eta,alpha,dmin,dmax", [
    ("textured", 0.01, 0.1, 0, 31),
    ("lowtex", 0.01, 0.1, 0, 31),
    ("textured", 0.0, 0.1, 0, 31),      # flat slopes: only the candidate-set cells bound d
    ("lowtex", -0.02, 0.3, 0, 31),      # negative eta: E < 0, slopes reversed
    ("textured", 0.05, 0.0, 0, 31),
    ("textured", 0.01, 0.1, 4, 20),     # clamps at d_min - 5 / d_max + 5 bind
    ("lowtex", 0.5, 1.0, 0, 31),        # steep smoothness term, alpha = 1
    ("textured", -0.5, 0.0, 0, 31),     # steep negative eta: costs can turn negative
    ("lowtex", 1e-6, 0.1, -8, 23),      # near-flat slopes, negative disparities
])
def test_certified_trace_bit_exact(ss, orc, kind, eta, alpha, dmin, dmax):
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    L, R, _ = stereo_pair(kind, 480, 270, 32, seed=91)
    p = params_for(32, eta_smooth=eta, alpha=alpha, d_min=dmin, d_max=dmax)
    d, v = orc.cleanup_pass(*orc.compute_disparity(L, R, p), p)
    a = orc.refine_disparities(d, v, L, R, p, trace=True)
    b = ss.refine_disparities(d, v, L, R, p, trace=True)
    for x, y, what in zip(a, b, ["disp", "valid", "trace o", "trace d"]):
        n = int((bits(x) != bits(y)).sum())
        assert n == 0, f"{what}: {n} mismatches"


def test_certificates_skip_most_repicks(ss):
    """C1-size textured frames through the batch API: after iteration 0 the
    certified path re-scores only a few percent of the (pixel, iteration)
    pairs (~0.5% at C1)."""
    from paper_2007_12623_b200.synth import as_rgb, params_for, stereo_pair
    pairs = [stereo_pair("textured", 960, 540, 64, seed=s)[:2] for s in (3, 4)]
    left = np.stack([as_rgb(l) for l, _ in pairs])
    right = np.stack([as_rgb(r) for _, r in pairs])
    p = params_for(64)
    ctx = ss.StereoContext(max_w=960, max_h=540, max_batch=2, params=p)
    try:
        ctx.reset_stats()
        out = ctx.run(left, right)
        st = ctx.stats()
    finally:
        ctx.close()
    valid = int(out["valid"].sum())
    later = valid * (p["refine_iterations"] - 1)  # (pixel, iteration) pairs after iteration 0
    assert 0 < st["refine_scored"] < 0.05 * later, (st, later)


def test_graph_chain_matches_direct_launches(ss, monkeypatch):
    """The batch chain launched as a captured CUDA graph (from the third call
    of a configuration) returns what the kernel-by-kernel launches return."""
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    frames = [stereo_pair("textured", 320, 192, 32, seed=s)[:2] for s in (5, 6)]
    left = np.stack([as_rgb(l) for l, _ in frames])
    right = np.stack([as_rgb(r) for _, r in frames])
    p = params_for(32)
    rig = default_rig(320, 192)
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD

    def run(no_graphs):
        if no_graphs:
            monkeypatch.setenv("SS_NO_GRAPHS", "1")
        else:
            monkeypatch.delenv("SS_NO_GRAPHS", raising=False)
        ctx = ss.StereoContext(max_w=320, max_h=192, max_batch=2, params=p, rig=rig)
        try:
            outs = [ctx.run(left, right, out_flags=flags) for _ in range(4)]
            return outs, ctx.stats()["graph_launches"]
        finally:
            ctx.close()

    direct, g0 = run(True)
    graphed, g1 = run(False)
    assert g0 == 0 and g1 >= 1, (g0, g1)
    for o in direct + graphed:
        for k in direct[0]:
            assert np.array_equal(o[k], direct[0][k]), k
