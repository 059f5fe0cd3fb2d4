"""Normals parity against the reference's eigensolver (cloud.cpp:62-90).

The reference fits each normal with Eigen::SelfAdjointEigenSolver<Matrix3d>
(cloud.cpp:78) and keeps it iff lambda1 > 1e-9 max(1, lambda2) (cloud.cpp:81),
else falls back to the sight ray. Eigen is not vendored, so the oracle
restates Eigen 3.4.0's algorithm operation by operation (oracle/ss_oracle.c:
eigen3_sym): pinned here as an eigensolver against LAPACK, and used as the
checker of the GPU's normals and fit/fallback decisions.

Contract (GPU vs restated Eigen):
  * decision: identical wherever the oracle's test is not within a relative
    margin of 1e-6 of its threshold; the exceptions are counted (and 0 here);
  * fitted normals: within 1e-3 rad where the oracle's eigen gap
    (l1 - l0) / l2 >= 1e-3 (the normal is ill-conditioned below that);
  * fallback normals: the sight ray within 1e-6 rad.
"""
import numpy as np
import pytest


def _ang(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.arctan2(np.linalg.norm(np.cross(a, b), axis=-1), np.abs((a * b).sum(-1)))


# ---------------- CPU: the restated Eigen solver ----------------

def test_eigen_restatement_vs_lapack(orc):
    rng = np.random.default_rng(7)
    worst_val = worst_res = 0.0
    for t in range(6000):
        k = t % 5
        if k == 0:
            A = rng.standard_normal((3, 3))
            A = A + A.T
        elif k == 1:  # plane-like neighbourhood covariance
            P = rng.standard_normal((49, 3)) * [10, 10, 1e-3]
            P = P @ np.linalg.qr(rng.standard_normal((3, 3)))[0]
            P -= P.mean(0)
            A = P.T @ P
        elif k == 2:  # line-like (rank ~1)
            P = rng.standard_normal((49, 1)) * [[1, 2, 3]] + rng.standard_normal((49, 3)) * 1e-9
            P -= P.mean(0)
            A = P.T @ P
        elif k == 3:  # diagonal / repeated eigenvalues
            A = np.diag(rng.choice([0.0, 1.0, 2.0], 3))
        else:  # tiny and huge scales
            A = rng.standard_normal((3, 3)) * 10.0 ** rng.integers(-150, 150)
            A = A + A.T
        ev, vec, ok = orc.eigen3_sym(A)
        assert ok
        w = np.linalg.eigvalsh(A)
        s = max(np.abs(w).max(), 1e-300)
        worst_val = max(worst_val, np.abs(ev - w).max() / s)
        worst_res = max(worst_res, np.abs(A @ vec - vec * ev).max() / s)
        assert np.all(np.diff(ev) >= 0)  # ascending, as Eigen sorts
        assert np.allclose(vec.T @ vec, np.eye(3), atol=1e-12)
    assert worst_val < 1e-13 and worst_res < 1e-13, (worst_val, worst_res)


def test_eigen_restatement_exact_cases(orc):
    ev, vec, ok = orc.eigen3_sym(np.zeros((3, 3)))
    assert ok and np.all(ev == 0) and np.array_equal(vec, np.eye(3))
    ev, vec, ok = orc.eigen3_sym(np.diag([3.0, 1.0, 2.0]))
    assert ok and np.array_equal(ev, [1.0, 2.0, 3.0])
    assert np.array_equal(np.abs(vec), np.eye(3)[:, [1, 2, 0]])


def test_oracle_cloud_spec_examples(orc):
    """SPEC.md:185-187 on the restated cloud (on-axis point, fronto-parallel
    normal, slanted plane)."""
    rig = dict(fx=1000.0, fy=1000.0, cx=10.0, cy=8.0, width=21, height=17, baseline_mm=5.0)
    d = np.full((17, 21), 50.0, np.float32)
    v = np.ones((17, 21), np.uint8)
    cl = orc.disparity_to_cloud(d, v, np.zeros((17, 21, 3), np.uint8), rig)
    assert np.allclose(cl.points[cl.index[8, 10]], [0.0, 0.0, 100.0])
    assert np.all(_ang(cl.normals, [0, 0, -1.0]) < 1e-3)
    yy, xx = np.mgrid[0:17, 0:21]
    a = 0.3
    z = 100.0 / (1.0 - a * (xx - 10.0) / 1000.0)
    cl = orc.disparity_to_cloud((5000.0 / z).astype(np.float32), v, np.zeros((17, 21, 3), np.uint8),
                                rig)
    n_true = np.array([a, 0.0, -1.0]) / np.sqrt(1 + a * a)
    assert np.all(_ang(cl.normals, n_true) < np.radians(1.0))
    assert np.all(cl.decision > 0)


# ---------------- GPU vs restated Eigen ----------------

def _maps(W, H):
    """Disparity maps whose neighbourhoods cover clear fits, rank-1 lines
    (fallback), sparse masks (count < 3) and mixtures."""
    from oracle.oracle import Oracle
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    orc = Oracle("orc")
    rng = np.random.default_rng(3)
    L, R, _ = stereo_pair("textured", W, H, 24, seed=2)
    p = params_for(24)
    d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p), L, R, p)
    yield "refined", d, v
    lines = np.zeros((H, W), np.uint8)
    lines[:, ::9] = 1            # vertical 1-px lines: rank-1 neighbourhoods
    lines[::11, :] = 1           # horizontal lines crossing them
    lines[np.arange(H), np.arange(H) % W] = 1  # a diagonal
    yield "lines", d, lines
    sparse = (rng.random((H, W)) < 0.04).astype(np.uint8)  # mostly < 3 neighbours
    yield "sparse", d, sparse
    mix = ((rng.random((H, W)) < 0.5) | (lines == 1)).astype(np.uint8)
    yield "mixed", d + rng.standard_normal(d.shape).astype(np.float32) * 0.3, mix


@pytest.mark.gpu
def test_gpu_normals_and_decisions_vs_restated_eigen():
    import paper_2007_12623_b200 as ss
    from oracle.oracle import Oracle
    from paper_2007_12623_b200.synth import as_rgb, default_rig, stereo_pair
    orc = Oracle("orc")
    W, H = 200, 150
    rigs = [default_rig(W, H), dict(fx=3000.0, fy=2500.0, cx=40.0, cy=120.0, width=W, height=H,
                                    baseline_mm=60.0)]
    L = stereo_pair("textured", W, H, 24, seed=2)[0]
    totals = {"points": 0, "fitted": 0, "fallback": 0, "near_threshold": 0}
    for rig in rigs:
        for name, d, v in _maps(W, H):
            want = orc.disparity_to_cloud(d, v, as_rgb(L), rig)
            got = ss.disparity_to_cloud(d, v, as_rgb(L), rig)
            assert np.array_equal(got.index, want.index), name
            near = np.abs(want.decision) <= 1e-6
            dec = want.decision > 0
            bad = (got.fitted.astype(bool) != dec) & ~near
            assert not bad.any(), f"{name}: {int(bad.sum())} fit/fallback decisions differ"
            totals["points"] += len(dec)
            totals["fitted"] += int(dec.sum())
            totals["fallback"] += int((~dec).sum())
            totals["near_threshold"] += int(near.sum())
            ok = dec & (want.eigen_gap >= 1e-3) & got.fitted.astype(bool)
            if ok.any():
                assert _ang(got.normals[ok], want.normals[ok]).max() <= 1e-3, name
            fb = ~dec & ~near
            if fb.any():
                assert _ang(got.normals[fb], want.normals[fb]).max() <= 1e-6, name
            # orientation (cloud.cpp:89): towards the camera; a grazing normal
            # (n . p-hat within 1e-6 of 0) may flip on the float copy of p
            cos_np = np.sum(got.normals * got.points, axis=1) / np.linalg.norm(got.points, axis=1)
            assert np.all(cos_np <= 1e-6), name
    assert totals["fitted"] > 1000 and totals["fallback"] > 1000, totals
    assert totals["near_threshold"] == 0, totals
