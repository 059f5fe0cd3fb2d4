"""Fusion consumer (SPEC.md:440-476 [MODULE] fusion).

The reference has no source for this module, so parity is "unpinned" against
reference code: the oracle restatement (oracle/ss_oracle.c orc_rasterize /
orc_fuse_frame) is held to the SPEC's examples and properties on CPU, and the
GPU (ss_fusion_*) is held bit-exact to the oracle over multi-frame sequences.
"""
import math

import numpy as np
import pytest

RIG = {"fx": 200.0, "fy": 210.0, "cx": 79.5, "cy": 59.5, "width": 160, "height": 120,
       "baseline_mm": 5.0}
I34 = np.hstack([np.eye(3), np.zeros((3, 1))])
EMPTY = {"pos": np.zeros((0, 3)), "normal": np.zeros((0, 3)), "color": np.zeros((0, 3)),
         "weight": np.zeros(0), "color_weight": np.zeros(0)}


def pose_of(rx, ry, rz, t):
    cx, sx, cy, sy, cz, sz = (math.cos(rx), math.sin(rx), math.cos(ry), math.sin(ry),
                              math.cos(rz), math.sin(rz))
    R = (np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]]) @
         np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]]) @
         np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]]))
    return np.hstack([R, np.asarray(t, float).reshape(3, 1)])


def cloud_from_depth(depth, rgb, rig=RIG, valid=None):
    """A StereoCloud-like dict from a depth map (camera frame), raster order."""
    h, w = depth.shape
    valid = np.ones_like(depth, bool) if valid is None else valid
    index = np.full((h, w), -1, np.int32)
    vs, us = np.nonzero(valid)
    index[vs, us] = np.arange(len(us))
    z = depth[vs, us]
    x = z * (us - rig["cx"]) / rig["fx"]
    y = z * (vs - rig["cy"]) / rig["fy"]
    pts = np.stack([x, y, z], 1)
    nrm = np.tile([0.0, 0.0, -1.0], (len(us), 1))
    return index, pts, nrm, rgb[vs, us].reshape(-1, 3).astype(np.uint8)


def one_pixel_cloud(u, v, z, color=(200, 100, 50)):
    d = np.zeros((RIG["height"], RIG["width"]))
    m = np.zeros_like(d, bool)
    d[v, u], m[v, u] = z, True
    rgb = np.zeros((RIG["height"], RIG["width"], 3), np.uint8)
    rgb[v, u] = color
    return cloud_from_depth(d, rgb, valid=m)


# ---------------- SPEC examples on the oracle (CPU) ----------------

def test_rasterize_kats(orc):
    ids, dep = orc.rasterize([[0.0, 0.0, 100.0]], I34, RIG)
    v, u = np.argwhere(ids == 0)[0]
    assert (u, v) == (80, 60)  # floor(79.5 + 0.5), floor(59.5 + 0.5)
    assert dep[v, u] == 100.0
    ids, dep = orc.rasterize([[0.0, 0.0, 100.0], [0.0, 0.0, 50.0]], I34, RIG)
    assert ids[60, 80] == 1 and dep[60, 80] == 50.0  # depth-50 wins
    ids, _ = orc.rasterize([[0.0, 0.0, -10.0]], I34, RIG)
    assert (ids == -1).all()  # behind the camera
    ids, _ = orc.rasterize([[0.0, 0.0, 70.0], [0.0, 0.0, 70.0]], I34, RIG)
    assert ids[60, 80] == 0  # tie -> smaller id


def test_fuse_kats(orc):
    m = orc.fuse_frame(EMPTY, *one_pixel_cloud(80, 60, 10.0), I34, RIG)
    assert len(m["weight"]) == 1  # empty raster cell -> new surfel
    m = orc.fuse_frame(m, *one_pixel_cloud(80, 60, 10.2), I34, RIG)
    assert len(m["weight"]) == 1 and abs(m["pos"][0, 2] - 10.1) < 1e-12
    assert m["weight"][0] == 2.0
    # far beyond the gate: a new surfel
    m2 = orc.fuse_frame(m, *one_pixel_cloud(80, 60, 30.0), I34, RIG)
    assert len(m2["weight"]) == 2
    # colour weight: centre observation > border observation
    c = orc.fuse_frame(EMPTY, *one_pixel_cloud(80, 60, 10.0), I34, RIG)["color_weight"][0]
    b = orc.fuse_frame(EMPTY, *one_pixel_cloud(2, 3, 10.0), I34, RIG)["color_weight"][0]
    assert c > b >= 0.1


def test_fuse_properties(orc):
    rng = np.random.default_rng(0)
    h, w = RIG["height"], RIG["width"]
    depth = 500.0 + rng.normal(0, 0.3, (h, w))
    rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    m = orc.fuse_frame(EMPTY, *cloud_from_depth(depth, rgb), I34, RIG)
    assert len(m["weight"]) == h * w
    # weight cap
    for _ in range(55):
        m = orc.fuse_frame(m, *cloud_from_depth(depth + rng.normal(0, 0.3, (h, w)), rgb), I34, RIG)
    assert m["weight"].max() == 50.0 and len(m["weight"]) == h * w
    # count grows by exactly the unassociated valid pixels
    valid = rng.random((h, w)) < 0.5
    far = depth + 100.0
    before = len(m["weight"])
    m = orc.fuse_frame(m, *cloud_from_depth(far, rgb, valid=valid), I34, RIG)
    assert len(m["weight"]) == before + int(valid.sum())
    # order independence of the averaging within 1e-9
    a, b, c = (one_pixel_cloud(80, 60, z) for z in (100.0, 101.0, 102.5))
    m1 = orc.fuse_frame(orc.fuse_frame(orc.fuse_frame(EMPTY, *a, I34, RIG), *b, I34, RIG), *c, I34, RIG)
    m2 = orc.fuse_frame(orc.fuse_frame(orc.fuse_frame(EMPTY, *a, I34, RIG), *c, I34, RIG), *b, I34, RIG)
    assert abs(m1["pos"][0, 2] - m2["pos"][0, 2]) < 1e-9


def test_noise_averaging(orc):
    # n = 16 noisy observations of a point: fused error std <= 2 sigma / sqrt(n)
    rng = np.random.default_rng(1)
    sigma, errs = 0.5, []
    for _ in range(300):
        m = EMPTY
        for _ in range(16):
            m = orc.fuse_frame(m, *one_pixel_cloud(80, 60, 200.0 + rng.normal(0, sigma)), I34, RIG)
        errs.append(m["pos"][0, 2] - 200.0)
    assert np.std(errs) <= 2 * sigma / 4


# ---------------- GPU vs the oracle ----------------

@pytest.fixture(scope="module")
def ss():
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    if ss.device_count() < 1:
        pytest.fail("no CUDA device visible to the GPU tests")
    return ss


class _Cloud:
    def __init__(self, index, pts, nrm, col):
        self.index, self.points, self.normals, self.colors = index, pts, nrm, col


def _same(a, b):
    for k in ("pos", "normal", "color", "weight", "color_weight"):
        assert a[k].shape == b[k].shape, k
        assert np.array_equal(a[k].view(np.uint64), np.asarray(b[k], np.float64).view(np.uint64)), k


@pytest.mark.gpu
def test_gpu_fusion_sequence_matches_oracle(ss, orc):
    rng = np.random.default_rng(7)
    h, w = RIG["height"], RIG["width"]
    gpu = ss.fusion.SurfelModel(0)
    model = EMPTY
    yy, xx = np.mgrid[0:h, 0:w]
    for f in range(6):
        depth = 400.0 + 0.5 * xx + 0.3 * yy + rng.normal(0, 0.8, (h, w))
        valid = rng.random((h, w)) < 0.85
        rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        pose = pose_of(0.01 * f, -0.008 * f, 0.005 * f, [1.5 * f, -0.7 * f, 0.4 * f])
        idx, pts, nrm, col = cloud_from_depth(depth, rgb, valid=valid)
        nrm = nrm + rng.normal(0, 0.05, nrm.shape)
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        gids, gdep = gpu.rasterize(pose, RIG)
        oids, odep = orc.rasterize(model["pos"], pose, RIG)
        assert np.array_equal(gids, oids) and np.array_equal(gdep.view(np.uint64), odep.view(np.uint64))
        gpu.fuse_frame(_Cloud(idx, pts, nrm, col), pose, RIG)
        model = orc.fuse_frame(model, idx, pts, nrm, col, pose, RIG)
        _same(gpu.download(), model)
    assert len(model["weight"]) > h * w  # some pixels were new in later frames
    gpu.close()


@pytest.mark.gpu
def test_gpu_fusion_device_path(ss, orc):
    """Clouds straight from the batch API's device outputs (float points)."""
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D = 192, 112, 24
    p = params_for(D)
    rig = default_rig(W, H)
    frames = [stereo_pair("textured", W, H, D, seed=s)[:2] for s in (1, 2)]
    Ls = np.stack([as_rgb(f[0]) for f in frames])
    Rs = np.stack([as_rgb(f[1]) for f in frames])
    ctx = ss.StereoContext(0, W, H, 2, ss.StereoParams(**p), ss.StereoRig(**rig))
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    out = ctx.run(Ls, Rs, flags)  # host copies for the oracle
    import torch
    dl, dr = torch.from_numpy(Ls).cuda(), torch.from_numpy(Rs).cuda()
    torch.cuda.synchronize()
    ctx.run_device(2, W, H, dl.data_ptr(), dr.data_ptr(), flags)  # results stay in the ctx
    dev = ctx.device_outputs()
    gpu = ss.fusion.SurfelModel(0)
    model = EMPTY
    N = W * H
    for f in range(2):
        pose = pose_of(0.0, 0.002 * f, 0.0, [0.3 * f, 0.0, 0.0])
        gpu.fuse_device(dev["index"] + 4 * N * f, dev["points"] + 12 * N * f,
                        dev["normals"] + 12 * N * f, dev["colors"] + 3 * N * f, pose, rig,
                        stream=ctx.stream)
        k = int(out["n_points"][f])
        model = orc.fuse_frame(model, out["index"][f], out["points"][f][:k].astype(np.float64),
                               out["normals"][f][:k].astype(np.float64), out["colors"][f][:k],
                               pose, rig)
        _same(gpu.download(), model)
    gpu.close()
    ctx.close()
