"""Compact transfer formats of the batch API (include/ss_stereo.h):
SS_OUT_NORMALS_OCT (octahedral snorm16 normals) and SS_OUT_TRIM (cloud
arrays leave the GPU with n_points entries per frame). Both are opt-in; the
default outputs stay the reference's."""
import numpy as np
import pytest


def _oct_encode(n):
    """The k_cloud_normals encoding, restated in numpy (test helper)."""
    n = np.asarray(n, np.float32)
    a = np.abs(n).sum(-1)
    x, y = n[..., 0] / a, n[..., 1] / a
    neg = n[..., 2] < 0
    xs = np.where(neg, (1 - np.abs(y)) * np.where(x < 0, -1.0, 1.0), x)
    ys = np.where(neg, (1 - np.abs(x)) * np.where(y < 0, -1.0, 1.0), y)
    q = lambda t: np.rint(np.clip(t, -1, 1) * 32767.0).astype(np.int16)  # noqa: E731
    return np.stack([q(xs), q(ys)], -1)


def test_oct_round_trip_error():
    from paper_2007_12623_b200 import decode_oct_normals
    rng = np.random.default_rng(0)
    n = rng.standard_normal((200000, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    n = np.concatenate([n, np.eye(3), -np.eye(3), [[0, 0, -1.0], [1e-9, 0, -1.0]]])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    d = decode_oct_normals(_oct_encode(n)).astype(np.float64)
    ang = np.arctan2(np.linalg.norm(np.cross(d, n), axis=1), (d * n).sum(1))
    assert ang.max() < 1e-4, ang.max()


@pytest.mark.gpu
def test_trim_and_oct_match_full_outputs():
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D, n = 256, 160, 32, 5
    pairs = [stereo_pair("lowtex" if i % 2 else "textured", W, H, D, seed=90 + i) for i in range(n)]
    Ls = np.stack([as_rgb(a) for a, _, _ in pairs])
    Rs = np.stack([as_rgb(b) for _, b, _ in pairs])
    ctx = ss.StereoContext(0, W, H, 2, ss.StereoParams(**params_for(D)),
                           ss.StereoRig(**default_rig(W, H)))
    full = ctx.run(Ls, Rs, ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS)
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS_OCT | ss.SS_OUT_TRIM
    out = ss.StereoContext.alloc_outputs(n, H, W, flags)
    for k in ("points", "colors", "normals_oct"):
        out[k].view(np.uint8).fill(0x55)  # sentinel: trimmed entries past n_points must stay untouched
    ctx.run(Ls, Rs, flags, out=out)
    ctx.close()
    for k in ("disparity", "valid", "index", "n_points"):
        assert np.array_equal(out[k], full[k]), k
    for f in range(n):
        m = int(full["n_points"][f])
        assert m < W * H
        assert np.array_equal(out["points"][f][:m], full["points"][f][:m])
        assert np.array_equal(out["colors"][f][:m], full["colors"][f][:m])
        d = ss.decode_oct_normals(out["normals_oct"][f][:m]).astype(np.float64)
        r = full["normals"][f][:m].astype(np.float64)
        ang = np.arctan2(np.linalg.norm(np.cross(d, r), axis=1), (d * r).sum(1))
        assert ang.max() < 1e-4, ang.max()
        assert np.all(out["points"][f][m:].view(np.uint8) == 0x55)
        assert np.all(out["normals_oct"][f][m:].view(np.uint8) == 0x55)


@pytest.mark.gpu
def test_device_outputs_written_in_place_with_oct():
    """ss_stereo_batch_device writes straight into the caller's buffers (the
    oct normals included) and ss_ctx_device_outputs then names them."""
    import torch

    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D, n = 192, 112, 24, 3
    pairs = [stereo_pair("textured", W, H, D, seed=40 + i) for i in range(n)]
    Ls = torch.from_numpy(np.stack([as_rgb(a) for a, _, _ in pairs])).cuda()
    Rs = torch.from_numpy(np.stack([as_rgb(b) for _, b, _ in pairs])).cuda()
    ctx = ss.StereoContext(0, W, H, n, ss.StereoParams(**params_for(D)),
                           ss.StereoRig(**default_rig(W, H)))
    want = ctx.run(Ls.cpu().numpy(), Rs.cpu().numpy(),
                   ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS)
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS_OCT
    od = ss.StereoContext.alloc_outputs(
        n, H, W, flags,
        alloc=lambda s, dt: torch.empty(s, dtype=torch.from_numpy(np.empty(0, dt)).dtype,
                                        device="cuda"))
    ctx.run_device(n, W, H, Ls.data_ptr(), Rs.data_ptr(), flags,
                   d_out={k: t.data_ptr() for k, t in od.items()})
    ctx.sync()
    dev = ctx.device_outputs()
    assert dev["disparity"] == od["disparity"].data_ptr()
    assert dev["normals_oct"] == od["normals_oct"].data_ptr()
    ctx.close()
    for k in ("disparity", "valid", "index", "n_points"):
        assert np.array_equal(od[k].cpu().numpy(), want[k]), k
    for f in range(n):
        m = int(want["n_points"][f])
        d = ss.decode_oct_normals(od["normals_oct"][f][:m].cpu().numpy()).astype(np.float64)
        r = want["normals"][f][:m].astype(np.float64)
        ang = np.arctan2(np.linalg.norm(np.cross(d, r), axis=1), (d * r).sum(1))
        assert ang.max() < 1e-4


def test_oct_decode_c_abi_matches_python():
    """ss_oct_decode (host C-ABI helper) equals decode_oct_normals."""
    import ctypes as C

    from paper_2007_12623_b200 import _lib as L
    from paper_2007_12623_b200 import decode_oct_normals
    rng = np.random.default_rng(1)
    n = rng.standard_normal((5000, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    enc = np.ascontiguousarray(_oct_encode(n))
    out = np.empty((len(enc), 3), np.float32)
    L.lib().ss_oct_decode(enc.ctypes.data_as(C.c_void_p), len(enc), out.ctypes.data_as(C.c_void_p))
    assert np.allclose(out, decode_oct_normals(enc), atol=2e-7)
