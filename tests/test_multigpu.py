"""Multi-rank host logic on CPU (gloo, world_size 2): frame sharding, the
max-over-ranks step time and the frame-ordered gather are independent of the
rank count. The per-frame compute is the CPU oracle here (stand-in for the GPU
call the bench makes on each rank); what is tested is the host side of §8e.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2007_12623_b200.shard import frame_range


def test_frame_range_partitions():
    for n in (0, 1, 5, 256, 1024):
        for world in (1, 2, 3, 8):
            spans = [frame_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, result_path):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2007_12623_b200.shard import gather_frames, max_over_ranks
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("orc")
    p = params_for(8)
    start, end = frame_range(n_frames, rank, world)
    disp, valid = [], []
    for f in range(start, end):
        L, R, _ = stereo_pair("textured", 48, 32, 8, seed=f)
        d, v = orc.compute_disparity(L, R, p)
        disp.append(d)
        valid.append(v)
    local = {"disparity": np.stack(disp) if disp else np.zeros((0, 32, 48), np.float32),
             "valid": np.stack(valid) if valid else np.zeros((0, 32, 48), np.uint8)}
    t = max_over_ranks(float(rank + 1))
    out = gather_frames(local, n_frames, rank, world)
    if rank == 0:
        np.savez(result_path, t=t, **out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_gather_matches_single_rank(tmp_path, orc, world):
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    n_frames = 5
    path = str(tmp_path / "gathered.npz")
    mp.start_processes(_worker, args=(world, _free_port(), n_frames, path), nprocs=world,
                       join=True, start_method="spawn")
    g = np.load(path)
    assert float(g["t"]) == float(world)  # max over ranks
    p = params_for(8)
    for f in range(n_frames):
        L, R, _ = stereo_pair("textured", 48, 32, 8, seed=f)
        d, v = orc.compute_disparity(L, R, p)
        assert np.array_equal(g["disparity"][f], d) and np.array_equal(g["valid"][f], v)


@pytest.mark.gpu
def test_multi_device_api_matches_single_context():
    """ss_multi_* with two contexts on the visible GPU(s): the sharded batch,
    gathered into frame order on the host, equals one context over all frames
    (bit for bit, clouds included)."""
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.synth import as_rgb, default_rig, params_for, stereo_pair
    W, H, D = 192, 112, 24
    p = ss.StereoParams(**params_for(D))
    rig = ss.StereoRig(**default_rig(W, H))
    frames = [stereo_pair("textured" if i % 2 else "lowtex", W, H, D, seed=i)[:2] for i in range(5)]
    Ls = np.stack([as_rgb(f[0]) for f in frames])
    Rs = np.stack([as_rgb(f[1]) for f in frames])
    flags = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
    ctx = ss.StereoContext(0, W, H, 2, p, rig)
    want = ctx.run(Ls, Rs, flags)
    ctx.close()
    n_dev = max(1, ss.device_count())
    devices = [k % n_dev for k in range(3)]  # three entries: repeats on a one-GPU box
    multi = ss.StereoMulti(devices, W, H, 2, p, rig)
    assert len(multi) == 3
    got = multi.run(Ls, Rs, flags)
    multi.close()
    for k in ("disparity", "valid", "index", "n_points"):
        assert np.array_equal(got[k], want[k]), k
    for f in range(len(frames)):
        m = int(want["n_points"][f])
        for k in ("points", "normals", "colors"):
            assert np.array_equal(got[k][f][:m], want[k][f][:m]), (k, f)
