"""Frame sharding across GPUs: no collective on the data path.

Stereo pairs are independent, so a batch or video splits into
contiguous frame blocks, one per rank (one process per GPU). The only
inter-rank traffic is control: a barrier, the max-over-ranks step time, and a
host-side gather of per-frame results into frame order on rank 0.
"""
from __future__ import annotations

import numpy as np


def frame_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, end) of frames for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the step time); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_frames(local: dict, n_frames: int, rank: int, world: int, dst: int = 0):
    """Host-side gather of frame-major per-rank outputs into global frame order.

    `local` maps names to arrays whose first axis indexes this rank's frames
    (frame_range order). Returns the assembled dict on `dst`, None elsewhere.
    """
    import torch.distributed as dist
    if world == 1:
        return {k: np.asarray(v) for k, v in local.items()}
    start, end = frame_range(n_frames, rank, world)
    payload = (start, end, {k: np.asarray(v) for k, v in local.items()})
    parts = [None] * world if rank == dst else None
    dist.gather_object(payload, parts, dst=dst)
    if rank != dst:
        return None
    out = {}
    for s, e, arrays in sorted(parts, key=lambda p: p[0]):
        for k, v in arrays.items():
            if k not in out:
                out[k] = np.empty((n_frames,) + v.shape[1:], v.dtype)
            out[k][s:e] = v
    return out
