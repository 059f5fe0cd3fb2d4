"""Python mirror of the reference's feature front end
(/root/reference/proj/include/stereoscan/features/features.hpp:45-70).

    detect_corners(gray, max_count, threshold) -> corners (N x 3 int32: u, v, score)
    describe(gray, corners)                    -> (positions N x 2 f64, descriptors N x 4 u64)
    match_features(pos_a, desc_a, pos_b, desc_b, max_hamming)
                                               -> dict(index_a, index_b, hamming, displacement)
    histogram_vote(matches, bin_size)          -> matches permuted by priority, with ``rank``

The first three run on the B200 through the C-ABI (ss_detect_corners,
ss_describe, ss_match_features) and are bit-identical to the reference.
histogram_vote is the reference's host-side ranking of a few hundred matches
(features.cpp:210-258), restated here on the host like the scalar helpers.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L
from .stereo import _check, _ptr, _u8


def detect_corners(gray, max_count: int, threshold: int) -> np.ndarray:
    g = _u8(gray)
    h, w = g.shape
    cap = max(int(max_count), 0)
    u = np.zeros(cap, np.int32)
    v = np.zeros(cap, np.int32)
    s = np.zeros(cap, np.int32)
    n = C.c_int32(0)
    _check(L.lib().ss_detect_corners(_ptr(g), w, h, int(max_count), int(threshold), _ptr(u),
                                     _ptr(v), _ptr(s), C.byref(n)))
    k = n.value
    return np.stack([u[:k], v[:k], s[:k]], axis=1) if k else np.zeros((0, 3), np.int32)


def describe(gray, corners):
    g = _u8(gray)
    h, w = g.shape
    c = np.ascontiguousarray(np.asarray(corners, np.int32).reshape(-1, 3))
    nc = len(c)
    u, v, s = (np.ascontiguousarray(c[:, i]) for i in range(3))
    pos = np.zeros((max(nc, 1), 2), np.float64)
    desc = np.zeros((max(nc, 1), 4), np.uint64)
    n = C.c_int32(0)
    _check(L.lib().ss_describe(_ptr(g), w, h, _ptr(u), _ptr(v), _ptr(s), nc, _ptr(pos),
                               _ptr(desc), C.byref(n)))
    return pos[:n.value].copy(), desc[:n.value].copy()


def match_features(pos_a, desc_a, pos_b, desc_b, max_hamming: int) -> dict:
    pa = np.ascontiguousarray(pos_a, np.float64).reshape(-1, 2)
    pb = np.ascontiguousarray(pos_b, np.float64).reshape(-1, 2)
    da = np.ascontiguousarray(desc_a, np.uint64).reshape(-1, 4)
    db = np.ascontiguousarray(desc_b, np.uint64).reshape(-1, 4)
    na, nb = len(da), len(db)
    cap = max(min(na, nb), 1)
    ia = np.zeros(cap, np.int32)
    ib = np.zeros(cap, np.int32)
    hm = np.zeros(cap, np.int32)
    dp = np.zeros((cap, 2), np.float64)
    n = C.c_int32(0)
    _check(L.lib().ss_match_features(_ptr(pa), _ptr(da), na, _ptr(pb), _ptr(db), nb,
                                     int(max_hamming), _ptr(ia), _ptr(ib), _ptr(hm), _ptr(dp),
                                     C.byref(n)))
    k = n.value
    return {"index_a": ia[:k].copy(), "index_b": ib[:k].copy(), "hamming": hm[:k].copy(),
            "displacement": dp[:k].copy()}


def histogram_vote(matches: dict, bin_size: float) -> dict:
    """features.cpp:210-258: priority = matches in the 3x3 bins around the
    match's displacement bin; order by priority desc, hamming asc, index asc."""
    if not (bin_size > 0.0):
        raise ValueError("histogram_vote: bin_size must be > 0")
    d = np.asarray(matches["displacement"], np.float64).reshape(-1, 2)
    n = len(d)
    if n == 0:
        return {k: np.asarray(v)[:0] for k, v in matches.items()} | {"rank": np.zeros(0, np.int32)}
    bins = [(math.floor(x / bin_size), math.floor(y / bin_size)) for x, y in d]
    hist = {}
    for b in bins:
        hist[b] = hist.get(b, 0) + 1
    prio = [sum(hist.get((bu + du, bv + dv), 0) for dv in (-1, 0, 1) for du in (-1, 0, 1))
            for bu, bv in bins]
    ham = np.asarray(matches["hamming"])
    order = sorted(range(n), key=lambda i: (-prio[i], int(ham[i]), i))
    out = {k: np.asarray(v)[order] for k, v in matches.items()}
    out["rank"] = np.arange(n, dtype=np.int32)
    out["order"] = np.asarray(order, np.int32)
    return out
