"""Seeded synthetic stereo pairs (SURVEY.md §8d recipes C1-C5).

Pure numpy, deterministic for a given (kind, width, height, D, seed) on any
machine with the same numpy major version (PCG64 stream). The oracle and the
CUDA path consume the identical bytes.

* ``textured``    — C1/C3/C4: 128 + 40 N(0,1) texture, right view sampled with
  linear interpolation at x + d(x, y), d = 0.25D + 0.5D x/W + 0.1D sin(0.01 y),
  per-view noise sigma 1.
* ``lowtex``      — C2: same geometry; ~1/3 of the texture is flat (zero
  variance), amplitude sigma 1.75 elsewhere, and a band of period-16 stripes
  (period < D) that produces wrong matches and outliers for cleanup.
* ``video``       — C5: textured with a per-frame drift of the disparity field.
* ``plane`` / ``sphere`` — SPEC.md:610 (acceptance #2): a textured slanted
  plane, and a sphere in front of a slanted plane, with +-0.5 gray-level noise.

Images are returned as (H, W) uint8 gray planes; ``as_rgb`` replicates them
into interleaved RGB (luma of (g, g, g) is g, so to_gray is the identity).
"""
from __future__ import annotations

import numpy as np


def _disparity_field(w, h, D, phase=0.0, shape="wave"):
    """Disparity in RIGHT-image coordinates (x, y): the recipes' smooth field
    ("wave"), the SPEC acceptance #2 slanted plane, or a sphere in front of a
    slanted background plane."""
    x = np.arange(w, dtype=np.float64)[None, :]
    y = np.arange(h, dtype=np.float64)[:, None]
    if shape == "plane":
        return 0.2 * D + 0.45 * D * x / w + 0.15 * D * y / h + 0.0 * y
    if shape == "sphere":
        base = 0.2 * D + 0.25 * D * x / w + 0.1 * D * y / h
        cx, cy, rad = 0.5 * w, 0.5 * h, 0.35 * min(w, h)
        r2 = (x - cx) ** 2 + (y - cy) ** 2
        cap = np.sqrt(np.maximum(rad * rad - r2, 0.0)) / rad  # unit hemisphere height
        return base + 0.3 * D * cap
    return 0.25 * D + 0.5 * D * x / w + 0.1 * D * np.sin(0.01 * y + phase)


def _sample(tex, xs):
    """Linear interpolation of tex rows at fractional x positions xs (H, W)."""
    h = tex.shape[0]
    x0 = np.floor(xs).astype(np.int64)
    f = xs - x0
    rows = np.arange(h)[:, None]
    return tex[rows, x0] * (1.0 - f) + tex[rows, x0 + 1] * f


def _to_u8(a):
    return np.clip(np.rint(a), 0, 255).astype(np.uint8)


def stereo_pair(kind: str = "textured", width: int = 960, height: int = 540, D: int = 64,
                seed: int = 1234, frame: int = 0):
    """Return (left, right, true_disparity) for the named recipe."""
    rng = np.random.default_rng(seed)
    w, h = width, height
    margin = D + 8
    if kind in ("textured", "video", "plane", "sphere"):
        tex = 128.0 + 40.0 * rng.standard_normal((h, w + margin))
    elif kind == "lowtex":
        tex = 100.0 + 1.75 * rng.standard_normal((h, w + margin))
        xt = np.arange(w + margin)[None, :]
        yt = np.arange(h)[:, None]
        bx, by = max(12, w // 10), max(9, h * 2 // 15)
        flat = ((xt // bx) + (yt // by)) % 3 == 0
        tex = np.where(flat, 100.0, tex)
        band = (yt >= int(0.55 * h)) & (yt < int(0.70 * h))
        stripes = 100.0 + 20.0 * np.sin(2 * np.pi * xt / 16.0) + 1.0 * rng.standard_normal(
            (h, w + margin))
        tex = np.where(band & ~flat, stripes, tex)
    else:
        raise ValueError(f"unknown synthetic kind {kind!r}")
    phase = 0.05 * frame if kind == "video" else 0.0
    shape = kind if kind in ("plane", "sphere") else "wave"
    dtrue = _disparity_field(w, h, D, phase, shape)
    xs = np.arange(w, dtype=np.float64)[None, :] + dtrue
    left = tex[:, :w].copy()
    right = _sample(tex, xs)
    if kind in ("plane", "sphere"):  # +-0.5 gray-level noise
        left = left + rng.uniform(-0.5, 0.5, (h, w))
        right = right + rng.uniform(-0.5, 0.5, (h, w))
    elif kind != "lowtex":
        left = left + rng.standard_normal((h, w))
        right = right + rng.standard_normal((h, w))
    else:
        bx, by = max(12, w // 10), max(9, h * 2 // 15)
        flat_l = ((np.arange(w)[None, :] // bx) + (np.arange(h)[:, None] // by)) % 3 == 0
        left = left + np.where(flat_l, 0.0, 0.5 * rng.standard_normal((h, w)))
        flat_r = ((np.floor(xs).astype(np.int64) // bx) + (np.arange(h)[:, None] // by)) % 3 == 0
        right = right + np.where(flat_r, 0.0, 0.5 * rng.standard_normal((h, w)))
    # Ground truth in LEFT coordinates: left u sees the point right x sees when
    # x + d(x) = u; solve x = u - d(x) by fixed-point iteration (|d'| << 1).
    u = np.arange(w, dtype=np.float64)[None, :]
    rows = np.arange(h)[:, None]
    xr = u - dtrue
    for _ in range(30 if shape == "sphere" else 6):
        # field value at the fractional right-image positions xr (linear
        # interpolation of the per-column field; exact for the linear ones)
        xi = np.clip(xr, 0, w - 1)
        x0 = np.floor(xi).astype(np.int64)
        x1 = np.minimum(x0 + 1, w - 1)
        t = xi - x0
        dr = dtrue[rows, x0] * (1 - t) + dtrue[rows, x1] * t
        xr = u - dr
    dleft = u - xr
    return _to_u8(left), _to_u8(right), dleft


def as_rgb(gray):
    return np.repeat(gray[..., None], 3, axis=-1).copy()


def default_rig(width: int, height: int):
    """A rectified rig consistent with the synthetic geometry (dict form)."""
    return dict(fx=1000.0, fy=1000.0, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                width=width, height=height, baseline_mm=5.0)


def params_for(D: int, **kw):
    """StereoParams defaults (params.hpp:8-21) with d in [0, D-1] (SURVEY §8 convention)."""
    p = dict(window=11, d_min=0, d_max=D - 1, neighbor_jump_threshold=2.5,
             outlier_radius_start=10, outlier_radius_step=10, cleanup_iterations=3,
             fill_radius_radial=50, fill_radius_disc=20, smoothing_radius=15, alpha=0.1,
             eta_smooth=0.01, refine_iterations=10, min_zncc=0.5)
    p.update(kw)
    return p
