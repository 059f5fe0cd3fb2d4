"""Surfel-model fusion on the GPU (SPEC.md:440-476 [MODULE] fusion; SURVEY.md
§8f row 2): rasterize + fuse_frame through the C-ABI (include/ss_stereo.h,
ss_fusion_*). The model stays in HBM; keyframe clouds from the batch API can
be fused without leaving the device (``fuse_device``).

    m = SurfelModel(device=0)                      # SPEC defaults (trunc 10 mm,
                                                   # cap 50, gate 5 mm, omega_min 0.1)
    m.fuse_frame(cloud, pose, rig)                 # host StereoCloud (stereo.py)
    ids, depth = m.rasterize(pose, rig)
    model = m.download()                           # dict of numpy arrays

pose: 3x4 (or 4x4) world->camera matrix [R | t], X_cam = R X_world + t.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .stereo import _check, _ptr, _rig


def _pose(pose) -> np.ndarray:
    p = np.ascontiguousarray(np.asarray(pose, np.float64)[:3, :4]).reshape(12)
    return p


class SurfelModel:
    def __init__(self, device=0, trunc_mm=10.0, weight_cap=50.0, association_gate_mm=5.0,
                 omega_min=0.1):
        self._f = C.c_void_p()
        prm = L.SsFusionParams(trunc_mm, weight_cap, association_gate_mm, omega_min)
        _check(L.lib().ss_fusion_create(device, C.byref(prm), C.byref(self._f)))

    def close(self):
        if self._f:
            _check(L.lib().ss_fusion_destroy(self._f))
            self._f = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        n = C.c_int32(0)
        _check(L.lib().ss_fusion_size(self._f, C.byref(n)))
        return n.value

    def upload(self, pos, normal, color, weight, color_weight):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (pos, normal, color, weight,
                                                              color_weight)]
        _check(L.lib().ss_fusion_upload(self._f, len(arrs[3]), *[_ptr(a) for a in arrs]))

    def download(self) -> dict:
        n = len(self)
        out = {"pos": np.zeros((n, 3)), "normal": np.zeros((n, 3)), "color": np.zeros((n, 3)),
               "weight": np.zeros(n), "color_weight": np.zeros(n)}
        _check(L.lib().ss_fusion_download(self._f, *[_ptr(out[k]) for k in
                                                      ("pos", "normal", "color", "weight",
                                                       "color_weight")]))
        return out

    def rasterize(self, pose, rig):
        r = _rig(rig)
        ids = np.zeros((r.height, r.width), np.int32)
        depth = np.zeros((r.height, r.width), np.float64)
        p = _pose(pose)
        _check(L.lib().ss_fusion_rasterize(self._f, _ptr(p), C.byref(r), _ptr(ids), _ptr(depth)))
        return ids, depth

    def fuse_frame(self, cloud, pose, rig):
        """cloud: stereo.StereoCloud (index per pixel, points / normals, colors)."""
        r = _rig(rig)
        idx = np.ascontiguousarray(cloud.index, np.int32)
        pts = np.ascontiguousarray(cloud.points, np.float64).reshape(-1, 3)
        nrm = np.ascontiguousarray(cloud.normals, np.float64).reshape(-1, 3)
        col = np.ascontiguousarray(cloud.colors, np.uint8).reshape(-1, 3)
        p = _pose(pose)
        _check(L.lib().ss_fusion_fuse_frame(self._f, _ptr(idx), len(pts), _ptr(pts), _ptr(nrm),
                                            _ptr(col), r.width, r.height, _ptr(p), C.byref(r)))

    def fuse_device(self, d_index, d_points, d_normals, d_colors, pose, rig, stream=None):
        """Fuse one frame straight from device arrays (int/ptr addresses), e.g.
        the batch API's outputs for frame f."""
        r = _rig(rig)
        p = _pose(pose)
        _check(L.lib().ss_fusion_fuse_device(self._f, C.c_void_p(d_index), C.c_void_p(d_points),
                                             C.c_void_p(d_normals), C.c_void_p(d_colors),
                                             r.width, r.height, _ptr(p), C.byref(r),
                                             C.c_void_p(stream) if stream else None))
