"""ORACLE loader — test infrastructure only.

ctypes front-end for the two CPU oracles declared in ``oracle/ss_oracle.h``:

* ``Oracle("ref")`` — the UNMODIFIED reference sources compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libss_ref.so``;
* ``Oracle("orc")`` — the plain-C restatement ``oracle/ss_oracle.c``
  (``oracle/build/libss_oracle.so``), the only source of
  ``disparity_to_cloud`` (the reference's needs Eigen).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "ref": os.path.join(HERE, "_ref", "libss_ref.so"),
    "orc": os.path.join(HERE, "build", "libss_oracle.so"),
}


class OrcParams(C.Structure):
    """Field-for-field ``stereoscan::StereoParams`` (params.hpp:7-24)."""

    _fields_ = [
        ("window", C.c_int32),
        ("d_min", C.c_int32),
        ("d_max", C.c_int32),
        ("neighbor_jump_threshold", C.c_double),
        ("outlier_radius_start", C.c_int32),
        ("outlier_radius_step", C.c_int32),
        ("cleanup_iterations", C.c_int32),
        ("fill_radius_radial", C.c_int32),
        ("fill_radius_disc", C.c_int32),
        ("smoothing_radius", C.c_int32),
        ("alpha", C.c_double),
        ("eta_smooth", C.c_double),
        ("refine_iterations", C.c_int32),
        ("min_zncc", C.c_double),
    ]


class OrcRig(C.Structure):
    _fields_ = [
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("baseline_mm", C.c_double),
    ]


PARAM_DEFAULTS = dict(
    window=11, d_min=-20, d_max=80, neighbor_jump_threshold=2.5,
    outlier_radius_start=10, outlier_radius_step=10, cleanup_iterations=3,
    fill_radius_radial=50, fill_radius_disc=20, smoothing_radius=15,
    alpha=0.1, eta_smooth=0.01, refine_iterations=10, min_zncc=0.5,
)


def to_orc_params(p=None, **kw) -> OrcParams:
    vals = dict(PARAM_DEFAULTS)
    if p is not None:
        for k in PARAM_DEFAULTS:
            if hasattr(p, k):
                vals[k] = getattr(p, k)
            elif isinstance(p, dict) and k in p:
                vals[k] = p[k]
    vals.update(kw)
    return OrcParams(**vals)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class CloudResult:
    index: np.ndarray
    points: np.ndarray
    normals: np.ndarray
    colors: np.ndarray
    pixels: np.ndarray
    eigen_gap: np.ndarray
    decision: np.ndarray = None  # (l1 - t) / t, t = 1e-9 max(1, l2) (cloud.cpp:81)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


_U8 = C.c_uint8
_F32 = C.c_float
_F64 = C.c_double
_I32 = C.c_int32


class Oracle:
    def __init__(self, kind: str = "orc"):
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        pre = kind + "_"
        self._f = lambda name: getattr(self.lib, pre + name)
        self._f("last_error").restype = C.c_char_p
        self._f("zncc_chessboard").restype = C.c_double
        self._f("disc_neighbor_count").restype = C.c_int32
        self._f("disc_fill_min_support").restype = C.c_int32

    @staticmethod
    def available(kind: str) -> bool:
        return os.path.exists(LIB_PATHS[kind])

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f("last_error")().decode())

    # --- API mirroring the reference's per-stage entry points ---
    def to_gray(self, rgb):
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        h, w = rgb.shape[:2]
        out = np.empty((h, w), np.uint8)
        self._check(self._f("to_gray")(_p(rgb, _U8), w, h, _p(out, _U8)))
        return out

    def zncc_chessboard(self, left, right, lu, lv, ru, rv, window):
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = left.shape
        d = _I32(0)
        v = self._f("zncc_chessboard")(_p(left, _U8), _p(right, _U8), w, h, lu, lv, ru, rv,
                                       window, C.byref(d))
        return v if d.value else None

    def compute_disparity(self, left, right, params=None, naive=False):
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = left.shape
        disp = np.zeros((h, w), np.float32)
        valid = np.zeros((h, w), np.uint8)
        fn = self.lib.ref_naive_compute_disparity if naive else self._f("compute_disparity")
        pp = to_orc_params(params)
        self._check(fn(C.byref(pp), _p(left, _U8), _p(right, _U8), w, h, _p(disp, _F32),
                       _p(valid, _U8)))
        return disp, valid

    def compute_disparity_right(self, left, right, params=None):
        """Right-view WTA (restatement only; the LR-check extension)."""
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = left.shape
        disp = np.zeros((h, w), np.float32)
        valid = np.zeros((h, w), np.uint8)
        pp = to_orc_params(params)
        self._check(self.lib.orc_compute_disparity_right(
            C.byref(pp), _p(left, _U8), _p(right, _U8), w, h, _p(disp, _F32), _p(valid, _U8)))
        return disp, valid

    def lr_check(self, disp, valid, disp_r, valid_r, max_diff=1):
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        disp_r = np.ascontiguousarray(disp_r, np.float32)
        valid_r = np.ascontiguousarray(valid_r, np.uint8)
        h, w = disp.shape
        od = np.empty_like(disp)
        ov = np.empty_like(valid)
        self._check(self.lib.orc_lr_check(_p(disp, _F32), _p(valid, _U8), _p(disp_r, _F32),
                                          _p(valid_r, _U8), w, h, max_diff, _p(od, _F32),
                                          _p(ov, _U8)))
        return od, ov

    def compute_disparity_lr(self, left, right, params=None, max_diff=1):
        d, v = self.compute_disparity(left, right, params)
        dr, vr = self.compute_disparity_right(left, right, params)
        od, ov = self.lr_check(d, v, dr, vr, max_diff)
        return od, ov, dr, vr

    # --- feature front end (reference only: features.cpp) ---
    def detect_corners(self, gray, max_count, threshold):
        g = np.ascontiguousarray(gray, np.uint8)
        h, w = g.shape
        cap = max(int(max_count), 0)
        u, v, sc = (np.zeros(max(cap, 1), np.int32) for _ in range(3))
        n = _I32(0)
        self._check(self.lib.ref_detect_corners(_p(g, _U8), w, h, int(max_count), int(threshold),
                                                _p(u, _I32), _p(v, _I32), _p(sc, _I32),
                                                C.byref(n)))
        k = n.value
        return np.stack([u[:k], v[:k], sc[:k]], axis=1) if k else np.zeros((0, 3), np.int32)

    def describe(self, gray, corners):
        g = np.ascontiguousarray(gray, np.uint8)
        h, w = g.shape
        c = np.ascontiguousarray(np.asarray(corners, np.int32).reshape(-1, 3))
        nc = len(c)
        u, v, sc = (np.ascontiguousarray(c[:, i]) for i in range(3))
        pos = np.zeros((max(nc, 1), 2), np.float64)
        desc = np.zeros((max(nc, 1), 4), np.uint64)
        n = _I32(0)
        self._check(self.lib.ref_describe(_p(g, _U8), w, h, _p(u, _I32), _p(v, _I32),
                                          _p(sc, _I32), nc, _p(pos, _F64),
                                          desc.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          C.byref(n)))
        return pos[:n.value].copy(), desc[:n.value].copy()

    def match_features(self, pos_a, desc_a, pos_b, desc_b, max_hamming):
        pa = np.ascontiguousarray(pos_a, np.float64).reshape(-1, 2)
        pb = np.ascontiguousarray(pos_b, np.float64).reshape(-1, 2)
        da = np.ascontiguousarray(desc_a, np.uint64).reshape(-1, 4)
        db = np.ascontiguousarray(desc_b, np.uint64).reshape(-1, 4)
        cap = max(min(len(da), len(db)), 1)
        ia, ib, hm = (np.zeros(cap, np.int32) for _ in range(3))
        dp = np.zeros((cap, 2), np.float64)
        n = _I32(0)
        u64 = C.POINTER(C.c_uint64)
        self._check(self.lib.ref_match_features(
            _p(pa, _F64), da.ctypes.data_as(u64), len(da), _p(pb, _F64), db.ctypes.data_as(u64),
            len(db), int(max_hamming), _p(ia, _I32), _p(ib, _I32), _p(hm, _I32), _p(dp, _F64),
            C.byref(n)))
        k = n.value
        return {"index_a": ia[:k].copy(), "index_b": ib[:k].copy(), "hamming": hm[:k].copy(),
                "displacement": dp[:k].copy()}

    def histogram_vote(self, matches, bin_size):
        ia = np.ascontiguousarray(matches["index_a"], np.int32)
        ib = np.ascontiguousarray(matches["index_b"], np.int32)
        hm = np.ascontiguousarray(matches["hamming"], np.int32)
        dp = np.ascontiguousarray(matches["displacement"], np.float64).reshape(-1, 2)
        order = np.zeros(max(len(ia), 1), np.int32)
        self._check(self.lib.ref_histogram_vote(_p(ia, _I32), _p(ib, _I32), _p(hm, _I32),
                                                _p(dp, _F64), len(ia), C.c_double(bin_size),
                                                _p(order, _I32)))
        return order[:len(ia)].copy()

    # --- fusion consumer (restatement only: SPEC.md:440-476, no reference source) ---
    def rasterize(self, pos, pose, rig):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
        P = np.ascontiguousarray(np.asarray(pose, np.float64)[:3, :4]).reshape(12)
        w, h = int(rig["width"]), int(rig["height"])
        ids = np.zeros((h, w), np.int32)
        dep = np.zeros((h, w), np.float64)
        self._check(self.lib.orc_rasterize(_p(pos, _F64), len(pos), _p(P, _F64),
                                           C.c_double(rig["fx"]), C.c_double(rig["fy"]),
                                           C.c_double(rig["cx"]), C.c_double(rig["cy"]), w, h,
                                           _p(ids, _I32), _p(dep, _F64)))
        return ids, dep

    def fuse_frame(self, model, index, points, normals, colors, pose, rig, trunc=10.0, cap=50.0,
                   gate=5.0, omega_min=0.1):
        """model: dict pos/normal/color (n x 3), weight/color_weight (n); returns the new one."""
        n0 = len(model["weight"])
        index = np.ascontiguousarray(index, np.int32)
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        capn = n0 + int((index >= 0).sum()) + 1
        arr = {}
        for k, per in (("pos", 3), ("normal", 3), ("color", 3), ("weight", 1), ("color_weight", 1)):
            a = np.zeros((capn, per) if per == 3 else capn, np.float64)
            a[:n0] = model[k]
            arr[k] = a
        n = _I32(n0)
        P = np.ascontiguousarray(np.asarray(pose, np.float64)[:3, :4]).reshape(12)
        nrm = np.ascontiguousarray(normals, np.float64).reshape(-1, 3)
        col = np.ascontiguousarray(colors, np.uint8).reshape(-1, 3)
        w, h = int(rig["width"]), int(rig["height"])
        self._check(self.lib.orc_fuse_frame(
            _p(arr["pos"], _F64), _p(arr["normal"], _F64), _p(arr["color"], _F64),
            _p(arr["weight"], _F64), _p(arr["color_weight"], _F64), C.byref(n), capn,
            _p(index, _I32), _p(pts, _F64), _p(nrm, _F64), _p(col, _U8), w, h, _p(P, _F64),
            C.c_double(rig["fx"]), C.c_double(rig["fy"]), C.c_double(rig["cx"]),
            C.c_double(rig["cy"]), C.c_double(trunc), C.c_double(cap), C.c_double(gate),
            C.c_double(omega_min)))
        return {k: v[:n.value] for k, v in arr.items()}

    def remove_outliers(self, disp, valid, radius, threshold, naive=False):
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        h, w = disp.shape
        od = np.empty_like(disp)
        ov = np.empty_like(valid)
        fn = self.lib.ref_naive_remove_outliers if naive else self._f("remove_outliers")
        self._check(fn(_p(disp, _F32), _p(valid, _U8), w, h, radius, C.c_double(threshold),
                       _p(od, _F32), _p(ov, _U8)))
        return od, ov

    def fill_holes(self, disp, valid, mode, radius, min_support):
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        h, w = disp.shape
        od = np.empty_like(disp)
        ov = np.empty_like(valid)
        m = 0 if mode in (0, "radial", "Radial") else 1
        self._check(self._f("fill_holes")(_p(disp, _F32), _p(valid, _U8), w, h, m, radius,
                                          min_support, _p(od, _F32), _p(ov, _U8)))
        return od, ov

    def disc_neighbor_count(self, r):
        return int(self._f("disc_neighbor_count")(r))

    def disc_fill_min_support(self, r):
        return int(self._f("disc_fill_min_support")(r))

    def cleanup_pass(self, disp, valid, params=None):
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        h, w = disp.shape
        od = np.empty_like(disp)
        ov = np.empty_like(valid)
        pp = to_orc_params(params)
        self._check(self._f("cleanup_pass")(C.byref(pp), _p(disp, _F32), _p(valid, _U8), w, h,
                                            _p(od, _F32), _p(ov, _U8)))
        return od, ov

    def refine_disparities(self, disp, valid, left, right, params=None, trace=False):
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        h, w = disp.shape
        pp = to_orc_params(params)
        od = np.empty_like(disp)
        ov = np.empty_like(valid)
        td = ts = None
        if trace:
            td = np.zeros((pp.refine_iterations, h, w), np.float64)
            ts = np.zeros((pp.refine_iterations, h, w), np.float64)
        null = C.POINTER(_F64)()
        self._check(self._f("refine_disparities")(
            C.byref(pp), _p(disp, _F32), _p(valid, _U8), _p(left, _U8), _p(right, _U8), w, h,
            _p(od, _F32), _p(ov, _U8), _p(td, _F64) if trace else null,
            _p(ts, _F64) if trace else null))
        return (od, ov, td, ts) if trace else (od, ov)

    def disparity_to_cloud(self, disp, valid, rgb, rig) -> CloudResult:
        if self.kind != "orc":
            raise NotImplementedError("the reference's disparity_to_cloud needs Eigen (absent)")
        disp = np.ascontiguousarray(disp, np.float32)
        valid = np.ascontiguousarray(valid, np.uint8)
        rgb = np.ascontiguousarray(rgb, np.uint8)
        h, w = disp.shape
        ch, cw = rgb.shape[:2]
        n = w * h
        index = np.empty((h, w), np.int32)
        pts = np.empty((n, 3), np.float64)
        nrm = np.empty((n, 3), np.float64)
        col = np.empty((n, 3), np.uint8)
        pix = np.empty((n, 2), np.int32)
        gap = np.empty((n,), np.float64)
        dec = np.empty((n,), np.float64)
        npts = _I32(0)
        r = rig if isinstance(rig, OrcRig) else OrcRig(**rig)
        self._check(self.lib.orc_disparity_to_cloud(
            _p(disp, _F32), _p(valid, _U8), w, h, _p(rgb, _U8), cw, ch, C.byref(r),
            _p(index, _I32), _p(pts, _F64), _p(nrm, _F64), _p(col, _U8), _p(pix, _I32),
            C.byref(npts), _p(gap, _F64), _p(dec, _F64)))
        k = npts.value
        return CloudResult(index, pts[:k].copy(), nrm[:k].copy(), col[:k].copy(),
                           pix[:k].copy(), gap[:k].copy(), dec[:k].copy())

    def eigen3_sym(self, a):
        """Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d> restatement: (evals
        ascending, evecs as columns, converged)."""
        a = np.ascontiguousarray(a, np.float64).reshape(3, 3)
        ev = np.empty(3, np.float64)
        vec = np.empty((3, 3), np.float64)
        rc = self.lib.orc_eigen3_sym(_p(a, _F64), _p(ev, _F64), _p(vec, _F64))
        return ev, vec, rc == 0

    def stereo_frame(self, left_rgb, right_rgb, rig, params=None):
        """run_stereo_only order: to_gray -> compute_disparity
        -> cleanup_pass -> refine_disparities -> disparity_to_cloud."""
        lg = self.to_gray(left_rgb)
        rg = self.to_gray(right_rgb)
        d, v = self.compute_disparity(lg, rg, params)
        d, v = self.cleanup_pass(d, v, params)
        d, v = self.refine_disparities(d, v, lg, rg, params)
        cloud = Oracle("orc").disparity_to_cloud(d, v, left_rgb, rig) if self.kind != "orc" \
            else self.disparity_to_cloud(d, v, left_rgb, rig)
        return d, v, cloud
