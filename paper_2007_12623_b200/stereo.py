"""Python host mirror of the reference's stereo entry points (numpy in/out).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/stereoscan/stereo/*.hpp; every call goes through
the C-ABI (include/ss_stereo.h) to the sm_100a kernels.

    compute_disparity(left, right, params)         -> (disparity, valid)
    compute_disparity_lr(left, right, params, max_diff)  opt-in LR consistency
    remove_outliers(disp, valid, radius, thr)      -> (disparity, valid)
    fill_holes(disp, valid, mode, radius, support) -> (disparity, valid)
    cleanup_pass(disp, valid, params)              -> (disparity, valid)
    refine_disparities(disp, valid, left, right, params, trace=False)
    disparity_to_cloud(disp, valid, rgb, rig)      -> StereoCloud
    StereoContext                                   batch throughput API

Errors: ``InvalidArgument`` (std::invalid_argument) and ``StereoError``
(stereoscan::Error; also CUDA failures and "no CUDA device").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class StereoError(RuntimeError):
    """stereoscan::Error (types.hpp:18-21) and device failures."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(StereoError, ValueError):
    """std::invalid_argument (contract violations)."""


def _check(rc):
    if rc != L.SS_OK:
        msg = L.lib().ss_last_error().decode()
        raise (InvalidArgument if rc == L.SS_EINVAL else StereoError)(rc, msg)


@dataclass
class StereoParams:
    """stereoscan::StereoParams (params.hpp:7-24), same defaults."""

    window: int = 11
    d_min: int = -20
    d_max: int = 80
    neighbor_jump_threshold: float = 2.5
    outlier_radius_start: int = 10
    outlier_radius_step: int = 10
    cleanup_iterations: int = 3
    fill_radius_radial: int = 50
    fill_radius_disc: int = 20
    smoothing_radius: int = 15
    alpha: float = 0.1
    eta_smooth: float = 0.01
    refine_iterations: int = 10
    min_zncc: float = 0.5

    def validate(self):
        _check(L.lib().ss_params_validate(C.byref(_params(self))))


@dataclass
class StereoRig:
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    baseline_mm: float = 0.0

    def validate(self):
        _check(L.lib().ss_rig_validate(C.byref(_rig(self))))


@dataclass
class StereoCloud:
    width: int
    height: int
    index: np.ndarray
    points: np.ndarray
    normals: np.ndarray
    colors: np.ndarray
    pixels: np.ndarray = field(default=None)
    fitted: np.ndarray = field(default=None)  # 1: plane fit, 0: sight-ray fallback (cloud.cpp:81)


def _params(p) -> L.SsParams:
    if p is None:
        p = StereoParams()
    if isinstance(p, dict):
        base = StereoParams()
        for k, v in p.items():
            setattr(base, k, v)
        p = base
    return L.SsParams(**{k: getattr(p, k) for k, _ in L.SsParams._fields_})


def _rig(r) -> L.SsRig:
    if isinstance(r, dict):
        return L.SsRig(**r)
    return L.SsRig(**{k: getattr(r, k) for k, _ in L.SsRig._fields_})


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _batch_inputs(left, right, in_format, rgb_ndim):
    """uint8, C-contiguous, equal shapes; the format follows the rank
    (rgb_ndim dims = interleaved RGB) unless given, and must agree with it."""
    left, right = _u8(left), _u8(right)
    if left.shape != right.shape:
        raise InvalidArgument(L.SS_EINVAL, f"stereo batch: left {left.shape} and right "
                                           f"{right.shape} shapes differ")
    if in_format is None:
        in_format = L.SS_IN_RGB if left.ndim == rgb_ndim else L.SS_IN_GRAY
    want = rgb_ndim if in_format == L.SS_IN_RGB else rgb_ndim - 1
    if left.ndim != want or (in_format == L.SS_IN_RGB and left.shape[-1] != 3):
        raise InvalidArgument(L.SS_EINVAL, f"stereo batch: input shape {left.shape} does not "
                                           f"match the {'RGB' if in_format == L.SS_IN_RGB else 'gray'} format")
    dims = left.shape[:rgb_ndim - 1]
    return left, right, in_format, dims


def _batch_outputs(out, n, h, w, out_flags):
    """Allocate, or check dtype / shape / contiguity of caller-given outputs."""
    want = StereoContext.alloc_outputs(n, h, w, out_flags, alloc=lambda s, dt: (s, np.dtype(dt)))
    if out is None:
        return StereoContext.alloc_outputs(n, h, w, out_flags)
    for k, (shape, dt) in want.items():
        a = out.get(k)
        if a is None:
            continue
        if not isinstance(a, np.ndarray) or a.dtype != dt or tuple(a.shape) != tuple(shape) \
                or not a.flags.c_contiguous:
            raise InvalidArgument(L.SS_EINVAL, f"stereo batch: output {k!r} must be a C-contiguous "
                                               f"{dt} array of shape {shape}")
    return out


def device_count() -> int:
    return int(L.lib().ss_device_count())


def to_gray(rgb):
    rgb = _u8(rgb)
    h, w = rgb.shape[:2]
    out = np.empty((h, w), np.uint8)
    _check(L.lib().ss_to_gray(_ptr(rgb), w, h, _ptr(out)))
    return out


def compute_disparity(left, right, params=None):
    left, right = _u8(left), _u8(right)
    (lh, lw), (rh, rw) = left.shape, right.shape
    disp = np.zeros((lh, lw), np.float32)
    valid = np.zeros((lh, lw), np.uint8)
    _check(L.lib().ss_compute_disparity(C.byref(_params(params)), _ptr(left), lw, lh,
                                        _ptr(right), rw, rh, _ptr(disp), _ptr(valid)))
    return disp, valid


def compute_disparity_lr(left, right, params=None, max_diff=1):
    """compute_disparity + opt-in left-right consistency (extension; the
    reference has none). Returns (disparity, valid, right_disparity,
    right_valid): the LR-checked left map and the right-view WTA map."""
    left, right = _u8(left), _u8(right)
    (lh, lw), (rh, rw) = left.shape, right.shape
    disp = np.zeros((lh, lw), np.float32)
    valid = np.zeros((lh, lw), np.uint8)
    rdisp = np.zeros((lh, lw), np.float32)
    rvalid = np.zeros((lh, lw), np.uint8)
    _check(L.lib().ss_compute_disparity_lr(C.byref(_params(params)), _ptr(left), lw, lh,
                                           _ptr(right), rw, rh, int(max_diff), _ptr(disp),
                                           _ptr(valid), _ptr(rdisp), _ptr(rvalid)))
    return disp, valid, rdisp, rvalid


def remove_outliers(disp, valid, radius, threshold):
    disp, valid = _f32(disp), _u8(valid)
    h, w = disp.shape
    od, ov = np.empty_like(disp), np.empty_like(valid)
    _check(L.lib().ss_remove_outliers(_ptr(disp), _ptr(valid), w, h, radius, float(threshold),
                                      _ptr(od), _ptr(ov)))
    return od, ov


def fill_holes(disp, valid, mode, radius, min_support):
    disp, valid = _f32(disp), _u8(valid)
    h, w = disp.shape
    od, ov = np.empty_like(disp), np.empty_like(valid)
    m = 0 if mode in (0, "radial", "Radial") else 1
    _check(L.lib().ss_fill_holes(_ptr(disp), _ptr(valid), w, h, m, radius, min_support,
                                 _ptr(od), _ptr(ov)))
    return od, ov


def disc_neighbor_count(radius):
    return int(L.lib().ss_disc_neighbor_count(radius))


def disc_fill_min_support(radius):
    return int(L.lib().ss_disc_fill_min_support(radius))


def cleanup_pass(disp, valid, params=None):
    disp, valid = _f32(disp), _u8(valid)
    h, w = disp.shape
    od, ov = np.empty_like(disp), np.empty_like(valid)
    _check(L.lib().ss_cleanup_pass(C.byref(_params(params)), _ptr(disp), _ptr(valid), w, h,
                                   _ptr(od), _ptr(ov)))
    return od, ov


def refine_disparities(disp, valid, left, right, params=None, trace=False):
    disp, valid, left, right = _f32(disp), _u8(valid), _u8(left), _u8(right)
    h, w = disp.shape
    pp = _params(params)
    od, ov = np.empty_like(disp), np.empty_like(valid)
    td = ts = None
    if trace:
        it = max(pp.refine_iterations, 0)
        td = np.zeros((it, h, w), np.float64)
        ts = np.zeros((it, h, w), np.float64)
    _check(L.lib().ss_refine_disparities(C.byref(pp), _ptr(disp), _ptr(valid), w, h, _ptr(left),
                                         left.shape[1], left.shape[0], _ptr(right),
                                         right.shape[1], right.shape[0], _ptr(od), _ptr(ov),
                                         _ptr(td), _ptr(ts)))
    return (od, ov, td, ts) if trace else (od, ov)


def disparity_to_cloud(disp, valid, rgb, rig) -> StereoCloud:
    disp, valid = _f32(disp), _u8(valid)
    h, w = disp.shape
    rgb = _u8(rgb) if rgb is not None else None
    ch, cw = (rgb.shape[0], rgb.shape[1]) if rgb is not None else (0, 0)
    n = w * h
    index = np.empty((h, w), np.int32)
    pts = np.empty((n, 3), np.float64)
    nrm = np.empty((n, 3), np.float64)
    col = np.empty((n, 3), np.uint8)
    pix = np.empty((n, 2), np.int32)
    fit = np.empty((n,), np.uint8)
    np_ = C.c_int32(0)
    _check(L.lib().ss_disparity_to_cloud(_ptr(disp), _ptr(valid), w, h, _ptr(rgb), cw, ch,
                                         C.byref(_rig(rig)), _ptr(index), _ptr(pts), _ptr(nrm),
                                         _ptr(col), _ptr(pix), C.byref(np_), _ptr(fit)))
    k = np_.value
    return StereoCloud(w, h, index, pts[:k].copy(), nrm[:k].copy(), col[:k].copy(),
                       pix[:k].copy(), fit[:k].copy())


class StereoContext:
    """Batch throughput API (ss_ctx_*): the whole chain for a batch of frames on
    one GPU. ``run`` takes host arrays (pinned via ``pinned_empty`` for speed);
    ``run_device`` takes raw device pointers (e.g. torch ``data_ptr()``)."""

    def __init__(self, device=0, max_w=960, max_h=540, max_batch=8, params=None, rig=None,
                 lr_check=False, lr_max_diff=1):
        self._ctx = C.c_void_p()
        self.params = params
        r = C.byref(_rig(rig)) if rig is not None else None
        _check(L.lib().ss_ctx_create(device, max_w, max_h, max_batch,
                                     C.byref(_params(params)), r, C.byref(self._ctx)))
        self.max_batch = max_batch
        if lr_check:
            self.set_lr_check(True, lr_max_diff)

    def set_lr_check(self, enable=True, max_diff=1):
        """Opt-in left-right consistency after the WTA (off: reference output)."""
        _check(L.lib().ss_ctx_set_lr_check(self._ctx, 1 if enable else 0, int(max_diff)))

    def close(self):
        if self._ctx:
            _check(L.lib().ss_ctx_destroy(self._ctx))
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(L.lib().ss_ctx_stream(self._ctx) or 0)

    def sync(self):
        _check(L.lib().ss_ctx_sync(self._ctx))

    def stats(self) -> dict:
        st = L.SsCtxStats()
        _check(L.lib().ss_ctx_get_stats(self._ctx, C.byref(st)))
        return {k: int(getattr(st, k)) for k, _ in L.SsCtxStats._fields_}

    def reset_stats(self):
        _check(L.lib().ss_ctx_reset_stats(self._ctx))

    def enable_timing(self, on=True):
        _check(L.lib().ss_ctx_enable_timing(self._ctx, 1 if on else 0))

    def stage_times(self) -> dict:
        """{stage: (ms, launches)} summed since the last reset (synchronizes)."""
        ms = (C.c_double * L.SS_N_STAGES)()
        ln = (C.c_int64 * L.SS_N_STAGES)()
        _check(L.lib().ss_ctx_stage_times(self._ctx, ms, ln))
        return {name: (ms[i], int(ln[i])) for i, name in enumerate(L.STAGE_NAMES)}

    def run(self, left, right, out_flags=L.SS_OUT_DISPARITY, in_format=None, out=None):
        """left/right: (n, H, W, 3) RGB or (n, H, W) gray uint8 host arrays."""
        left, right, in_format, (n, h, w) = _batch_inputs(left, right, in_format, 4)
        out = _batch_outputs(out, n, h, w, out_flags)
        bo = L.SsBatchOut(*[_ptr(out.get(k)) if out.get(k) is not None else None
                            for k, _ in L.SsBatchOut._fields_])
        _check(L.lib().ss_stereo_batch(self._ctx, n, w, h, in_format, _ptr(left), _ptr(right),
                                       out_flags, C.byref(bo)))
        return out

    @staticmethod
    def alloc_outputs(n, h, w, out_flags, alloc=np.empty):
        o = {"disparity": alloc((n, h, w), np.float32), "valid": alloc((n, h, w), np.uint8)}
        oct_ = bool(out_flags & L.SS_OUT_NORMALS_OCT)
        if out_flags & (L.SS_OUT_CLOUD | L.SS_OUT_NORMALS) or oct_:
            o.update(index=alloc((n, h, w), np.int32), points=alloc((n, h * w, 3), np.float32),
                     colors=alloc((n, h * w, 3), np.uint8), n_points=alloc((n,), np.int32))
        if oct_:
            o["normals_oct"] = alloc((n, h * w, 2), np.int16)
        elif out_flags & L.SS_OUT_NORMALS:
            o["normals"] = alloc((n, h * w, 3), np.float32)
        return o

    def run_device(self, n, w, h, d_left, d_right, out_flags=L.SS_OUT_DISPARITY,
                   in_format=L.SS_IN_RGB, stream=None, d_out=None):
        """Asynchronous on `stream` (default: the ctx stream). ``d_out``: optional
        dict of device pointers (keys of SsBatchOut); otherwise results stay in
        the ctx buffers (see device_outputs)."""
        bo = None
        if d_out:
            bo = C.byref(L.SsBatchOut(*[d_out.get(k) for k, _ in L.SsBatchOut._fields_]))
        _check(L.lib().ss_stereo_batch_device(self._ctx, n, w, h, in_format, C.c_void_p(d_left),
                                              C.c_void_p(d_right), out_flags, bo,
                                              C.c_void_p(stream) if stream else None))

    def device_outputs(self) -> dict:
        bo = L.SsBatchOut()
        _check(L.lib().ss_ctx_device_outputs(self._ctx, C.byref(bo)))
        return {k: getattr(bo, k) for k, _ in L.SsBatchOut._fields_}


class StereoMulti:
    """In-process frame sharding across GPUs (ss_multi_*): one context and one
    host thread per device entry; each device writes its contiguous block of
    frames into the shared, frame-ordered outputs (the host-side gather)."""

    def __init__(self, devices, max_w=960, max_h=540, max_batch=8, params=None, rig=None,
                 lr_check=False, lr_max_diff=1):
        self._m = C.c_void_p()
        dev = (C.c_int32 * len(devices))(*devices)
        r = C.byref(_rig(rig)) if rig is not None else None
        rc = L.lib().ss_multi_create(len(devices), dev, max_w, max_h, max_batch,
                                     C.byref(_params(params)), r, C.byref(self._m))
        _check(rc)
        if lr_check:
            _check(L.lib().ss_multi_set_lr_check(self._m, 1, int(lr_max_diff)))

    def close(self):
        if self._m:
            L.lib().ss_multi_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return int(L.lib().ss_multi_size(self._m))

    def run(self, left, right, out_flags=L.SS_OUT_DISPARITY, in_format=None, out=None):
        left, right, in_format, (n, h, w) = _batch_inputs(left, right, in_format, 4)
        out = _batch_outputs(out, n, h, w, out_flags)
        bo = L.SsBatchOut(*[_ptr(out.get(k)) if out.get(k) is not None else None
                            for k, _ in L.SsBatchOut._fields_])
        rc = L.lib().ss_multi_stereo_batch(self._m, n, w, h, in_format, _ptr(left), _ptr(right),
                                           out_flags, C.byref(bo))
        if rc != L.SS_OK:
            raise (InvalidArgument if rc == L.SS_EINVAL else StereoError)(
                rc, L.lib().ss_multi_last_error().decode())
        return out


def stereo_frame(left, right, params=None, rig=None, out_flags=L.SS_OUT_DISPARITY):
    """One pair through the whole chain (ss_stereo_frame): host arrays in, a
    dict of host arrays out (the keys of StereoContext.alloc_outputs, frame
    axis of length 1)."""
    left, right, in_format, (h, w) = _batch_inputs(left, right, None, 3)
    out = _batch_outputs(None, 1, h, w, out_flags)
    bo = L.SsBatchOut(*[_ptr(out.get(k)) if out.get(k) is not None else None
                        for k, _ in L.SsBatchOut._fields_])
    r = C.byref(_rig(rig)) if rig is not None else None
    _check(L.lib().ss_stereo_frame(C.byref(_params(params)), r, w, h, in_format, _ptr(left),
                                   _ptr(right), out_flags, C.byref(bo)))
    return out


def decode_oct_normals(enc):
    """SS_OUT_NORMALS_OCT payload (..., 2) int16 -> unit normals (..., 3) float32
    (the inverse octahedral map of ss_oct_decode in include/ss_stereo.h)."""
    e = np.asarray(enc, np.float32) / 32767.0
    x, y = e[..., 0], e[..., 1]
    z = 1.0 - np.abs(x) - np.abs(y)
    neg = z < 0
    xs = np.where(neg, (1.0 - np.abs(y)) * np.where(x < 0, -1.0, 1.0), x)
    ys = np.where(neg, (1.0 - np.abs(x)) * np.where(y < 0, -1.0, 1.0), y)
    n = np.stack([xs, ys, z], axis=-1).astype(np.float32)
    ln = np.linalg.norm(n, axis=-1, keepdims=True)
    return n / np.where(ln > 0, ln, 1.0)


def pinned_empty(shape, dtype):
    """numpy array backed by pinned (page-locked) host memory; the pages are
    released (cudaFreeHost) when the last view of the array is gone."""
    import weakref
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    p = L.lib().ss_host_alloc(max(nbytes, 1))
    if not p:
        raise StereoError(L.SS_ENOMEM, "cudaHostAlloc failed")
    buf = (C.c_uint8 * max(nbytes, 1)).from_address(p)
    weakref.finalize(buf, L.lib().ss_host_free, C.c_void_p(p))
    return np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)
