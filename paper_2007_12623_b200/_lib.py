"""ctypes binding of include/ss_stereo.h (libstereoscan_b200.so, built in-tree).

There is no fallback: if the library is missing, importing the bindings raises,
and without a CUDA device every compute call raises ``StereoError`` (SS_ENODEV).
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                        "libstereoscan_b200.so")

SS_OK, SS_EINVAL, SS_EPARAM, SS_ECUDA, SS_ENOMEM, SS_ENODEV = range(6)
SS_IN_RGB, SS_IN_GRAY = 0, 1
SS_OUT_DISPARITY, SS_OUT_CLOUD, SS_OUT_NORMALS = 1, 2, 4
SS_OUT_NORMALS_OCT, SS_OUT_TRIM = 8, 16
SS_N_STAGES = 14
STAGE_NAMES = ["luma", "stats", "wta_sweep", "wta_resolve", "cleanup", "refine", "cloud",
               "cleanup_outliers", "cleanup_radial", "cleanup_disc", "refine_scan", "refine_repick",
               "refine_exact", "cloud_normals"]


class SsParams(C.Structure):
    _fields_ = [
        ("window", C.c_int32), ("d_min", C.c_int32), ("d_max", C.c_int32),
        ("neighbor_jump_threshold", C.c_double), ("outlier_radius_start", C.c_int32),
        ("outlier_radius_step", C.c_int32), ("cleanup_iterations", C.c_int32),
        ("fill_radius_radial", C.c_int32), ("fill_radius_disc", C.c_int32),
        ("smoothing_radius", C.c_int32), ("alpha", C.c_double), ("eta_smooth", C.c_double),
        ("refine_iterations", C.c_int32), ("min_zncc", C.c_double),
    ]


class SsRig(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("baseline_mm", C.c_double)]


class SsFusionParams(C.Structure):
    _fields_ = [("trunc_mm", C.c_double), ("weight_cap", C.c_double),
                ("association_gate_mm", C.c_double), ("omega_min", C.c_double)]


class SsBatchOut(C.Structure):
    _fields_ = [("disparity", C.c_void_p), ("valid", C.c_void_p), ("index", C.c_void_p),
                ("points", C.c_void_p), ("normals", C.c_void_p), ("colors", C.c_void_p),
                ("n_points", C.c_void_p), ("normals_oct", C.c_void_p)]


class SsCtxStats(C.Structure):
    _fields_ = [("frames", C.c_int64), ("wta_resolved", C.c_int64),
                ("refine_resolved", C.c_int64), ("refine_scored", C.c_int64),
                ("kernel_launches", C.c_int64), ("disc_fill_pixels", C.c_int64),
                ("graph_launches", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -m paper_2007_12623_b200.build` "
            "(the stereo path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, f64 = C.c_void_p, C.c_int32, C.c_double
    P = C.POINTER
    sig = {
        "ss_last_error": (C.c_char_p, []),
        "ss_version": (C.c_char_p, []),
        "ss_params_default": (None, [P(SsParams)]),
        "ss_params_validate": (i32, [P(SsParams)]),
        "ss_rig_validate": (i32, [P(SsRig)]),
        "ss_disc_neighbor_count": (i32, [i32]),
        "ss_disc_fill_min_support": (i32, [i32]),
        "ss_device_count": (i32, []),
        "ss_to_gray": (i32, [vp, i32, i32, vp]),
        "ss_compute_disparity": (i32, [P(SsParams), vp, i32, i32, vp, i32, i32, vp, vp]),
        "ss_compute_disparity_lr": (i32, [P(SsParams), vp, i32, i32, vp, i32, i32, i32, vp, vp,
                                          vp, vp]),
        "ss_detect_corners": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, P(i32)]),
        "ss_describe": (i32, [vp, i32, i32, vp, vp, vp, i32, vp, vp, P(i32)]),
        "ss_match_features": (i32, [vp, vp, i32, vp, vp, i32, i32, vp, vp, vp, vp, P(i32)]),
        "ss_fusion_params_default": (None, [P(SsFusionParams)]),
        "ss_fusion_create": (i32, [i32, P(SsFusionParams), P(vp)]),
        "ss_fusion_destroy": (i32, [vp]),
        "ss_fusion_size": (i32, [vp, P(i32)]),
        "ss_fusion_upload": (i32, [vp, i32, vp, vp, vp, vp, vp]),
        "ss_fusion_download": (i32, [vp, vp, vp, vp, vp, vp]),
        "ss_fusion_rasterize": (i32, [vp, vp, P(SsRig), vp, vp]),
        "ss_fusion_fuse_frame": (i32, [vp, vp, i32, vp, vp, vp, i32, i32, vp, P(SsRig)]),
        "ss_fusion_fuse_device": (i32, [vp, vp, vp, vp, vp, i32, i32, vp, P(SsRig), vp]),
        "ss_remove_outliers": (i32, [vp, vp, i32, i32, i32, f64, vp, vp]),
        "ss_fill_holes": (i32, [vp, vp, i32, i32, i32, i32, i32, vp, vp]),
        "ss_cleanup_pass": (i32, [P(SsParams), vp, vp, i32, i32, vp, vp]),
        "ss_refine_disparities": (i32, [P(SsParams), vp, vp, i32, i32, vp, i32, i32, vp, i32,
                                        i32, vp, vp, vp, vp]),
        "ss_disparity_to_cloud": (i32, [vp, vp, i32, i32, vp, i32, i32, P(SsRig), vp, vp, vp,
                                        vp, vp, P(i32), vp]),
        "ss_ctx_create": (i32, [i32, i32, i32, i32, P(SsParams), P(SsRig), P(vp)]),
        "ss_ctx_destroy": (i32, [vp]),
        "ss_ctx_stream": (vp, [vp]),
        "ss_ctx_sync": (i32, [vp]),
        "ss_ctx_get_stats": (i32, [vp, P(SsCtxStats)]),
        "ss_ctx_reset_stats": (i32, [vp]),
        "ss_stereo_batch": (i32, [vp, i32, i32, i32, i32, vp, vp, C.c_uint32, P(SsBatchOut)]),
        "ss_stereo_frame": (i32, [P(SsParams), P(SsRig), i32, i32, i32, vp, vp,
                                  C.c_uint32, P(SsBatchOut)]),
        "ss_stereo_batch_device": (i32, [vp, i32, i32, i32, i32, vp, vp, C.c_uint32,
                                         P(SsBatchOut), vp]),
        "ss_ctx_device_outputs": (i32, [vp, P(SsBatchOut)]),
        "ss_ctx_set_lr_check": (i32, [vp, i32, i32]),
        "ss_ctx_enable_timing": (i32, [vp, i32]),
        "ss_ctx_stage_times": (i32, [vp, P(C.c_double), P(C.c_int64)]),
        "ss_multi_create": (i32, [i32, P(i32), i32, i32, i32, P(SsParams), P(SsRig), P(vp)]),
        "ss_multi_destroy": (i32, [vp]),
        "ss_multi_size": (i32, [vp]),
        "ss_multi_set_lr_check": (i32, [vp, i32, i32]),
        "ss_multi_stereo_batch": (i32, [vp, i32, i32, i32, i32, vp, vp, C.c_uint32,
                                        P(SsBatchOut)]),
        "ss_multi_last_error": (C.c_char_p, []),
        "ss_host_alloc": (vp, [C.c_size_t]),
        "ss_host_free": (None, [vp]),
        "ss_oct_decode": (None, [vp, C.c_int64, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
