"""stereoscan-b200: B200-native (sm_100a) per-frame dense stereo path of
arXiv:2007.12623 — ZNCC WTA, outlier removal + hole filling, improved-Laplacian
refinement and back-projection — behind the reference's own entry points.

The compute lives in ``lib/libstereoscan_b200.so`` (csrc/, C-ABI in
include/ss_stereo.h). This package is the host-side mirror of the reference
interface; it has no CPU fallback.
"""
from .stereo import (  # noqa: F401
    InvalidArgument,
    StereoCloud,
    StereoContext,
    StereoMulti,
    StereoError,
    StereoParams,
    StereoRig,
    cleanup_pass,
    compute_disparity,
    compute_disparity_lr,
    decode_oct_normals,
    device_count,
    disc_fill_min_support,
    disc_neighbor_count,
    disparity_to_cloud,
    fill_holes,
    pinned_empty,
    refine_disparities,
    remove_outliers,
    stereo_frame,
    to_gray,
)
from . import features, fusion  # noqa: F401
from ._lib import (SS_IN_GRAY, SS_IN_RGB, SS_OUT_CLOUD, SS_OUT_DISPARITY, SS_OUT_NORMALS,  # noqa: F401
                   SS_OUT_NORMALS_OCT, SS_OUT_TRIM)
