/*
 * ss_stereo.h — C-ABI of the B200-native per-frame dense stereo path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/stereoscan/stereo/*.hpp). Every entry point
 * takes plain pointers and sizes; no C++ or torch types cross it. The C++
 * header tree include/stereoscan/ re-declares the reference's functions on top
 * of these calls (INTEGRATION.md shows the reference-side binding).
 *
 *   ss_to_gray              replaces to_gray             image.hpp:44, matcher.cpp:21-30
 *   ss_compute_disparity    replaces compute_disparity   matcher.hpp:35-36, matcher.cpp:166-211
 *   ss_remove_outliers      replaces remove_outliers     cleanup.hpp:12, cleanup.cpp:12-42
 *   ss_fill_holes           replaces fill_holes          cleanup.hpp:21-22, cleanup.cpp:44-92
 *   ss_cleanup_pass         replaces cleanup_pass        cleanup.hpp:32, cleanup.cpp:111-123
 *   ss_refine_disparities   replaces refine_disparities  smoothing.hpp:22-24, smoothing.cpp:68-159
 *   ss_disparity_to_cloud   replaces disparity_to_cloud  cloud.hpp:34-35, cloud.cpp:14-94
 *   ss_params_validate      replaces StereoParams::validate  params.hpp:23, matcher.cpp:9-19
 *   ss_rig_validate         replaces StereoRig::validate     types.hpp:39, geometry.cpp:7-19
 *   ss_detect_corners       replaces features::detect_corners  features.hpp:52, features.cpp:86-124
 *   ss_describe             replaces features::describe        features.hpp:57, features.cpp:126-166
 *   ss_match_features       replaces features::match_features  features.hpp:61, features.cpp:168-208
 *   ss_fusion_*             the SPEC's fusion module (no reference source)
 *
 * Throughput entry (no reference analogue): ss_ctx_* run the
 * whole run_stereo_only chain for a batch of frames on one
 * GPU, device-resident between stages.
 *
 * Errors: functions return ss_status; on failure ss_last_error() holds the
 * message for the calling thread. SS_EINVAL maps to std::invalid_argument and
 * SS_EPARAM to stereoscan::Error in the C++ layer (same messages as the
 * reference). There is no CPU fallback: without a CUDA device every compute
 * entry point returns SS_ENODEV.
 */
#ifndef SS_STEREO_H
#define SS_STEREO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ss_status;
#define SS_OK 0
#define SS_EINVAL 1   /* contract violation   -> std::invalid_argument */
#define SS_EPARAM 2   /* parameter/geometry   -> stereoscan::Error      */
#define SS_ECUDA 3    /* CUDA runtime failure                           */
#define SS_ENOMEM 4   /* device allocation failure                      */
#define SS_ENODEV 5   /* no CUDA device: the path refuses to run on CPU */

/* Field-for-field stereoscan::StereoParams (params.hpp:7-24). */
typedef struct ss_stereo_params {
  int32_t window;                  /* 11 */
  int32_t d_min;                   /* -20 */
  int32_t d_max;                   /* 80 */
  double neighbor_jump_threshold;  /* 2.5 */
  int32_t outlier_radius_start;    /* 10 */
  int32_t outlier_radius_step;     /* 10 */
  int32_t cleanup_iterations;      /* 3 */
  int32_t fill_radius_radial;      /* 50 */
  int32_t fill_radius_disc;        /* 20 */
  int32_t smoothing_radius;        /* 15 */
  double alpha;                    /* 0.1 */
  double eta_smooth;               /* 0.01 */
  int32_t refine_iterations;       /* 10 */
  double min_zncc;                 /* 0.5 */
} ss_stereo_params;

/* CameraIntrinsics + StereoRig (types.hpp:23-40). */
typedef struct ss_stereo_rig {
  double fx, fy, cx, cy;
  int32_t width, height;
  double baseline_mm;
} ss_stereo_rig;

/* fill_holes modes (cleanup.hpp:14). */
#define SS_FILL_RADIAL 0
#define SS_FILL_DISC 1

const char* ss_last_error(void);
const char* ss_version(void);
void ss_params_default(ss_stereo_params* p);
ss_status ss_params_validate(const ss_stereo_params* p);
ss_status ss_rig_validate(const ss_stereo_rig* rig);
int32_t ss_disc_neighbor_count(int32_t radius);    /* cleanup.cpp:94-104 */
int32_t ss_disc_fill_min_support(int32_t radius);  /* cleanup.cpp:106-109 */
int32_t ss_device_count(void);

/* ---- per-stage drop-ins: host buffers in, host buffers out (synchronous) ---- */

ss_status ss_to_gray(const uint8_t* rgb, int32_t w, int32_t h, uint8_t* gray);

ss_status ss_compute_disparity(const ss_stereo_params* p, const uint8_t* left, int32_t lw,
                               int32_t lh, const uint8_t* right, int32_t rw, int32_t rh,
                               float* disparity, uint8_t* valid);

/* Opt-in left-right consistency (no reference analogue: an extension named by
 * the north star). compute_disparity plus the right-view
 * WTA d_R(x) = first argmax over d of zncc(left at x + d, right at x); a valid
 * left pixel u with disparity d is kept iff x = u - d is inside the image, the
 * right view is valid there and |d_R(x) - d| <= max_diff, else it becomes
 * (0, invalid). right_disparity / right_valid (nullable) receive the
 * right-view map in right-image coordinates. */
ss_status ss_compute_disparity_lr(const ss_stereo_params* p, const uint8_t* left, int32_t lw,
                                  int32_t lh, const uint8_t* right, int32_t rw, int32_t rh,
                                  int32_t max_diff, float* disparity, uint8_t* valid,
                                  float* right_disparity, uint8_t* right_valid);

ss_status ss_remove_outliers(const float* disparity, const uint8_t* valid, int32_t w,
                             int32_t h, int32_t radius, double threshold, float* out_disparity,
                             uint8_t* out_valid);

ss_status ss_fill_holes(const float* disparity, const uint8_t* valid, int32_t w, int32_t h,
                        int32_t mode, int32_t radius, int32_t min_support,
                        float* out_disparity, uint8_t* out_valid);

ss_status ss_cleanup_pass(const ss_stereo_params* p, const float* disparity,
                          const uint8_t* valid, int32_t w, int32_t h, float* out_disparity,
                          uint8_t* out_valid);

/* trace_discrete / trace_smooth: NULL or refine_iterations * w * h doubles,
 * the RefineTrace snapshots of smoothing.hpp:10-13 (smoothing.cpp:148-151). */
ss_status ss_refine_disparities(const ss_stereo_params* p, const float* disparity,
                                const uint8_t* valid, int32_t w, int32_t h,
                                const uint8_t* left, int32_t lw, int32_t lh,
                                const uint8_t* right, int32_t rw, int32_t rh,
                                float* out_disparity, uint8_t* out_valid,
                                double* trace_discrete, double* trace_smooth);

/* StereoCloud (cloud.hpp:14-29): index[w*h]; per point (capacity w*h):
 * points xyz, normals xyz (double), colors rgb, pixels (u,v). fitted
 * (optional, may be NULL): 1 where the normal is the plane fit, 0 where the
 * fit/fallback test of cloud.cpp:81 chose the sight-ray fallback. */
ss_status ss_disparity_to_cloud(const float* disparity, const uint8_t* valid, int32_t w,
                                int32_t h, const uint8_t* rgb, int32_t cw, int32_t ch,
                                const ss_stereo_rig* rig, int32_t* index, double* points,
                                double* normals, uint8_t* colors, int32_t* pixels,
                                int32_t* n_points, uint8_t* fitted);

/* ---- feature front end (features.hpp:45-66) ----
 * Same results as the reference (integer work, bit-exact). */

/* detect_corners (features.hpp:52, features.cpp:86-124): u/v/score arrays of
 * capacity max_count, sorted by score descending then raster order; *n gets
 * the count. threshold < 1 -> SS_EINVAL "detect_corners: threshold must be >= 1". */
ss_status ss_detect_corners(const uint8_t* gray, int32_t w, int32_t h, int32_t max_count,
                            int32_t threshold, int32_t* u, int32_t* v, int32_t* score,
                            int32_t* n);

/* describe (features.hpp:57, features.cpp:126-166): for the given corners (in
 * order; those within 16 px of the border dropped) the position (u, v) as
 * doubles and the 256-bit descriptor as 4 x uint64 (Descriptor256::bits);
 * capacity n_corners; *n gets the count. */
ss_status ss_describe(const uint8_t* gray, int32_t w, int32_t h, const int32_t* u,
                      const int32_t* v, const int32_t* score, int32_t n_corners, double* pos,
                      uint64_t* desc, int32_t* n);

/* match_features (features.hpp:61, features.cpp:168-208): mutual Hamming
 * nearest neighbours gated at max_hamming, in index_a order; per match
 * index_a, index_b, hamming and displacement (b - a, 2 doubles); capacity
 * min(na, nb); *n gets the count. */
ss_status ss_match_features(const double* pos_a, const uint64_t* desc_a, int32_t na,
                            const double* pos_b, const uint64_t* desc_b, int32_t nb,
                            int32_t max_hamming, int32_t* index_a, int32_t* index_b,
                            int32_t* hamming, double* displacement, int32_t* n);

/* ---- fusion consumer (SPEC.md:440-476 [MODULE] fusion) ----
 * The surfel model lives on the GPU; keyframe clouds are fused where they
 * were produced. The reference has no source for this module: the rules are
 * the SPEC's (DESIGN.md §12 lists the conventions), with the SPEC's defaults.
 *   pose[12]: row-major [R | t] mapping world to camera (X_cam = R X_world + t).
 *   rasterize: surfels with X_cam.z > 0 project to pixel (floor(fx x/z + cx +
 *     0.5), floor(fy y/z + cy + 0.5)); the smallest depth wins, then the smaller
 *     surfel id; ids -1 / depth 0 where empty.
 *   fuse: every pixel with a point (raster order) associates with the raster's
 *     surfel when |z - z_surfel| <= gate: increment clamped to trunc_mm, weight
 *     average (new observation weight 1), weight <- min(weight + 1, cap), normal
 *     re-normalised, colour averaged with omega(u,v) = clamp(1 - r/R, omega_min,
 *     1) (r: distance to the image centre, R: half-diagonal); other pixels are
 *     appended as new surfels (weight 1) in raster order. */
typedef struct ss_fusion_params {
  double trunc_mm;            /* 10 */
  double weight_cap;          /* 50 */
  double association_gate_mm; /* 5 */
  double omega_min;           /* 0.1 */
} ss_fusion_params;

typedef struct ss_fusion ss_fusion;

void ss_fusion_params_default(ss_fusion_params* p);
ss_status ss_fusion_create(int32_t device, const ss_fusion_params* p, ss_fusion** out);
ss_status ss_fusion_destroy(ss_fusion* f);
ss_status ss_fusion_size(ss_fusion* f, int32_t* n);
/* Replace / read the model: pos, normal, colour (3 doubles each), weight,
 * colour weight per surfel (NULL outputs are skipped). */
ss_status ss_fusion_upload(ss_fusion* f, int32_t n, const double* pos, const double* normal,
                           const double* color, const double* weight,
                           const double* color_weight);
ss_status ss_fusion_download(ss_fusion* f, double* pos, double* normal, double* color,
                             double* weight, double* color_weight);
/* rasterize: ids / depth of rig->width * rig->height pixels. */
ss_status ss_fusion_rasterize(ss_fusion* f, const double* pose, const ss_stereo_rig* rig,
                              int32_t* ids, double* depth);
/* fuse_frame from host arrays: a StereoCloud (index per
 * pixel, points / normals as doubles in the camera frame, colours). */
ss_status ss_fusion_fuse_frame(ss_fusion* f, const int32_t* index, int32_t n_points,
                               const double* points, const double* normals,
                               const uint8_t* colors, int32_t w, int32_t h, const double* pose,
                               const ss_stereo_rig* rig);
/* Same from DEVICE arrays of one frame as the batch API leaves them
 * (ss_ctx_device_outputs / ss_stereo_batch_device: index, float points and
 * normals, colours); `stream` (nullable) is the producer stream to wait on. */
ss_status ss_fusion_fuse_device(ss_fusion* f, const int32_t* d_index, const float* d_points,
                                const float* d_normals, const uint8_t* d_colors, int32_t w,
                                int32_t h, const double* pose, const ss_stereo_rig* rig,
                                void* stream);

/* ---- throughput API: a batch of frames through the whole chain on one GPU ---- */

typedef struct ss_ctx ss_ctx;

#define SS_IN_RGB 0   /* interleaved 8-bit RGB, luma by to_gray */
#define SS_IN_GRAY 1  /* 8-bit gray */

#define SS_OUT_DISPARITY 1u  /* disparity (f32) + valid (u8) per pixel */
#define SS_OUT_CLOUD 2u      /* packed cloud: index, points f32x3, colors */
#define SS_OUT_NORMALS 4u    /* normals f32x3 (needs SS_OUT_CLOUD) */
/* Compact transfer formats (opt-in; the default outputs are the reference's):
 * SS_OUT_NORMALS_OCT  normals as 2 x int16 octahedral snorm per point in
 *                     `normals_oct` instead of f32x3 in `normals` (4 B instead
 *                     of 12 B; decoded direction within 1e-4 rad, see
 *                     ss_oct_decode); implies SS_OUT_NORMALS.
 * SS_OUT_TRIM         host API only: points / normals / colors leave the GPU
 *                     with n_points entries per frame instead of the full
 *                     per-frame capacity (one count read-back per chunk). */
#define SS_OUT_NORMALS_OCT 8u
#define SS_OUT_TRIM 16u

/* Per-batch outputs. Host pointers for ss_stereo_batch, device pointers for
 * ss_stereo_batch_device. Arrays are frame-major: frame f of n starts at
 * f*w*h (index, disparity, valid) or f*w*h*3 (points, normals, colors).
 * Points of a frame are packed in raster order (cloud.cpp:23-39). */
typedef struct ss_batch_out {
  float* disparity;
  uint8_t* valid;
  int32_t* index;
  float* points;
  float* normals;
  uint8_t* colors;
  int32_t* n_points; /* n entries */
  int16_t* normals_oct; /* SS_OUT_NORMALS_OCT: [n][w*h][2] */
} ss_batch_out;

/* Decode n SS_OUT_NORMALS_OCT normals (octahedral map, snorm16) on the host:
 * enc[2k], enc[2k+1] -> unit xyz in out[3k..3k+2]. */
void ss_oct_decode(const int16_t* enc, int64_t n, float* out);

typedef struct ss_ctx_stats {
  int64_t frames;            /* frames processed */
  int64_t wta_resolved;      /* pixels whose WTA pick went through the exact FP64 resolve */
  int64_t refine_resolved;   /* (pixel, iteration) re-picks resolved in exact FP64 */
  int64_t refine_scored;     /* (pixel, iteration) re-picks scored; the others were certified
                                unchanged (window 11, smoothing radius 15) */
  int64_t kernel_launches;   /* kernels launched by this ctx */
  int64_t disc_fill_pixels;  /* pixels that went through the disc fill (all cleanup rounds) */
  int64_t graph_launches;    /* batch chains launched as one captured CUDA graph */
} ss_ctx_stats;

ss_status ss_ctx_create(int32_t device, int32_t max_w, int32_t max_h, int32_t max_batch,
                        const ss_stereo_params* p, const ss_stereo_rig* rig, ss_ctx** out);
ss_status ss_ctx_destroy(ss_ctx* ctx);
/* cudaStream_t the ctx launches on (as void*). */
void* ss_ctx_stream(ss_ctx* ctx);
ss_status ss_ctx_sync(ss_ctx* ctx);
ss_status ss_ctx_get_stats(ss_ctx* ctx, ss_ctx_stats* st);
ss_status ss_ctx_reset_stats(ss_ctx* ctx);
/* Opt-in LR consistency inside the batch chain (after the WTA, before the
 * cleanup); off by default, which keeps the reference's output. */
ss_status ss_ctx_set_lr_check(ss_ctx* ctx, int32_t enable, int32_t max_diff);

/* Per-stage device time (CUDA events on the ctx stream), the Table III-style
 * RuntimeReport of SPEC.md:566-569 for the stereo stage. Stages:
 * 0 luma, 1 stats+planes, 2 cost sweep/WTA (k_wta11), 3 FP64 resolve,
 * 4 cleanup, 5 refine, 6 cloud; kernel groups nested inside them:
 * 7 outlier removal, 8 radial fill, 9 disc fill (inside 4), 10 refine row
 * prefix scans, 11 gather + re-picks (k_d_gather + k_repick_list; iteration 0:
 * k_d_repick), 12 exact re-picks of iteration 0 (inside 5), 13 normals
 * (inside 6). Timing is off by default; with timing on the batch chain is
 * launched kernel by kernel instead of as one CUDA graph. */
#define SS_N_STAGES 14
ss_status ss_ctx_enable_timing(ss_ctx* ctx, int32_t on);
/* Sums (ms) and launch counts per stage since the last reset; synchronizes. */
ss_status ss_ctx_stage_times(ss_ctx* ctx, double* ms, int64_t* launches);

/* Whole chain for n frames of w x h from HOST memory (pinned for full speed):
 * H2D, kernels, D2H on the ctx stream; returns after the outputs landed. */
ss_status ss_stereo_batch(ss_ctx* ctx, int32_t n, int32_t w, int32_t h, int32_t in_format,
                          const uint8_t* left, const uint8_t* right, uint32_t out_flags,
                          const ss_batch_out* out);

/* One pair through the whole chain (the fused per-frame entry of SURVEY.md
 * §8b): host buffers in and out, on the calling thread's lazily created
 * per-device context, synchronous. Equal to a one-frame ss_stereo_batch with
 * the same params / rig (rig may be NULL without SS_OUT_CLOUD / _NORMALS). */
ss_status ss_stereo_frame(const ss_stereo_params* p, const ss_stereo_rig* rig, int32_t w,
                          int32_t h, int32_t in_format, const uint8_t* left,
                          const uint8_t* right, uint32_t out_flags, const ss_batch_out* out);

/* Same with DEVICE inputs/outputs; asynchronous on `stream` (NULL = ctx
 * stream). Output device pointers may be NULL to keep results in the ctx's
 * own buffers (see ss_ctx_device_outputs). */
ss_status ss_stereo_batch_device(ss_ctx* ctx, int32_t n, int32_t w, int32_t h,
                                 int32_t in_format, const uint8_t* d_left,
                                 const uint8_t* d_right, uint32_t out_flags,
                                 const ss_batch_out* d_out, void* stream);

/* Device pointers of the ctx-owned result buffers of the last batch. */
ss_status ss_ctx_device_outputs(ss_ctx* ctx, ss_batch_out* d_out);

/* ---- in-process frame sharding across GPUs ----
 * One ctx and one host thread per device entry; a batch splits into
 * contiguous frame blocks (sizes differ by <= 1) and each device writes its
 * block straight into the caller's frame-ordered host outputs (the host-side
 * gather; no collective). Entries may repeat a device. Results are identical
 * to one ss_stereo_batch over all frames. On failure ss_multi_last_error()
 * names the device. */
typedef struct ss_multi ss_multi;
ss_status ss_multi_create(int32_t n_devices, const int32_t* devices, int32_t max_w, int32_t max_h,
                          int32_t max_batch, const ss_stereo_params* p, const ss_stereo_rig* rig,
                          ss_multi** out);
ss_status ss_multi_destroy(ss_multi* m);
int32_t ss_multi_size(const ss_multi* m);
ss_ctx* ss_multi_ctx(ss_multi* m, int32_t k);
ss_status ss_multi_set_lr_check(ss_multi* m, int32_t enable, int32_t max_diff);
ss_status ss_multi_stereo_batch(ss_multi* m, int32_t n, int32_t w, int32_t h, int32_t in_format,
                                const uint8_t* left, const uint8_t* right, uint32_t out_flags,
                                const ss_batch_out* out);
const char* ss_multi_last_error(void);

/* Pinned host memory helpers (cudaHostAlloc / cudaFreeHost). */
void* ss_host_alloc(size_t bytes);
void ss_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* SS_STEREO_H */
