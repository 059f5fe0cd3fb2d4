/*
 * ORACLE — test infrastructure only. Nothing in the product links this.
 *
 * One C interface, two implementations:
 *   ref_*  oracle/ref_capi.cpp: thin extern "C" wrapper around the UNMODIFIED
 *          reference sources /root/reference/proj/src/stereo/{matcher,
 *          reference,cleanup,smoothing}.cpp, built by oracle/Makefile into
 *          oracle/_ref/libss_ref.so (only where /root/reference exists).
 *   orc_*  oracle/ss_oracle.c: a plain-C restatement of the same algorithms
 *          (plus disparity_to_cloud, which the reference cannot build without
 *          Eigen), built into oracle/build/libss_oracle.so.
 *
 * Tests, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference arm are the only callers.
 *
 * Status codes: 0 ok, 1 std::invalid_argument, 2 stereoscan::Error.
 * The message of the last failure on the calling thread is X_last_error().
 */
#ifndef SS_ORACLE_H
#define SS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field-for-field copy of stereoscan::StereoParams (params.hpp:7-24). */
typedef struct {
  int32_t window;
  int32_t d_min;
  int32_t d_max;
  double neighbor_jump_threshold;
  int32_t outlier_radius_start;
  int32_t outlier_radius_step;
  int32_t cleanup_iterations;
  int32_t fill_radius_radial;
  int32_t fill_radius_disc;
  int32_t smoothing_radius;
  double alpha;
  double eta_smooth;
  int32_t refine_iterations;
  double min_zncc;
} orc_params;

/* CameraIntrinsics + StereoRig (types.hpp:23-40). */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double baseline_mm;
} orc_rig;

#define SS_ORACLE_DECLARE(P)                                                   \
  const char* P##last_error(void);                                            \
  int P##to_gray(const uint8_t* rgb, int32_t w, int32_t h, uint8_t* gray);    \
  double P##zncc_chessboard(const uint8_t* left, const uint8_t* right,        \
                            int32_t w, int32_t h, int32_t lu, int32_t lv,     \
                            int32_t ru, int32_t rv, int32_t window,           \
                            int32_t* defined);                                \
  int P##compute_disparity(const orc_params* p, const uint8_t* left,          \
                           const uint8_t* right, int32_t w, int32_t h,        \
                           float* disp, uint8_t* valid);                      \
  int P##remove_outliers(const float* disp, const uint8_t* valid, int32_t w,  \
                         int32_t h, int32_t radius, double threshold,         \
                         float* out_disp, uint8_t* out_valid);                \
  int P##fill_holes(const float* disp, const uint8_t* valid, int32_t w,       \
                    int32_t h, int32_t mode, int32_t radius,                  \
                    int32_t min_support, float* out_disp,                     \
                    uint8_t* out_valid);                                      \
  int32_t P##disc_neighbor_count(int32_t radius);                             \
  int32_t P##disc_fill_min_support(int32_t radius);                           \
  int P##cleanup_pass(const orc_params* p, const float* disp,                 \
                      const uint8_t* valid, int32_t w, int32_t h,             \
                      float* out_disp, uint8_t* out_valid);                   \
  int P##refine_disparities(const orc_params* p, const float* disp,           \
                            const uint8_t* valid, const uint8_t* left,        \
                            const uint8_t* right, int32_t w, int32_t h,       \
                            float* out_disp, uint8_t* out_valid,              \
                            double* trace_discrete, double* trace_smooth);

SS_ORACLE_DECLARE(ref_)
SS_ORACLE_DECLARE(orc_)

/* Reference-only: the deliberately naive twins (reference.hpp:15,19). */
int ref_naive_compute_disparity(const orc_params* p, const uint8_t* left,
                                const uint8_t* right, int32_t w, int32_t h,
                                float* disp, uint8_t* valid);
int ref_naive_remove_outliers(const float* disp, const uint8_t* valid,
                              int32_t w, int32_t h, int32_t radius,
                              double threshold, float* out_disp,
                              uint8_t* out_valid);
int ref_params_validate(const orc_params* p);

/* Reference-only: the feature front end (features.cpp:86-258; SURVEY.md §8f
 * row 4), the oracle of the GPU feature kernels. */
int ref_detect_corners(const uint8_t* gray, int32_t w, int32_t h, int32_t max_count,
                       int32_t threshold, int32_t* us, int32_t* vs, int32_t* scores,
                       int32_t* n);
int ref_describe(const uint8_t* gray, int32_t w, int32_t h, const int32_t* us,
                 const int32_t* vs, const int32_t* scores, int32_t nc, double* pos,
                 uint64_t* desc, int32_t* n);
int ref_match_features(const double* pos_a, const uint64_t* desc_a, int32_t na,
                       const double* pos_b, const uint64_t* desc_b, int32_t nb,
                       int32_t max_hamming, int32_t* ia, int32_t* ib, int32_t* ham,
                       double* disp, int32_t* n);
int ref_histogram_vote(const int32_t* ia, const int32_t* ib, const int32_t* ham,
                       const double* disp, int32_t n, double bin_size, int32_t* order);

/* Restatement-only: disparity_to_cloud (cloud.cpp:14-94); the normals'
 * eigensolver restates Eigen 3.4.0 SelfAdjointEigenSolver (orc_eigen3_sym).
 * Outputs are sized for w*h points; *n_points receives the count.
 * points/normals are xyz doubles per point, colors rgb bytes, pixels (u,v).
 * eigen_gap (optional): (l1 - l0) / l2 of fitted points, -1 otherwise;
 * decision (optional): (l1 - t) / t with t = 1e-9 max(1, l2), the relative
 * margin of the fit/fallback test of cloud.cpp:81 (> 0: fitted; -inf: fewer
 * than 3 neighbours). */
int orc_disparity_to_cloud(const float* disp, const uint8_t* valid, int32_t w,
                           int32_t h, const uint8_t* rgb, int32_t cw,
                           int32_t ch, const orc_rig* rig, int32_t* index,
                           double* points, double* normals, uint8_t* colors,
                           int32_t* pixels, int32_t* n_points,
                           double* eigen_gap, double* decision);
/* Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d> restatement on a row-major
 * 3x3 (lower triangle read): ascending evals, evec9[r*3+k] = component r of
 * eigenvector k. Returns 1 on NoConvergence. */
int orc_eigen3_sym(const double* a9, double* evals, double* evec9);
/* Restatement-only: opt-in left-right consistency (extension, no reference
 * analogue): right-view WTA and the check (ss_compute_disparity_lr). */
int orc_compute_disparity_right(const orc_params* p, const uint8_t* left,
                                const uint8_t* right, int32_t w, int32_t h,
                                float* disp, uint8_t* valid);
int orc_lr_check(const float* disp, const uint8_t* valid, const float* disp_r,
                 const uint8_t* valid_r, int32_t w, int32_t h, int32_t max_diff,
                 float* out_disp, uint8_t* out_valid);
/* Restatement-only: the fusion consumer (no reference
 * source; conventions in ss_oracle.c). */
int orc_rasterize(const double* pos, int32_t n, const double* pose, double fx, double fy,
                  double cx, double cy, int32_t w, int32_t h, int32_t* ids, double* depth);
int orc_fuse_frame(double* pos, double* nrm, double* col, double* wgt, double* cwgt, int32_t* n,
                   int32_t cap, const int32_t* index, const double* pts, const double* nrms,
                   const uint8_t* colors, int32_t w, int32_t h, const double* pose, double fx,
                   double fy, double cx, double cy, double trunc, double weight_cap,
                   double gate, double omega_min);
int orc_params_validate(const orc_params* p);
int orc_rig_validate(const orc_rig* rig);

#ifdef __cplusplus
}
#endif

#endif /* SS_ORACLE_H */
