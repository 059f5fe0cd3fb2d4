// Internal declarations shared by the sm_100a kernels and the runtime.
//
// HBM layout of one frame (all frame-major; frame f of a batch at f * stride):
//   gray[N]                  u8  row-major luma (exact path, cloud colours)
//   plane[H][2][PP]          u8  parity-split rows: [.][0] even columns,
//                                [.][1] odd columns, PB bytes of zero padding
//                                each side -> any 4-byte window of a chessboard
//                                row is two aligned loads + one funnel shift
//   lstat[N]                 int2 {chessboard sum, float bits of 1/sqrt(var)}
//   rstat[H][SP]             int2 same for the right image, SPAD padded
//                                columns each side hold {0, NaN}
//   win[N][kWin]             f16 s(c) = num(c) / sqrt(var_l var_r) for the
//                                16 candidates c = wbase[N] + q around the
//                                pixel's disparity (refinement re-pick input)
//   disp/valid               f32/u8 DisparityMap (image.hpp:46-67)
//   refine state             f64 o, d, avg, b; psum[H][W+1]; cnt[N] (int)
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssb {

constexpr int kDB = 16;        // disparities per thread in the WTA sweep
constexpr int kRefineR = 5;    // kRefineSearchRadius (params.hpp:38)
constexpr double kZnccEps = 1e-3;  // kZnccCostEpsilon (params.hpp:34)
constexpr int kWin = 16;           // candidate window per pixel for the refinement
// Window scores are stored as fp16 (32 B per pixel, one sector): the re-pick
// filter's error budget covers it (|cost_f - cost| <= 5.4e-4 rel).
typedef __half wscore_t;
__device__ __forceinline__ uint32_t pack_score2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
constexpr int kNoWin = -2147483647 - 1;  // INT_MIN: no window / no defined candidate

// Window [base, base + kWin) around an anchor disparity, kept inside the
// candidate range [cmin, cmin + NC).
__host__ __device__ inline int window_base(int anchor, int cmin, int NC) {
  const int hi = NC > kWin ? cmin + NC - kWin : cmin;
  const int b = anchor - 7;
  return b < cmin ? cmin : (b > hi ? hi : b);
}

struct Geom {
  int W, H;        // frame size
  int half;        // window / 2
  int dmin, dmax;  // candidate range of the WTA
  int cmin, NC;    // volume range [cmin, cmin + NC)
  int NCP;         // per-pixel volume pitch (NC rounded up to 4 floats)
  int PB, PP;      // plane padding (bytes) and row pitch (bytes)
  int SPAD, SP;    // right-stat padding (elements) and row pitch
  long N() const { return (long)W * H; }
};

// ---- launchers (stream-ordered, frame index in blockIdx.z / y) ----
void launch_to_gray(const uint8_t* rgb, uint8_t* gray, long n_pixels, int frames,
                    long in_stride, long out_stride, cudaStream_t s);
void launch_planes(const uint8_t* gray, uint8_t* plane, const Geom& g, int frames,
                   long gray_stride, long plane_stride, cudaStream_t s);
void launch_stats(const uint8_t* gray, int2* lstat, int2* rstat, int is_right, const Geom& g,
                  int frames, long gray_stride, long stat_stride, cudaStream_t s);
// Sweep + WTA. Also writes, per interior pixel, the refinement's candidate
// window: kWin scores s(c) = g(c) / sqrt(var_l) for c = wbase .. wbase+kWin-1,
// wbase centred on the WTA pick, or on base_map[pixel] when base_map != NULL
// (per-stage refine). wbase = kNoWin when var_l == 0 (no defined score).
void launch_wta11(const uint8_t* lplane, const uint8_t* rplane, const int2* lstat,
                  const int2* rstat, wscore_t* win, int* wbase, const int* base_map, float* disp,
                  uint8_t* valid, int* flag_list, unsigned int* flag_count, const Geom& g,
                  double min_zncc, int frames, long plane_stride, long lstat_stride,
                  long rstat_stride, long map_stride, int do_argmax, cudaStream_t s);
// After cleanup: every valid pixel whose window is not centred on its
// (possibly filled) disparity gets a freshly computed window.
void launch_window_fix(const float* disp, const uint8_t* valid, const uint8_t* lgray,
                       const uint8_t* rgray, const int2* lstat, const int2* rstat, wscore_t* win,
                       int* wbase, int* list, unsigned* count, const Geom& g, int frames,
                       long stride, long rstat_stride, cudaStream_t s);
void launch_wta_resolve(const uint8_t* lgray, const uint8_t* rgray, const int* flag_list,
                        const unsigned int* flag_count, float* disp, uint8_t* valid,
                        const Geom& g, double min_zncc, int frames, long gray_stride,
                        long map_stride, long flag_stride, unsigned long long* counters,
                        cudaStream_t s);
void launch_wta_generic(const uint8_t* lgray, const uint8_t* rgray, float* disp,
                        uint8_t* valid, const Geom& g, double min_zncc, int frames,
                        long gray_stride, long map_stride, cudaStream_t s);

void launch_remove_outliers(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                            int W, int H, int radius, double thr, int frames, long stride,
                            cudaStream_t s);
void launch_fill_radial(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                        int W, int H, int radius, int min_support, int frames, long stride,
                        cudaStream_t s);
// pcnt: scratch [frames][H][W+1] ints; list: scratch [frames][W*H]; count: [frames]
void launch_fill_disc(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                      int W, int H, int radius, int min_support, const double* wtab,
                      const int* span, int* pcnt, int* list, unsigned* count, int frames,
                      long stride, cudaStream_t s);

struct RefineArgs {
  Geom g;
  double alpha, one_minus_alpha, eta, lo, hi;
  float eta_f;
  int radius;       // smoothing_radius
  const int* span;  // [radius + 1]
};
void launch_refine_init(const float* disp, const uint8_t* valid, double* o, double* d,
                        int W, int H, int frames, long stride, cudaStream_t s);
// normal-layout per-row prefix counts (cleanup disc support)
void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s);
// ---- BT layout (row-blocked transposed, k_scan.cu): element (v, c) at
// ((v/32) * CW + c) * 32 + v%32; frame stride ceil(H/32) * CW * 32 ----
__host__ __device__ inline long bt_frame(int W, int H, int extra_col) { return (long)((H + 31) / 32) * (W + extra_col) * 32; }
void launch_mask_bt(const uint8_t* mask, uint8_t* mT, int W, int H, int frames, long stride,
                    cudaStream_t s);
void launch_ones_bt(const uint8_t* mask, int* outT, int W, int H, int frames, long stride,
                    cudaStream_t s);
void launch_double_bt(const double* val, const uint8_t* mask, double* outT, int W, int H,
                      int frames, long stride, cudaStream_t s);
void launch_int_bt(const int* val, const uint8_t* mask, int* outT, int W, int H, int frames,
                   long stride, cudaStream_t s);
void launch_b_bt(const int* so, const int* cnt, const int* o, const double* d, double alpha,
                 double one_minus_alpha, const uint8_t* mask, double* bT, int W, int H,
                 int frames, long stride, cudaStream_t s);
// masked serial row prefix (psum[.][0] = 0, W + 1 columns, BT layout)
void launch_scan_bt_d(const double* xT, const uint8_t* mT, double* pT, int W, int H, int frames,
                      cudaStream_t s);
void launch_scan_bt_i(const int* xT, const uint8_t* mT, int* pT, int W, int H, int frames,
                      cudaStream_t s);
// exact integer disc sums from an int BT prefix (disc counts, S_o)
void launch_disc_isum(const uint8_t* valid, const int* ipsumT, int* out, const RefineArgs& a,
                      int frames, long stride, cudaStream_t s);
// iteration 0: avg = disc mean of o (FP64, reference order), b (normal layout)
void launch_avg_b(const double* psumT, const uint8_t* valid, const int* cnt, const double* o,
                  const double* d, double* avg, double* b, const RefineArgs& a, int frames,
                  long stride, cudaStream_t s);
// avg: the double disc mean of o (iteration 0) or nullptr to use the exact
// integer disc sum `so` (iterations >= 1); o changes are appended to chg.
// Re-picks whose FP32 window filter is ambiguous, or whose candidates leave
// the window, are deferred to launch_repick_exact (warp per pixel, FP64).
struct Deferred {
  int pix, c_lo, mask, pad;  // mask: candidates c_lo + k to score exactly
  double d;
};
// o: integer disparities (written by every re-pick; read for the change list
// when avg == nullptr, i.e. iterations >= 1).
void launch_d_repick(const double* psumT, const uint8_t* valid, const int* cnt,
                     const double* avg, const int* so, double* d, int* o,
                     const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                     const int* wbase, int2* chg, unsigned* chg_count, Deferred* defer,
                     unsigned* defer_count, const RefineArgs& a, int frames, long stride,
                     long gray_stride, unsigned long long* counters, cudaStream_t s);
void launch_repick_exact(const Deferred* defer, const unsigned* defer_count, int* o,
                         const uint8_t* lgray, const uint8_t* rgray, int2* chg,
                         unsigned* chg_count, const RefineArgs& a, int frames, long stride,
                         long gray_stride, unsigned long long* counters, cudaStream_t s);
// S_o += delta over the disc of every changed pixel (exact integers).
void launch_so_update(const int2* chg, const unsigned* chg_count, const uint8_t* valid,
                      int* so, const RefineArgs& a, int frames, long stride, cudaStream_t s);
void launch_refine_out(const double* d, const uint8_t* valid, const float* din, float* dout,
                       int W, int H, int frames, long stride, cudaStream_t s);
void launch_int_to_double(const int* x, const uint8_t* valid, double* y, long n,
                          cudaStream_t s);

struct CloudArgs {
  double fx, fy, cx, cy, baseline;
};
void launch_cloud_index(const float* disp, const uint8_t* valid, int* index, int* block_sums,
                        int* n_points, int W, int H, int frames, long stride, cudaStream_t s);
void launch_cloud_points(const float* disp, const int* index, const uint8_t* rgb, int cw,
                         int ch, int W, int H, const CloudArgs& c, double* pts_d,
                         float* pts_f, float4* pts4, uint8_t* colors, int* pixels, int frames,
                         long stride, long rgb_stride, cudaStream_t s);
void launch_cloud_normals(const float4* pts4, const float* disp, const int* index,
                          const CloudArgs& c, double* nrm_d, float* nrm_f, int W, int H,
                          int frames, long stride, cudaStream_t s);

}  // namespace ssb
