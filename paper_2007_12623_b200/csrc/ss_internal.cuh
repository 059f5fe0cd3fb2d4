// Internal declarations shared by the sm_100a kernels and the runtime.
//
// HBM layout of one frame (all frame-major; frame f of a batch at f * stride):
//   gray[N]                  u8  row-major luma (exact path, cloud colours)
//   ltap[N]                  uint4 left tap words of pixel (u, v): the 5 even-
//                                and 6 odd-offset bytes of its chessboard row
//                                window, packed for dp4a (k_ltap)
//   rcopy[H][2][4][PP]       u8  right parity-split rows ([.][0] even columns,
//                                [.][1] odd, PB bytes of zero padding each
//                                side) in 4 copies shifted by 0..3 bytes: any
//                                byte offset of a row starts an aligned word
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
// Window entries hold the re-pick's match cost M = 1/max(s, kZnccCostEpsilon)
// (>= 1) as fp16 of M - 1 (32 B per pixel), so the good matches, M near 1,
// keep 3-4 more bits than fp16(M) would: exactly 999 (M16 = 1000 = 1/1e-3 in
// double) when the score is undefined or certainly clamped (s_f < 0.99e-3),
// otherwise fp16(min(1/max(s_f, 1e-3), 999.5) - 1), so M16 = 1000 always
// means "exact". With M16 = 1 + h (exact in FP32):
//   |M16 - M| <= kMA |M16 - 1| + kMB M16
// (fp16 rounding of M - 1 and the 999.5 cap: 5.02e-4; the FP32 score's 5 ulp,
// the 1-ulp reciprocal and the FP32 subtraction: < 1e-6 M), used by the
// re-pick filter's error bars.
constexpr float kMA = 5.1e-4f, kMB = 2e-6f;
typedef __half wscore_t;
__device__ __forceinline__ unsigned short m_code(float s) {
  if (!(s >= 0.99e-3f)) return __half_as_ushort(__float2half_rn(999.f));
  float r;  // 1 ulp reciprocal of a normal number
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(s, 1e-3f)));
  return __half_as_ushort(__float2half_rn(fminf(r, 999.5f) - 1.f));
}
// Two m_codes in one packed conversion (bit-identical to m_code: 999 and the
// capped reciprocal minus 1 convert exactly as there).
__device__ __forceinline__ float m_value(float s) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(s, 1e-3f)));
  return s >= 0.99e-3f ? fminf(r, 999.5f) - 1.f : 999.f;
}
__device__ __forceinline__ uint32_t pack_m2(float s0, float s1) {
  const __half2 h = __floats2half2_rn(m_value(s0), m_value(s1));
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
void launch_ltap(const uint8_t* gray, uint4* ltap, const Geom& g, int frames, long gray_stride,
                 long tap_stride, cudaStream_t s);
void launch_rcopy(const uint8_t* gray, uint32_t* rcopy, const Geom& g, int frames,
                  long gray_stride, long copy_stride, cudaStream_t s);
void launch_stats(const uint8_t* gray, int2* lstat, int2* rstat, int is_right, const Geom& g,
                  int frames, long gray_stride, long stat_stride, cudaStream_t s);
// Sweep + WTA. Also writes, per interior pixel, the refinement's candidate
// window: kWin scores s(c) = g(c) / sqrt(var_l) for c = wbase .. wbase+kWin-1,
// wbase centred on the WTA pick, or on base_map[pixel] when base_map != NULL
// (per-stage refine). wbase = kNoWin when var_l == 0 (no defined score) or
// when the window would reach past [d_min, d_max] (launch_window_build then
// rebuilds it for the pixels the refinement uses).
// win == NULL: argmax only (the right-view sweep of the LR check).
// win / wbase are BT-indexed (bt_index, frame stride win_stride).
void launch_wta11(const uint4* ltap, const uint32_t* rcopy, const int2* lstat,
                  const int2* rstat, wscore_t* win, int* wbase, const int* base_map, float* disp,
                  uint8_t* valid, int* flag_list, unsigned int* flag_count, const Geom& g,
                  double min_zncc, int frames, long tap_stride, long copy_stride,
                  long lstat_stride, long rstat_stride, long map_stride, long win_stride,
                  int do_argmax, cudaStream_t s);
// After cleanup: every valid pixel whose window is not centred on its
// (possibly filled) disparity gets a freshly computed window. The pixels are
// queued by launch_refine_init's window check (list / count, count zeroed
// before it).
void launch_window_build(const float* disp, const uint8_t* lgray, const uint8_t* rgray,
                         const int2* lstat, const int2* rstat, wscore_t* win, int* wbase,
                         const int* list, const unsigned* count, const Geom& g, int frames,
                         long stride, long rstat_stride, long win_stride, cudaStream_t s);
void launch_wta_resolve(const uint8_t* lgray, const uint8_t* rgray, const int* flag_list,
                        const unsigned int* flag_count, float* disp, uint8_t* valid,
                        const Geom& g, double min_zncc, int frames, long gray_stride,
                        long map_stride, long flag_stride, unsigned long long* counters,
                        cudaStream_t s);
void launch_wta_generic(const uint8_t* lgray, const uint8_t* rgray, float* disp,
                        uint8_t* valid, const Geom& g, double min_zncc, int frames,
                        long gray_stride, long map_stride, cudaStream_t s);

// Left-right consistency (k_lr.cu): mirrored swapped pair for the right-view
// sweep, the check itself, and mirroring a right-view map back.
void launch_flip_pair(const uint8_t* gl, const uint8_t* gr, uint8_t* out_l, uint8_t* out_r,
                      int W, int H, int frames, long stride, cudaStream_t s);
void launch_lr_check(float* disp, uint8_t* valid, const float* disp_rm, const uint8_t* valid_rm,
                     int W, int H, int max_diff, int frames, long stride, cudaStream_t s);
void launch_unflip_map(const float* dm, const uint8_t* vm, float* d, uint8_t* v, int W, int H,
                       int frames, long stride, cudaStream_t s);

// Feature front end (k_features.cu; features.cpp:86-208).
void upload_feature_pattern(const int* pat4x256, cudaStream_t s);
void launch_fast_score(const uint8_t* g, int* score, int W, int H, int thr, cudaStream_t s);
void launch_corner_keys(const int* score, int W, int H, unsigned long long* keys,
                        unsigned* count, cudaStream_t s);
cudaError_t sort_corner_keys(void* tmp, size_t* tmp_bytes, const unsigned long long* keys,
                             unsigned long long* keys_out, int n, cudaStream_t s);
void launch_keys_to_corners(const unsigned long long* keys, int n, int* cu, int* cv, int* cs,
                            cudaStream_t s);
void launch_describe(const uint8_t* g, int W, int H, const int* cu, const int* cv, int n,
                     unsigned long long* desc_tmp, int* keep, double* pos,
                     unsigned long long* desc, int* n_out, cudaStream_t s);
void launch_match(const unsigned long long* da, const double* pa, int na,
                  const unsigned long long* db, const double* pb, int nb, int max_hamming,
                  int* best_b, int* best_b_d, int* best_a, int* best_a_d, int* keep, int* ia,
                  int* ib, int* ham, double* disp, int* n_out, cudaStream_t s);

// Fusion consumer (k_fusion.cu).
void launch_rasterize(const double* pos, int n, const double* pose12, double fx, double fy,
                      double cx, double cy, int w, int h, unsigned long long* zbits, int* ids,
                      cudaStream_t s);
void launch_raster_out(const unsigned long long* zbits, const int* ids, int* out_ids,
                       double* out_depth, long npx, cudaStream_t s);
void launch_fuse(double* pos, double* nrm, double* col, double* w, double* cw, const int* index,
                 const double* pd, const double* nd, const float* pf, const float* nf,
                 const uint8_t* colors, const double* pose12, double fx, double fy, double cx,
                 double cy, int W, int H, const unsigned long long* zbits, const int* ids,
                 double trunc, double cap, double gate, double omega_min, uint8_t* is_new,
                 int* block_new, int* total, int n0, cudaStream_t s);

// emap: scratch of edge_map_words(W, H) * frames words: the outlier pass's
// validity and smooth-edge bitmaps (five row-major planes of ceil(W/32) words
// per row), its result (a sixth row-major plane) and that result by columns
// and by both diagonals (lines of ceil(H/32) words) for the radial fill
inline long edge_map_words(int W, int H) {
  const long ww = (W + 31) / 32, hw = (H + 31) / 32;
  return 6L * H * ww + (long)W * hw + 2L * (W + H - 1) * hw;
}
// dout2/vout2/list/count (optional, nullptr = off): a second copy of the
// result and the per-frame list of invalid output pixels (the chain's radial
// fill then touches only those).
void launch_remove_outliers(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                            int W, int H, int radius, double thr, uint32_t* emap, int frames,
                            long stride, cudaStream_t s, float* dout2 = nullptr,
                            uint8_t* vout2 = nullptr, int* list = nullptr,
                            unsigned* count = nullptr);
// dout/vout must already hold din/vin; fills the listed pixels only. emap:
// the maps launch_remove_outliers left (its result is vin), searched by bits.
void launch_fill_radial_list(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                             int W, int H, int radius, int min_support, const int* list,
                             const unsigned* count, const uint32_t* emap, int frames, long stride,
                             cudaStream_t s);
void launch_fill_radial(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                        int W, int H, int radius, int min_support, int frames, long stride,
                        cudaStream_t s);
// pcnt: scratch [frames][H][W+1] ints; list: scratch [frames][W*H]; count: [frames];
// fx: scratch [frames][W*H] doubles; wtab: [(2R+1)^2] disc weights (dv-major);
// ctr[4] += disc-filled pixels
void launch_fill_disc(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                      int W, int H, int radius, int min_support, const double* wtab,
                      const int* span, int* pcnt, int* list, unsigned* count, double* fx,
                      unsigned long long* ctr, int frames, long stride, cudaStream_t s);

struct RefineArgs {
  Geom g;
  double alpha, one_minus_alpha, eta, lo, hi;
  float eta_f;
  float inv2eta_f;  // 1 / (2 eta) (+-inf for eta == 0): the certificate slopes
  int radius;       // smoothing_radius
  const int* span;  // [radius + 1]
};
// normal-layout per-row prefix counts (cleanup disc support)
void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s);

// ---- BT layout (row-blocked transposed): element (v, c) at
// ((v/32) * CW + c) * 32 + v%32; frame stride ceil(H/32) * CW * 32. Every
// refinement field is BT with CW = W (pixel fields, incl. the score windows
// and wbase) or CW = W + 1 (row prefixes). A warp owns 32 consecutive rows of
// one column: its loads and stores are single 128/256-byte lines. ----
// Warp-aggregated list append: the lanes with `pred` write `val` to
// consecutive slots of list[] reserved by ONE atomic per (converged part of a)
// warp, instead of one atomic per lane on the same counter.
__device__ __forceinline__ void warp_append(int* list, unsigned* count, bool pred, int val) {
  const unsigned active = __activemask();
  const unsigned m = __ballot_sync(active, pred);
  if (!m) return;
  unsigned lane;
  asm("mov.u32 %0, %%laneid;" : "=r"(lane));
  const int leader = __ffs(m) - 1;
  unsigned base = 0;
  if ((int)lane == leader) base = atomicAdd(count, (unsigned)__popc(m));
  base = __shfl_sync(active, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

__host__ __device__ inline long bt_frame(int W, int H, int extra_col) {
  return (long)((H + 31) / 32) * (W + extra_col) * 32;
}
__host__ __device__ inline long bt_index(int W, int v, int u) {
  return ((long)(v >> 5) * W + u) * 32 + (v & 31);
}
// Score windows: kWin/2 u32 words (2 fp16 scores each) per pixel, stored as
// BT word planes — word j of pixel (v, u) at ((v/32 * 8 + j) * W + u) * 32 +
// v%32; frame stride 8 * bt_frame(W, H, 0) words — so a tile's plane j is one
// contiguous range (a single bulk copy) and a warp reads it conflict-free.
__host__ __device__ inline long win_word(int W, int v, int u, int j) {
  return (((long)(v >> 5) * (kWin / 2) + j) * W + u) * 32 + (v & 31);
}
__host__ __device__ inline void bt_decode(int W, long idx, int& v, int& u) {
  const long q = idx >> 5;
  u = (int)(q % W);
  v = (int)(q / W) * 32 + (int)(idx & 31);
}
// normal (disp, valid) -> BT mask m, o = d = valid ? disp : 0 (double).
// wbase != NULL: also the post-cleanup window check — a valid pixel whose
// sweep window (wbase, BT) is not centred on its disparity is queued on
// list / count (per frame, stride `stride`); kNoWin where no window fits or
// var_l == 0 (lstat).
void launch_refine_init(const float* disp, const uint8_t* valid, uint8_t* mT, double* oT,
                        double* dT, int W, int H, int frames, long stride, long bs,
                        const int2* lstat, int* wbase, int* list, unsigned* count, const Geom& g,
                        cudaStream_t s);
// Row prefixes carry `ext` (= the smoothing radius) columns past psum[W]
// that repeat the row total: a disc span clipped at the right edge,
// min(W - 1, u + sx) + 1 = W, reads the same value unclipped at u + sx + 1,
// and columns left of 0 arrive as TMA zero fill = psum[0]. With all-zero
// rows past H (mask 0) and zero-filled rows above 0 (whose +0.0 terms leave
// the reference's double sum unchanged), every pixel takes the unclipped
// compile-time disc gather.
__host__ __device__ inline int psum_cw(int W, int ext) { return W + 1 + ext; }
// masked serial row prefix (psum[.][0] = 0, psum_cw(W, ext) columns, BT
// layout); xT == nullptr for the int scan means x = 1 (disc counts)
void launch_scan_bt_d(const double* xT, const uint8_t* mT, double* pT, int W, int H, int ext,
                      int frames, cudaStream_t s);
void launch_scan_bt_i(const int* xT, const uint8_t* mT, int* pT, int W, int H, int ext, int frames,
                      cudaStream_t s);
// iterations >= 1: b = (S_o / cnt - a o) - (1 - a) d formed inside the scan
void launch_scan_b(const int* soT, const int* cntT, const int* oT, const double* dT,
                   const uint8_t* mT, double alpha, double one_minus_alpha, double* pT, int W,
                   int H, int ext, int frames, cudaStream_t s);
// exact integer disc sums from an int BT prefix (disc counts, S_o)
void launch_disc_isum(const uint8_t* mT, const int* ipsumT, int* outT, const RefineArgs& a,
                      int frames, cudaStream_t s);
// iteration 0: avg = disc mean of o (FP64, reference order), b
void launch_avg_b(const double* psumT, const uint8_t* mT, const int* cntT, const double* oT,
                  const double* dT, double* avgT, double* bT, const RefineArgs& a, int frames,
                  cudaStream_t s);
// avg: the double disc mean of o (iteration 0) or nullptr to use the exact
// integer disc sum `so` (iterations >= 1); o changes are appended to chg.
// Re-picks whose FP32 window filter is ambiguous, or whose candidates leave
// the window, are deferred to launch_repick_exact (warp per pixel, FP64).
struct Deferred {
  int pix, c_lo, mask, pad;  // pix: BT index; mask: candidates c_lo + k to score exactly
  double d;
};
// o: integer disparities (written by every re-pick; read for the change list
// when avg == nullptr, i.e. iterations >= 1). All per-pixel arrays BT.
void launch_d_repick(const double* psumT, const uint8_t* mT, const int* cntT,
                     const double* avgT, const int* soT, double* dT, int* oT,
                     const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                     const int* wbase, int2* chg, unsigned* chg_count, Deferred* defer,
                     unsigned* defer_count, float2* ivT, const RefineArgs& a, int frames,
                     long gray_stride,
                     cudaStream_t s);
void launch_repick_exact(const Deferred* defer, const unsigned* defer_count, int* oT,
                         const uint8_t* lgray, const uint8_t* rgray, int2* chg,
                         unsigned* chg_count, const RefineArgs& a, int frames, long gray_stride,
                         unsigned long long* counters, cudaStream_t s);
// Certified re-pick path (window 11, smoothing radius 15, TMA tile): the
// gather stores d and lists the pixels whose d left their certificate
// interval ivT (float2 BT; iteration 0's k_d_repick stores the first ones);
// the list kernel re-picks them, stores their new intervals and settles
// ambiguous ones exactly inside the block.
bool certified_repick_ok(const RefineArgs& a, bool has_win);
void launch_d_gather(const double* psumT, const uint8_t* mT, const int* cntT, const int* soT,
                     const float2* ivT, double* dT, int* list, unsigned* list_count,
                     const RefineArgs& a, int frames, cudaStream_t s);
void launch_repick_list(const int* list, const unsigned* list_count, const double* dT, int* oT,
                        const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                        const int* wbase, float2* ivT, int2* chg, unsigned* chg_count,
                        const RefineArgs& a, int frames, long gray_stride,
                        unsigned long long* counters, cudaStream_t s);
// S_o += delta over the disc of every changed pixel (exact integers).
void launch_so_update(const int2* chg, const unsigned* chg_count, const uint8_t* mT, int* soT,
                      const RefineArgs& a, int frames, cudaStream_t s);
// BT -> normal: refined disparity (valid ? float(d) : din), trace rows
void launch_refine_out(const double* dT, const uint8_t* valid, const float* din, float* dout,
                       int W, int H, int frames, long stride, cudaStream_t s);
void launch_trace_rows(const int* oT, const double* dT, const uint8_t* valid, double* trace_o,
                       double* trace_d, int W, int H, cudaStream_t s);

struct CloudArgs {
  double fx, fy, cx, cy, baseline;
};
void launch_cloud_index(const float* disp, const uint8_t* valid, int* index, int* block_sums,
                        int* n_points, int W, int H, int frames, long stride, cudaStream_t s);
void launch_cloud_points(const float* disp, const int* index, const uint8_t* rgb, int cw,
                         int ch, int W, int H, const CloudArgs& c, double* pts_d,
                         float* pts_f, float4* pts4, uint8_t* colors, int* pixels, int frames,
                         long stride, long rgb_stride, cudaStream_t s);
// nrm_o (optional): octahedral snorm16 normals (SS_OUT_NORMALS_OCT);
// fitted (optional): per point, 1 = plane fit, 0 = sight-ray fallback
void launch_cloud_normals(const float4* pts4, const float* disp, const int* index,
                          const CloudArgs& c, double* nrm_d, float* nrm_f, short2* nrm_o,
                          uint8_t* fitted, int W, int H, int frames, long stride,
                          cudaStream_t s);

}  // namespace ssb
