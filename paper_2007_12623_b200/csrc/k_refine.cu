// Anti-shrink Laplacian refinement (refine_disparities, smoothing.cpp:68-159).
//
// Iteration 0 (o = the cleanup output, fractional where filled) follows the
// reference literally: FP64 row prefix of o (k_scan.cu), k_avg_b, FP64 row
// prefix of b, k_d_repick. After it, o is integer-valued, so its disc sum is an
// exact integer S_o (and the reference's double sum of it is exact too):
// S_o is built once (int prefix + k_disc_count) and then maintained by
// k_so_update from the few pixels whose o changed (hundreds to thousands per
// frame), and b is formed inside the b prefix scan (SrcB). Iterations >= 1 are
// therefore one serial FP64 scan + one tiled gather + a small scatter.
//   k_avg_b       disc mean of o (31 row-span differences, dy ascending,
//                 smoothing.cpp:43-63) fused with the correction
//                 b = (avg - a o) - (1-a) d_prev (smoothing.cpp:91-99).
//   k_d_repick    disc mean of b, d = clamp(avg - avg(b), lo, hi)
//                 (smoothing.cpp:104-111) fused with the re-pick
//                 (smoothing.cpp:114-146): argmin over integer candidates of
//                 1/max(zncc, 1e-3) + (eta diff) diff, strict < (first min).
//                 Candidate costs come from the WTA cost volume in FP32 with a
//                 rigorous 4e-6 relative margin (error <= 7 ulp = 4.2e-7); when more than one
//                 candidate lies within the margin of the minimum, those
//                 candidates are re-scored in exact FP64 (zncc_exact), so the
//                 pick equals the reference's. Without a volume (window != 11)
//                 every candidate is scored exactly.
// The mask is fixed, so the per-pixel disc count is computed once (k_disc_count).
#include <limits.h>
#include <math.h>

#include <type_traits>
#include <utility>

#include "exact.cuh"
#include "ss_internal.cuh"

namespace ssb {

__global__ void k_refine_init(const float* __restrict__ disp, const uint8_t* __restrict__ valid,
                              double* __restrict__ o, double* __restrict__ d, long n,
                              long stride) {
  const long f = blockIdx.y;
  disp += f * stride;
  valid += f * stride;
  o += f * stride;
  d += f * stride;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const double x = valid[i] ? (double)disp[i] : 0.0;
    o[i] = x;
    d[i] = x;
  }
}

void launch_refine_init(const float* disp, const uint8_t* valid, double* o, double* d,
                        int W, int H, int frames, long stride, cudaStream_t s) {
  const long n = (long)W * H;
  if (n <= 0 || frames <= 0) return;
  long blocks = (n + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  k_refine_init<<<dim3((unsigned)blocks, frames), 256, 0, s>>>(disp, valid, o, d, n, stride);
}

// ---- disc sums of a masked field from its row prefixes (smoothing.cpp:43-63) ----
//
// The reference sums, for dy ascending, the span difference
// psum[row][u1+1] - psum[row][u0] of each disc row. Both gathers run on a
// 32 x 16 pixel tile whose psum rows/columns (plus the radius halo) are staged
// in shared memory once, so the 2 (2R+1) reads per pixel are LDS, not L2
// round trips. Summation order and operands are the reference's: bit-exact.

constexpr int kTX = 32, kTY = 16, kBY = 16;  // tile = block = 32 x 16 pixels

template <typename T>
struct PsumTile {
  const T* t;         // smem [(kTY + 2R)][(kTX + 2R + 1)]
  int pitch, u0, v0;  // psum column of t[.][0] is u0 - R; row of t[0] is v0 - R
};

__host__ __device__ inline int tile_pitch(int R) { return kTX + 2 * R + 1; }
template <typename T>
__host__ __device__ inline size_t tile_bytes(int R) {
  return sizeof(T) * (size_t)(kTY + 2 * R) * tile_pitch(R) + sizeof(int) * (R + 1);
}
// re-pick: the tile, then each thread's 32-byte score window (16-byte aligned)
__host__ __device__ inline size_t repick_smem_bytes(int R) {
  return (tile_bytes<double>(R) + 15) / 16 * 16 + (size_t)kTX * kBY * kWin * sizeof(wscore_t);
}

__device__ __forceinline__ void cp_async_bytes(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Stage the BT-layout prefix rows [v0-R, v0+kTY+R) x columns [u0-R, u0+kTX+R]
// of one frame with cp.async (every copy in flight at once; lanes walk rows,
// contiguous within a BT row block). The caller may issue more copies, then
// calls tile_wait(). RF > 0 makes the tile geometry compile-time.
template <int RF, typename T>
__device__ __forceinline__ PsumTile<T> load_tile_issue(const T* __restrict__ psumT, int W, int H,
                                                       int Rr, const int* __restrict__ span_g,
                                                       int*& span) {
  extern __shared__ double tile_raw[];
  T* tile_mem = reinterpret_cast<T*>(tile_raw);
  const int R = RF > 0 ? RF : Rr;
  const int pitch = tile_pitch(R);
  const int rows = kTY + 2 * R;
  const int u0 = blockIdx.x * kTX, v0 = blockIdx.y * kTY;
  span = reinterpret_cast<int*>(tile_mem + (size_t)rows * pitch);
  const int tid = threadIdx.y * kTX + threadIdx.x;
  for (int k = tid; k <= R; k += kTX * kBY) span[k] = __ldg(span_g + k);
  // Lanes walk rows (contiguous within a BT row block), warps walk columns.
  if constexpr (RF > 0) {
    constexpr int P = kTX + 2 * RF + 1, ROWS = kTY + 2 * RF;
    constexpr int RCH = (ROWS + kTX - 1) / kTX, CCH = (P + kBY - 1) / kBY;
#pragma unroll
    for (int rc = 0; rc < RCH; ++rc) {
      const int r = threadIdx.x + rc * kTX;
      const int pr = v0 - RF + r;
      const bool row_ok = r < ROWS && pr >= 0 && pr < H;
      const T* src = psumT + ((long)(pr >> 5) * (W + 1)) * 32 + (pr & 31);
      T* dst = tile_mem + r * P;
#pragma unroll
      for (int cc = 0; cc < CCH; ++cc) {
        const int c = threadIdx.y + cc * kBY;
        const int pc = u0 - RF + c;
        if (r < ROWS && c < P) {
          if (row_ok && pc >= 0 && pc <= W) cp_async_bytes(dst + c, src + pc * 32, sizeof(T));
          else dst[c] = T(0);
        }
      }
    }
  } else {
    for (int r = threadIdx.x; r < rows; r += kTX) {
      const int pr = v0 - R + r;
      const bool row_ok = pr >= 0 && pr < H;
      const T* src = psumT + ((long)(pr >> 5) * (W + 1)) * 32 + (pr & 31);
      T* dst = tile_mem + r * pitch;
      for (int c = threadIdx.y; c < pitch; c += kBY) {
        const int pc = u0 - R + c;
        if (row_ok && pc >= 0 && pc <= W)
          cp_async_bytes(dst + c, src + (long)pc * 32, sizeof(T));
        else
          dst[c] = T(0);
      }
    }
  }
  return PsumTile<T>{tile_mem, pitch, u0, v0};
}

__device__ __forceinline__ void tile_wait() {
  cp_async_wait_all();
  __syncthreads();
}

template <int RF, typename T>
__device__ __forceinline__ PsumTile<T> load_tile(const T* __restrict__ psumT, int W, int H, int Rr,
                                                 const int* __restrict__ span_g, int*& span) {
  const PsumTile<T> P = load_tile_issue<RF>(psumT, W, H, Rr, span_g, span);
  tile_wait();
  return P;
}

template <typename T>
__device__ __forceinline__ T tsub(T a, T b) {
  if constexpr (std::is_same<T, double>::value) return __dsub_rn(a, b);
  else return a - b;
}
template <typename T>
__device__ __forceinline__ T tadd(T a, T b) {
  if constexpr (std::is_same<T, double>::value) return __dadd_rn(a, b);
  else return a + b;
}

template <typename T>
__device__ __forceinline__ T disc_sum_tile(const PsumTile<T>& P, const int* span, int W, int H,
                                           int u, int v, int R) {
  const int lo = max(-R, -v), hi = min(R, H - 1 - v);
  T s = T(0);
  for (int dy = lo; dy <= hi; ++dy) {
    const int sx = span[dy < 0 ? -dy : dy];
    const int c0 = max(0, u - sx) - (P.u0 - R);
    const int c1 = min(W - 1, u + sx) + 1 - (P.u0 - R);
    const T* row = P.t + (v + dy - (P.v0 - R)) * P.pitch;
    s = tadd(s, tsub(row[c1], row[c0]));
  }
  return s;
}

// Compile-time radius: interior pixels (no clamping) read the tile at
// immediate offsets from one base pointer — no index arithmetic per disc row.
__host__ __device__ constexpr int isqrt_floor(int x) {
  int r = 0;
  while ((r + 1) * (r + 1) <= x) ++r;
  return r;
}

template <typename T, int R, int DY>
__device__ __forceinline__ T span_diff(const T* q) {
  constexpr int P = kTX + 2 * R + 1;
  constexpr int SX = isqrt_floor(R * R - DY * DY);
  return tsub(q[DY * P + SX + 1], q[DY * P - SX]);
}

template <typename T, int R, int... I>
__device__ __forceinline__ T disc_sum_fixed(const T* q, std::integer_sequence<int, I...>) {
  T s = T(0);
  ((s = tadd(s, span_diff<T, R, I - R>(q))), ...);  // dy ascending, left to right
  return s;
}

template <int R, typename T>
__device__ __forceinline__ T disc_sum_any(const PsumTile<T>& P, const int* span, int W, int H,
                                          int u, int v, int Rr) {
  if constexpr (R > 0) {
    if (u >= R && u + R <= W - 1 && v >= R && v + R <= H - 1) {
      const T* q = P.t + (v - P.v0 + R) * P.pitch + (u - P.u0 + R);
      return disc_sum_fixed<T, R>(q, std::make_integer_sequence<int, 2 * R + 1>{});
    }
  }
  return disc_sum_tile(P, span, W, H, u, v, Rr);
}

// Exact integer disc sums (disc counts, S_o) from an int BT prefix.
template <int RF>
__global__ void __launch_bounds__(kTX * kBY)
    k_disc_isum(const uint8_t* __restrict__ valid, const int* __restrict__ ipsumT,
                int* __restrict__ out, RefineArgs a, long stride) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  int* span;
  const PsumTile<int> P = load_tile<RF>(ipsumT + f * bt_frame(W, H, 1), W, H, R, a.span, span);
  const int u = blockIdx.x * kTX + threadIdx.x;
#pragma unroll
  for (int rr = 0; rr < kTY / kBY; ++rr) {
    const int v = blockIdx.y * kTY + threadIdx.y + rr * kBY;
    if (u >= W || v >= H) continue;
    const long i = f * stride + (long)v * W + u;
    out[i] = valid[i] ? disc_sum_any<RF>(P, span, W, H, u, v, R) : 0;
  }
}

void launch_disc_isum(const uint8_t* valid, const int* ipsumT, int* out, const RefineArgs& a,
                      int frames, long stride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  const size_t smem = tile_bytes<int>(a.radius);
  dim3 bl(kTX, kBY);
  dim3 grid((a.g.W + kTX - 1) / kTX, (a.g.H + kTY - 1) / kTY, frames);
  if (a.radius == 15) {
    k_disc_isum<15><<<grid, bl, smem, s>>>(valid, ipsumT, out, a, stride);
  } else {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      cudaFuncSetAttribute(k_disc_isum<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      configured = smem;
    }
    k_disc_isum<0><<<grid, bl, smem, s>>>(valid, ipsumT, out, a, stride);
  }
}

template <int RF>
__global__ void __launch_bounds__(kTX * kBY)
    k_avg_b(const double* __restrict__ psumT, const uint8_t* __restrict__ valid,
            const int* __restrict__ cnt, const double* __restrict__ o,
            const double* __restrict__ d, double* __restrict__ avg, double* __restrict__ b,
            RefineArgs a, long stride) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  int* span;
  const PsumTile<double> T = load_tile<RF>(psumT + f * bt_frame(W, H, 1), W, H, R, a.span, span);
  const int u = blockIdx.x * kTX + threadIdx.x;
#pragma unroll
  for (int rr = 0; rr < kTY / kBY; ++rr) {
    const int v = blockIdx.y * kTY + threadIdx.y + rr * kBY;
    if (u >= W || v >= H) continue;
    const long i = f * stride + (long)v * W + u;
    if (!valid[i]) continue;
    const double s = disc_sum_any<RF>(T, span, W, H, u, v, R);
    const double av = __ddiv_rn(s, (double)cnt[i]);
    avg[i] = av;
    // averaged - alpha * discrete - (1 - alpha) * smooth, left to right.
    b[i] = __dsub_rn(__dsub_rn(av, __dmul_rn(a.alpha, o[i])), __dmul_rn(a.one_minus_alpha, d[i]));
  }
}

void launch_avg_b(const double* psumT, const uint8_t* valid, const int* cnt, const double* o,
                  const double* d, double* avg, double* b, const RefineArgs& a, int frames,
                  long stride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  const size_t smem = tile_bytes<double>(a.radius);
  dim3 bl(kTX, kBY);
  dim3 grid((a.g.W + kTX - 1) / kTX, (a.g.H + kTY - 1) / kTY, frames);
  if (a.radius == 15) {
    k_avg_b<15><<<grid, bl, smem, s>>>(psumT, valid, cnt, o, d, avg, b, a, stride);
  } else {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      cudaFuncSetAttribute(k_avg_b<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured = smem;
    }
    k_avg_b<0><<<grid, bl, smem, s>>>(psumT, valid, cnt, o, d, avg, b, a, stride);
  }
}

__device__ __forceinline__ double exact_cost(const uint8_t* L, const uint8_t* R, int W,
                                             int u, int v, int c, bool fits, int half,
                                             double dval, double eta) {
  double match = __ddiv_rn(1.0, kZnccEps);
  const int ru = u - c;
  if (fits && ru >= half && ru < W - half) {
    const ExactScore es = zncc_exact(L, R, W, u, v, ru, half, false);
    if (es.defined) match = __ddiv_rn(1.0, es.score < kZnccEps ? kZnccEps : es.score);
  }
  const double diff = __dsub_rn((double)c, dval);
  return __dadd_rn(match, __dmul_rn(__dmul_rn(eta, diff), diff));
}

constexpr int kMaxCand = 2 * kRefineR + 1;

// FP64 version for the rare paths: exact E (reference expression) and exact M
// when the score is undefined/clamped; err is the FP16-derived M uncertainty.
__device__ __forceinline__ void repick_cost_d(const RefineArgs& a, int u, int c, double dv,
                                              const wscore_t* wp, int W, int half, double& cost,
                                              double& err) {
  constexpr double kErrM = 6e-4;
  double m = 1000.0;
  err = 0.0;
  const int ru = u - c;
  if (ru >= half && ru < W - half) {
    const float sc = __half2float(wp[c]);
    if (!isnan(sc) && sc >= 0.99e-3f) {
      const float mf = 1.f / fmaxf(sc, 1e-3f);
      m = (double)mf;
      err = kErrM * mf;
    }
  }
  const double diff = __dsub_rn((double)c, dv);
  cost = __dadd_rn(m, __dmul_rn(__dmul_rn(a.eta, diff), diff));
}

__device__ __forceinline__ int defer_pixel(Deferred* defer, unsigned* defer_count, long pix,
                                           int c_lo, int mask, double dv) {
  Deferred* e = defer + atomicAdd(defer_count, 1u);
  int2* ei = reinterpret_cast<int2*>(e);  // Deferred is 8-byte aligned
  ei[0] = make_int2((int)pix, c_lo);
  ei[1] = make_int2(mask, 0);
  e->d = dv;
  return INT_MIN;
}

// Re-pick of one pixel (smoothing.cpp:119-144) given its smoothed d.
// Returns the new o, or INT_MIN when the pixel is deferred to the exact kernel.
//
// Filter error budget: window scores are fp16 copies of
// the FP32 sweep score s_f (|s_f - s| <= 5 ulp_f32), so |s16 - s| <= 2^-11 |s|
// + 3e-8; M = 1/max(s, 1e-3) then carries <= 5.3e-4 relative error and the
// float cost M + (eta diff) diff <= 5.4e-4. Candidates within 2.5e-3 of the
// float minimum are re-scored exactly; a single survivor is provably the
// reference's argmin.
__device__ __forceinline__ int repick(const RefineArgs& a, int u, int v, double dv,
                                      const uint8_t* L, const uint8_t* R,
                                      const wscore_t* win_row, int wb, long pix,
                                      Deferred* defer, unsigned* defer_count) {
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const int c_lo = max((int)ceil(__dsub_rn(dv, (double)kRefineR)), (int)ceil(a.lo));
  const int c_hi = min((int)floor(__dadd_rn(dv, (double)kRefineR)), (int)floor(a.hi));
  if (c_lo > c_hi) return INT_MIN;  // unreachable for a clamped d; mirrors `found`
  const bool fits = u >= half && u < W - half && v >= half && v < H - half;

  if (win_row == nullptr) {
    // Generic window size: every candidate in exact FP64 (no score windows).
    double best_cost = 0.0;
    int best = c_lo;
    for (int c = c_lo; c <= c_hi; ++c) {
      const double cost = exact_cost(L, R, W, u, v, c, fits, half, dv, a.eta);
      if (c == c_lo || cost < best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    return best;
  }
  if (!fits || wb == kNoWin) {
    // Window does not fit or var_l == 0: every match cost is exactly
    // 1/kZnccCostEpsilon, so the reference's double costs are computed as is.
    const double m = __ddiv_rn(1.0, kZnccEps);
    double best_cost = 0.0;
    int best = c_lo;
    for (int c = c_lo; c <= c_hi; ++c) {
      const double diff = __dsub_rn((double)c, dv);
      const double cost = __dadd_rn(m, __dmul_rn(__dmul_rn(a.eta, diff), diff));
      if (c == c_lo || cost < best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    return best;
  }
  int best = c_lo;
  if (c_lo >= wb && c_hi <= wb + kWin - 1) {
    // Common path, FP32. cost_f(c) = M_f + E_f with |cost_f - cost| <=
    // eps cost + errE, eps = 6e-4 (fp16 score -> M) + 1.2e-7 (FP32 sum),
    // errE from the FP32 copy of d. The first minimum is certified when the
    // runner-up's lower bound stays above the minimum's upper bound.
    const wscore_t* wp = win_row - wb;  // wp[c]: score of candidate c
    const float dv_f = (float)dv;
    const float delta = fabsf(dv_f) * 1.2e-7f;  // |dv_f - d|, and FP32 rounding of c - dv_f
    constexpr float kEps = 6e-4f + 1.2e-7f;
    // (with eta < 0, E < 0 and the M error, relative to M, is bounded via |E| <= 25|eta|)
    const float errE = fabsf(a.eta_f) * (11.f * delta + 25.f * 4e-7f + (a.eta_f < 0.f ? 25.f * kEps : 0.f));
    float best_cost = INFINITY, second = INFINITY;
    float cf = (float)c_lo;
#pragma unroll
    for (int k = 0; k < kMaxCand; ++k) {
      if (c_lo + k <= c_hi) {
        const float sc = __half2float(wp[c_lo + k]);  // NaN: undefined (incl. ru outside)
        const bool appr = sc >= 0.99e-3f;             // below: certainly clamped to 1000
        const float m = appr ? __fdividef(1.f, fmaxf(sc, 1e-3f)) : 1000.f;
        const float df = cf - dv_f;
        const float cost = m + a.eta_f * df * df;
        second = fminf(second, fmaxf(best_cost, cost));
        if (cost < best_cost) {
          best_cost = cost;
          best = c_lo + k;
        }
      }
      cf += 1.f;
    }
    if (second * (1.f - kEps) - errE > best_cost * (1.f + kEps) + errE) return best;
    // Ambiguous: FP64 costs (exact E, exact clamped/undefined M) with error
    // bars on the fp16-derived M only.
    double bc = INFINITY, up = INFINITY;
    for (int c = c_lo; c <= c_hi; ++c) {
      double cost, err;
      repick_cost_d(a, u, c, dv, wp, W, half, cost, err);
      if (cost < bc) {
        bc = cost;
        best = c;
      }
      up = fmin(up, cost + err);
    }
    int mask = 0, approx = 0;
    for (int c = c_lo; c <= c_hi; ++c) {
      double cost, err;
      repick_cost_d(a, u, c, dv, wp, W, half, cost, err);
      if (cost - err <= up) {
        mask |= 1 << (c - c_lo);
        if (err != 0.0) approx |= 1 << (c - c_lo);
      }
    }
    // A single survivor, or survivors whose costs are all reference-exact
    // doubles (first minimum already taken), is the reference's pick.
    if (__popc(mask) == 1 || approx == 0) return best;
    return defer_pixel(defer, defer_count, pix, c_lo, mask, dv);
  }
  // Window miss: score every candidate exactly.
  return defer_pixel(defer, defer_count, pix, c_lo, (1 << (c_hi - c_lo + 1)) - 1, dv);
}

template <int RF, bool USE_SO>
__global__ void __launch_bounds__(kTX * kBY)
    k_d_repick(const double* __restrict__ psumT, const uint8_t* __restrict__ valid,
               const int* __restrict__ cnt, const double* __restrict__ avg,
               const int* __restrict__ so, double* __restrict__ d, int* __restrict__ o,
               const uint8_t* __restrict__ lgray, const uint8_t* __restrict__ rgray,
               const wscore_t* __restrict__ win, const int* __restrict__ wbase,
               int2* __restrict__ chg, unsigned* __restrict__ chg_count,
               Deferred* __restrict__ defer, unsigned* __restrict__ defer_count, RefineArgs a,
               long stride, long gray_stride) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  const int u = blockIdx.x * kTX + threadIdx.x;
  const int v = blockIdx.y * kTY + threadIdx.y;
  const long pix = (long)v * W + u;
  const long i = f * stride + pix;
  const bool inside = u < W && v < H;
  // 1. issue every global->shared copy (prefix tile + this pixel's window)
  int* span;
  const PsumTile<double> T =
      load_tile_issue<RF>(psumT + f * bt_frame(W, H, 1), W, H, R, a.span, span);
  extern __shared__ double tile_raw[];
  wscore_t* swin = reinterpret_cast<wscore_t*>(reinterpret_cast<unsigned char*>(tile_raw) +
                                               (tile_bytes<double>(R) + 15) / 16 * 16) +
                   (threadIdx.y * kTX + threadIdx.x) * kWin;
  if (win && inside) {
    cp_async_bytes(swin, win + i * kWin, 16);
    cp_async_bytes(swin + 8, win + i * kWin + 8, 16);
  }
  // 2. per-pixel scalars while the copies fly
  const bool act = inside && valid[i];
  int cn = 1, sv = 0, ol = 0, wb = kNoWin;
  double av = 0.0;
  if (act) {
    cn = __ldg(cnt + i);
    if (USE_SO) {
      sv = __ldg(so + i);
      ol = o[i];
    } else {
      av = __ldg(avg + i);
    }
    if (win) wb = __ldg(wbase + i);
  }
  tile_wait();
  if (!act) return;
  const double s = disc_sum_any<RF>(T, span, W, H, u, v, R);
  const double c = (double)cn;
  const double bav = __ddiv_rn(s, c);
  // avg = s_o / c: with integer o the reference's double disc sum is exact,
  // so the integer sum reproduces it bit for bit.
  const double a_o = USE_SO ? __ddiv_rn((double)sv, c) : av;
  const double x = __dsub_rn(a_o, bav);
  const double dv = x < a.lo ? a.lo : (a.hi < x ? a.hi : x);  // std::clamp
  d[i] = dv;
  const int best = repick(a, u, v, dv, lgray + f * gray_stride, rgray + f * gray_stride,
                          win ? swin : nullptr, wb, pix, defer + f * stride, defer_count + f);
  if (best != INT_MIN) {
    if (USE_SO && best != ol)
      chg[f * stride + atomicAdd(chg_count + f, 1u)] = make_int2((int)pix, best - ol);
    o[i] = best;
  }
}

void launch_d_repick(const double* psumT, const uint8_t* valid, const int* cnt,
                     const double* avg, const int* so, double* d, int* o,
                     const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                     const int* wbase, int2* chg, unsigned* chg_count, Deferred* defer,
                     unsigned* defer_count, const RefineArgs& a, int frames, long stride,
                     long gray_stride, unsigned long long* counters, cudaStream_t s) {
  (void)counters;
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  const size_t smem = repick_smem_bytes(a.radius);
  dim3 bl(kTX, kBY);
  dim3 grid((a.g.W + kTX - 1) / kTX, (a.g.H + kTY - 1) / kTY, frames);
#define SS_REPICK_ARGS                                                                        \
  psumT, valid, cnt, avg, so, d, o, lgray, rgray, win, wbase, chg, chg_count, defer,          \
      defer_count, a, stride, gray_stride
  if (a.radius == 15) {
    if (avg) k_d_repick<15, false><<<grid, bl, smem, s>>>(SS_REPICK_ARGS);
    else k_d_repick<15, true><<<grid, bl, smem, s>>>(SS_REPICK_ARGS);
  } else {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      cudaFuncSetAttribute(k_d_repick<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      cudaFuncSetAttribute(k_d_repick<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      configured = smem;
    }
    if (avg) k_d_repick<0, false><<<grid, bl, smem, s>>>(SS_REPICK_ARGS);
    else k_d_repick<0, true><<<grid, bl, smem, s>>>(SS_REPICK_ARGS);
  }
#undef SS_REPICK_ARGS
}

// Deferred re-picks: one warp per pixel, lane k scores candidate c_lo + k in
// exact FP64 (zncc_exact, reference cost formula); the warp takes the first
// minimum (smallest candidate among equal costs), as smoothing.cpp:138 does.
__global__ void k_repick_exact(const Deferred* __restrict__ defer,
                               const unsigned* __restrict__ defer_count, int* __restrict__ o,
                               const uint8_t* __restrict__ lgray,
                               const uint8_t* __restrict__ rgray, int2* __restrict__ chg,
                               unsigned* __restrict__ chg_count, RefineArgs a, long stride,
                               long gray_stride, unsigned long long* __restrict__ counters) {
  const long f = blockIdx.y;
  const unsigned n = defer_count[f];
  if (blockIdx.x == 0 && threadIdx.x == 0 && counters) atomicAdd(counters, (unsigned long long)n);
  const int lane = threadIdx.x & 31;
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const uint8_t* L = lgray + f * gray_stride;
  const uint8_t* R = rgray + f * gray_stride;
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  for (unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nwarps) {
    const Deferred e = defer[f * stride + t];
    const int u = e.pix % W, v = e.pix / W;
    const bool fits = u >= half && u < W - half && v >= half && v < H - half;
    const bool mine = lane < kMaxCand && ((e.mask >> lane) & 1);
    double cost = INFINITY;
    if (mine) cost = exact_cost(L, R, W, u, v, e.c_lo + lane, fits, half, e.d, a.eta);
    int k = mine ? lane : 64;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oc = __shfl_down_sync(0xffffffffu, cost, off);
      const int ok = __shfl_down_sync(0xffffffffu, k, off);
      if (oc < cost || (oc == cost && ok < k)) {
        cost = oc;
        k = ok;
      }
    }
    if (lane == 0 && k < 64) {
      const int best = e.c_lo + k;
      const long i = f * stride + e.pix;
      if (chg) {
        const int old = o[i];
        if (best != old) chg[f * stride + atomicAdd(chg_count + f, 1u)] = make_int2(e.pix, best - old);
      }
      o[i] = best;
    }
  }
}

void launch_repick_exact(const Deferred* defer, const unsigned* defer_count, int* o,
                         const uint8_t* lgray, const uint8_t* rgray, int2* chg,
                         unsigned* chg_count, const RefineArgs& a, int frames, long stride,
                         long gray_stride, unsigned long long* counters, cudaStream_t s) {
  if (frames <= 0) return;
  k_repick_exact<<<dim3(64, frames), 256, 0, s>>>(defer, defer_count, o, lgray, rgray, chg,
                                                  chg_count, a, stride, gray_stride, counters);
}

__global__ void k_int_to_double(const int* __restrict__ x, const uint8_t* __restrict__ valid,
                                double* __restrict__ y, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    if (valid[i]) y[i] = (double)x[i];
}

void launch_int_to_double(const int* x, const uint8_t* valid, double* y, long n,
                          cudaStream_t s) {
  if (n <= 0) return;
  long blocks = (n + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  k_int_to_double<<<(unsigned)blocks, 256, 0, s>>>(x, valid, y, n);
}

// One warp per changed pixel j: S_o(i) += delta_j for every valid i whose disc
// contains j (the disc relation is symmetric, clipped to the image exactly as
// the reference's row spans are).
__global__ void k_so_update(const int2* __restrict__ chg, const unsigned* __restrict__ chg_count,
                            const uint8_t* __restrict__ valid, int* __restrict__ so,
                            RefineArgs a, long stride) {
  const long f = blockIdx.y;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  const unsigned n = chg_count[f];
  const int lane = threadIdx.x & 31;
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  for (unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nwarps) {
    const int2 e = chg[f * stride + t];
    const int v = e.x / W, u = e.x % W;
    for (int dy = max(-R, -v); dy <= min(R, H - 1 - v); ++dy) {
      const int sx = __ldg(a.span + (dy < 0 ? -dy : dy));
      const int u0 = max(0, u - sx), u1 = min(W - 1, u + sx);
      const long row = f * stride + (long)(v + dy) * W;
      for (int x = u0 + lane; x <= u1; x += 32)
        if (__ldg(valid + row + x)) atomicAdd(so + row + x, e.y);
    }
  }
}

void launch_so_update(const int2* chg, const unsigned* chg_count, const uint8_t* valid,
                      int* so, const RefineArgs& a, int frames, long stride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  k_so_update<<<dim3(148, frames), 256, 0, s>>>(chg, chg_count, valid, so, a, stride);
}

__global__ void k_refine_out(const double* __restrict__ d, const uint8_t* __restrict__ valid,
                             const float* __restrict__ din, float* __restrict__ dout, long n,
                             long stride) {
  const long f = blockIdx.y;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const long k = f * stride + i;
    dout[k] = valid[k] ? (float)d[k] : din[k];
  }
}

void launch_refine_out(const double* d, const uint8_t* valid, const float* din, float* dout,
                       int W, int H, int frames, long stride, cudaStream_t s) {
  const long n = (long)W * H;
  if (n <= 0 || frames <= 0) return;
  long blocks = (n + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  k_refine_out<<<dim3((unsigned)blocks, frames), 256, 0, s>>>(d, valid, din, dout, n, stride);
}

}  // namespace ssb
