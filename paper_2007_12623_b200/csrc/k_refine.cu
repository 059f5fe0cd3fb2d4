// Anti-shrink Laplacian refinement (refine_disparities, smoothing.cpp:68-159).
//
// One iteration = 2 scans + 2 gathers, all FP64 in the reference's order:
//   k_row_scan    serial left-to-right masked row prefix (smoothing.cpp:25-41);
//                 one thread per (frame, row) — latency-bound, hidden by the
//                 frame batch.
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
#include <math.h>

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

__global__ void k_row_count(const uint8_t* __restrict__ valid, int* __restrict__ pcnt, int W,
                            int H, long stride, long pstride) {
  const long f = blockIdx.y;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= H) return;
  const uint8_t* m = valid + f * stride + (long)v * W;
  int* p = pcnt + f * pstride + (long)v * (W + 1);
  int c = 0;
  p[0] = 0;
  for (int u = 0; u < W; ++u) {
    c += m[u] ? 1 : 0;
    p[u + 1] = c;
  }
}

void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_row_count<<<dim3((H + 63) / 64, frames), 64, 0, s>>>(valid, pcnt, W, H, stride, pstride);
}

__global__ void k_disc_count(const uint8_t* __restrict__ valid, const int* __restrict__ pcnt,
                             int* __restrict__ cnt, RefineArgs a, long stride, long pstride) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = (long)v * W + u;
  valid += f * stride;
  pcnt += f * pstride;
  if (!valid[i]) {
    cnt[f * stride + i] = 0;
    return;
  }
  const int r = a.radius;
  const int lo = max(-r, -v), hi = min(r, H - 1 - v);
  int c = 0;
  for (int dy = lo; dy <= hi; ++dy) {
    const int sx = a.span[dy < 0 ? -dy : dy];
    const int u0 = max(0, u - sx), u1 = min(W - 1, u + sx);
    const int* row = pcnt + (long)(v + dy) * (W + 1);
    c += row[u1 + 1] - row[u0];
  }
  cnt[f * stride + i] = c;
}

void launch_disc_count(const uint8_t* valid, const int* pcnt, int* cnt, const RefineArgs& a,
                       int frames, long stride, long pstride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  dim3 grid((a.g.W + 31) / 32, (a.g.H + 7) / 8, frames);
  k_disc_count<<<grid, b, 0, s>>>(valid, pcnt, cnt, a, stride, pstride);
}

// Serial masked row prefix in double: the reference's exact summation order.
__global__ void k_row_scan(const double* __restrict__ val, const uint8_t* __restrict__ valid,
                           double* __restrict__ psum, int W, int H, long stride, long pstride) {
  const long f = blockIdx.y;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= H) return;
  const double* x = val + f * stride + (long)v * W;
  const uint8_t* m = valid + f * stride + (long)v * W;
  double* p = psum + f * pstride + (long)v * (W + 1);
  double s = 0.0;
  p[0] = 0.0;
  for (int u = 0; u < W; ++u) {
    if (m[u]) s = __dadd_rn(s, x[u]);
    p[u + 1] = s;
  }
}

void launch_row_scan(const double* val, const uint8_t* valid, double* psum, int W, int H,
                     int frames, long stride, long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_row_scan<<<dim3((H + 31) / 32, frames), 32, 0, s>>>(val, valid, psum, W, H, stride,
                                                        pstride);
}

// Disc sum of a masked field from its row prefixes, dy ascending.
__device__ __forceinline__ double disc_sum(const double* __restrict__ psum, int W, int H,
                                           int u, int v, int r, const int* __restrict__ span) {
  const int lo = max(-r, -v), hi = min(r, H - 1 - v);
  double s = 0.0;
  for (int dy = lo; dy <= hi; ++dy) {
    const int sx = __ldg(span + (dy < 0 ? -dy : dy));
    const int u0 = max(0, u - sx), u1 = min(W - 1, u + sx);
    const double* row = psum + (long)(v + dy) * (W + 1);
    s = __dadd_rn(s, __dsub_rn(__ldg(row + u1 + 1), __ldg(row + u0)));
  }
  return s;
}

__global__ void k_avg_b(const double* __restrict__ psum, const uint8_t* __restrict__ valid,
                        const int* __restrict__ cnt, const double* __restrict__ o,
                        const double* __restrict__ d, double* __restrict__ avg,
                        double* __restrict__ b, RefineArgs a, long stride, long pstride) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = f * stride + (long)v * W + u;
  if (!valid[i]) return;
  const double s = disc_sum(psum + f * pstride, W, H, u, v, a.radius, a.span);
  const double av = __ddiv_rn(s, (double)cnt[i]);
  avg[i] = av;
  // averaged - alpha * discrete - (1 - alpha) * smooth, left to right.
  b[i] = __dsub_rn(__dsub_rn(av, __dmul_rn(a.alpha, o[i])), __dmul_rn(a.one_minus_alpha, d[i]));
}

void launch_avg_b(const double* psum, const uint8_t* valid, const int* cnt, const double* o,
                  const double* d, double* avg, double* b, const RefineArgs& a, int frames,
                  long stride, long pstride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  dim3 bl(32, 8);
  dim3 grid((a.g.W + 31) / 32, (a.g.H + 7) / 8, frames);
  k_avg_b<<<grid, bl, 0, s>>>(psum, valid, cnt, o, d, avg, b, a, stride, pstride);
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

__global__ void k_d_repick(const double* __restrict__ psum, const uint8_t* __restrict__ valid,
                           const int* __restrict__ cnt, const double* __restrict__ avg,
                           double* __restrict__ d, double* __restrict__ o,
                           const uint8_t* __restrict__ lgray, const uint8_t* __restrict__ rgray,
                           const int2* __restrict__ lstat, const float* __restrict__ vol,
                           RefineArgs a, long stride, long pstride, long gray_stride,
                           long lstat_stride, long vol_stride,
                           unsigned long long* __restrict__ counters) {
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long pix = (long)v * W + u;
  const long i = f * stride + pix;
  if (!valid[i]) return;
  const double s = disc_sum(psum + f * pstride, W, H, u, v, a.radius, a.span);
  const double bav = __ddiv_rn(s, (double)cnt[i]);
  const double x = __dsub_rn(avg[i], bav);
  const double dv = x < a.lo ? a.lo : (a.hi < x ? a.hi : x);  // std::clamp
  d[i] = dv;

  const uint8_t* L = lgray + f * gray_stride;
  const uint8_t* R = rgray + f * gray_stride;
  const int c_lo = max((int)ceil(__dsub_rn(dv, (double)kRefineR)), (int)ceil(a.lo));
  const int c_hi = min((int)floor(__dadd_rn(dv, (double)kRefineR)), (int)floor(a.hi));
  if (c_lo > c_hi) return;  // unreachable for a clamped d; mirrors `found`
  const bool fits = u >= half && u < W - half && v >= half && v < H - half;

  if (vol == nullptr) {
    // Generic window: every candidate in exact FP64.
    double best_cost = 0.0;
    int best = c_lo;
    for (int c = c_lo; c <= c_hi; ++c) {
      const double cost = exact_cost(L, R, W, u, v, c, fits, half, dv, a.eta);
      if (c == c_lo || cost < best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    o[i] = best;
    const unsigned act = __activemask();
    if ((threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(counters, (unsigned long long)__popc(act));
    return;
  }

  float rl = __int_as_float(0x7fc00000);
  if (fits) rl = __int_as_float(__ldg(&lstat[f * lstat_stride + pix].y));
  if (isnan(rl)) {
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
    o[i] = best;
    return;
  }
  const float* vp = vol + f * vol_stride + pix;
  const long HW = (long)H * W;
  float cf[kMaxCand];
  float best_f = INFINITY;
  int best = c_lo;
#pragma unroll
  for (int k = 0; k < kMaxCand; ++k) {
    const int c = c_lo + k;
    cf[k] = INFINITY;
    if (c <= c_hi) {
      const int ru = u - c;
      float m = 1000.f;  // 1 / kZnccCostEpsilon, exact
      if (fits && ru >= half && ru < W - half) {
        const float sc = __ldg(vp + (long)(c - a.g.cmin) * HW) * rl;
        if (!isnan(sc)) m = 1.f / fmaxf(sc, 1e-3f);
      }
      const float df = (float)__dsub_rn((double)c, dv);
      cf[k] = m + a.eta_f * df * df;
      if (cf[k] < best_f) {
        best_f = cf[k];
        best = c;
      }
    }
  }
  // Any candidate whose exact cost could undercut the float minimum.
  const float thr = best_f * (1.0f + 4e-6f);
  int near = 0;
#pragma unroll
  for (int k = 0; k < kMaxCand; ++k) near += (cf[k] <= thr) ? 1 : 0;
  if (near > 1) {
    double best_cost = 0.0;
    bool found = false;
#pragma unroll 1
    for (int k = 0; k < kMaxCand; ++k) {
      if (!(cf[k] <= thr)) continue;
      const int c = c_lo + k;
      const double cost = exact_cost(L, R, W, u, v, c, fits, half, dv, a.eta);
      if (!found || cost < best_cost) {
        found = true;
        best_cost = cost;
        best = c;
      }
    }
    atomicAdd(counters, 1ull);
  }
  o[i] = best;
}

void launch_d_repick(const double* psum, const uint8_t* valid, const int* cnt,
                     const double* avg, double* d, double* o, const uint8_t* lgray,
                     const uint8_t* rgray, const int2* lstat, const float* vol,
                     const RefineArgs& a, int frames, long stride, long pstride,
                     long gray_stride, long lstat_stride, long vol_stride,
                     unsigned long long* counters, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  dim3 bl(32, 8);
  dim3 grid((a.g.W + 31) / 32, (a.g.H + 7) / 8, frames);
  k_d_repick<<<grid, bl, 0, s>>>(psum, valid, cnt, avg, d, o, lgray, rgray, lstat, vol, a,
                                 stride, pstride, gray_stride, lstat_stride, vol_stride,
                                 counters);
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
