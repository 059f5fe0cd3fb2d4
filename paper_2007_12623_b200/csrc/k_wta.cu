// ZNCC cost sweep + winner-take-all (compute_disparity, matcher.cpp:166-211).
//
// k_wta11 — the hot kernel, window 11 (the default and the paper's setting).
//   Block = 32 lanes (consecutive columns u) x NB warps (blocks of kDB = 16
//   consecutive candidates c of the volume range [d_min-5, d_max+5]). Each
//   thread sweeps a strip of rows; for every row y entering or leaving the
//   11-row window it forms the two chessboard half-sums of one image row
//       He(y) = sum_{du even} L(u+du, y) R(u-c+du, y)   (5 taps)
//       Ho(y) = sum_{du odd}  L(u+du, y) R(u-c+du, y)   (6 taps)
//   with 4 dp4a (u8 x u8 -> int32) on 4-byte windows of the parity-split rows,
//   and keeps two running sums per candidate so that the exact integer cross
//   sum slr(u, v, c) costs O(1) per row step instead of 61 MACs:
//       X(v+1) = Y(v) - He(v-5) + Ho(v+6),   Y(v+1) = X(v) + He(v+6) - Ho(v-5)
//   where X(v) = sum_{dv even} He(v+dv) + sum_{dv odd} Ho(v+dv) = slr(v).
//   num = 61 slr - sl sr is exact; g = float(num) / sqrt(var_r) (FP32, <= 3 ulp)
//   feeds a per-thread (best, second, arg) that NB warps merge through shared
//   memory, and is staged there so that, once a pixel's pick is known, the
//   kWin = 16 candidates around it are written as the refinement's score
//   window (64 B/pixel instead of a (D+10) x 4 B cost volume).
//   A pick is final only when it is separated from the runner-up and from the
//   min_zncc threshold by a margin far above the FP32 error (4e-6 relative);
//   otherwise the pixel is appended to a list for k_wta_exact (FP64, exact),
//   so the output is bit-identical to the reference's double argmax.
// k_wta_exact — one warp per pixel, lanes over d, reference arithmetic
//   (zncc_chessboard int64 statistics, double score, first maximum). Used for
//   the flagged pixels and, over all pixels, for windows other than 11.
#include <limits.h>
#include <math.h>

#include <utility>

#include "exact.cuh"
#include "ss_internal.cuh"

namespace ssb {

namespace {

constexpr int kRB = 4;  // output rows per shared-memory reduction chunk
constexpr int kNoArg = INT_MIN;  // "no defined candidate" (disparities may be negative)

__device__ __forceinline__ uint32_t ld_win(const uint8_t* row, int start) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
  const int wi = start >> 2;
  return __funnelshift_r(__ldg(w + wi), __ldg(w + wi + 1), (start & 3) * 8);
}

template <int O>
__device__ __forceinline__ uint32_t win(const uint32_t (&S)[4]) {
  static_assert(O >= 0 && O <= 12, "window offset");
  if constexpr ((O & 3) == 0) {
    return S[O >> 2];
  } else {
    return __funnelshift_r(S[O >> 2], S[(O >> 2) + 1], 8 * (O & 3));
  }
}

struct ThreadGeom {
  const uint8_t* lplane;
  const uint8_t* rplane;
  long PP;
  int p, q0;            // parity of u, parity of u - c0
  int Le, Lo;           // byte offsets of the left even / odd tap windows
  int wA, shA, wB, shB; // aligned word index + shift of the right streams A, B
};

// The 4-byte windows of one image row that the thread's kDB candidates need:
// the left tap words (fixed per thread) and the two right-image byte streams
// A and B pre-aligned to the thread's misalignment.
struct RowWords {
  uint32_t Lea, Leb, Loa, Lob;
  uint32_t SA[4], SB[4];
};

__device__ __forceinline__ RowWords row_words(const ThreadGeom& tg, int y) {
  RowWords w;
  const uint8_t* lre = tg.lplane + (long)(2 * y + tg.p) * tg.PP;
  const uint8_t* lro = tg.lplane + (long)(2 * y + 1 - tg.p) * tg.PP;
  w.Lea = ld_win(lre, tg.Le);
  w.Leb = ld_win(lre, tg.Le + 4) & 0xFFu;
  w.Loa = ld_win(lro, tg.Lo);
  w.Lob = ld_win(lro, tg.Lo + 4) & 0xFFFFu;
  const uint32_t* ar =
      reinterpret_cast<const uint32_t*>(tg.rplane + (long)(2 * y + tg.q0) * tg.PP) + tg.wA;
  const uint32_t* br =
      reinterpret_cast<const uint32_t*>(tg.rplane + (long)(2 * y + 1 - tg.q0) * tg.PP) + tg.wB;
  uint32_t a[5], b[5];
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    a[t] = __ldg(ar + t);
    b[t] = __ldg(br + t);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    w.SA[t] = __funnelshift_r(a[t], a[t + 1], tg.shA);
    w.SB[t] = __funnelshift_r(b[t], b[t + 1], tg.shB);
  }
  return w;
}

// He (even-offset taps, 5) and Ho (odd-offset taps, 6) of candidate I.
template <int I>
__device__ __forceinline__ uint32_t term_e(const RowWords& w) {
  constexpr int t = I >> 1;
  if constexpr ((I & 1) == 0) return __dp4a(w.Lea, win<8 - t>(w.SA), __dp4a(w.Leb, win<12 - t>(w.SA), 0u));
  else return __dp4a(w.Lea, win<7 - t>(w.SB), __dp4a(w.Leb, win<11 - t>(w.SB), 0u));
}
template <int I>
__device__ __forceinline__ uint32_t term_o(const RowWords& w) {
  constexpr int t = I >> 1;
  if constexpr ((I & 1) == 0) return __dp4a(w.Loa, win<7 - t>(w.SB), __dp4a(w.Lob, win<11 - t>(w.SB), 0u));
  else return __dp4a(w.Loa, win<7 - t>(w.SA), __dp4a(w.Lob, win<11 - t>(w.SA), 0u));
}

// One row step of the running sums for candidate I (center v-1 -> v):
//   X' = Y - He(v-6) + Ho(v+5),  Y' = X + He(v+5) - Ho(v-6)
template <int I>
__device__ __forceinline__ void step_i(const RowWords& wo, const RowWords& wn, int (&X)[kDB],
                                       int (&Y)[kDB]) {
  const int xn = Y[I] - (int)term_e<I>(wo) + (int)term_o<I>(wn);
  const int yn = X[I] + (int)term_e<I>(wn) - (int)term_o<I>(wo);
  X[I] = xn;
  Y[I] = yn;
}
template <int... Is>
__device__ __forceinline__ void step_all(const RowWords& wo, const RowWords& wn, int (&X)[kDB],
                                         int (&Y)[kDB], std::integer_sequence<int, Is...>) {
  (step_i<Is>(wo, wn, X, Y), ...);
}

// Warm-up accumulation of one row: dy even -> X += He, Y += Ho; odd swaps.
template <int I>
__device__ __forceinline__ void warm_i(const RowWords& w, bool even, int (&X)[kDB],
                                       int (&Y)[kDB]) {
  const int he = (int)term_e<I>(w), ho = (int)term_o<I>(w);
  X[I] += even ? he : ho;
  Y[I] += even ? ho : he;
}
template <int... Is>
__device__ __forceinline__ void warm_all(const RowWords& w, bool even, int (&X)[kDB],
                                         int (&Y)[kDB], std::integer_sequence<int, Is...>) {
  (warm_i<Is>(w, even, X, Y), ...);
}

}  // namespace

__global__ void __launch_bounds__(512) k_wta11(
    const uint8_t* __restrict__ lplane, const uint8_t* __restrict__ rplane,
    const int2* __restrict__ lstat, const int2* __restrict__ rstat, wscore_t* __restrict__ win,
    int* __restrict__ wbase, const int* __restrict__ base_map, float* __restrict__ disp,
    uint8_t* __restrict__ valid, int* __restrict__ flag_list,
    unsigned int* __restrict__ flag_count, Geom g, int TH, float min_zncc_f, float thr_tol,
    int do_argmax, long plane_stride, long lstat_stride, long rstat_stride, long map_stride,
    long win_stride) {
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x, j = threadIdx.y, NB = blockDim.y;
  const int NCB = NB * kDB;  // staged candidates per pixel
  float* s_best = reinterpret_cast<float*>(smem_raw);
  float* s_sec = s_best + kRB * NB * 32;
  int* s_arg = reinterpret_cast<int*>(s_sec + kRB * NB * 32);
  float* s_g = reinterpret_cast<float*>(s_arg + kRB * NB * 32);  // [kRB][NCB][32]

  const long fr = blockIdx.z;
  lplane += fr * plane_stride;
  rplane += fr * plane_stride;
  lstat += fr * lstat_stride;
  rstat += fr * rstat_stride;
  win += fr * win_stride * kWin;
  wbase += fr * win_stride;
  if (base_map) base_map += fr * map_stride;
  disp += fr * map_stride;
  valid += fr * map_stride;
  flag_list += fr * map_stride;
  flag_count += fr;

  constexpr int h = 5;
  const int W = g.W, H = g.H;
  const int u = h + blockIdx.x * 32 + lane;
  const int v_begin = h + blockIdx.y * TH;
  const int v_end = min(v_begin + TH, H - h);
  if (v_begin >= v_end) return;  // uniform over the block
  const int c0 = g.cmin + j * kDB;
  const int nact = min(kDB, g.NC - j * kDB);
  const bool active = (u < W - h) && (nact > 0);
  // candidates of this thread that take part in the WTA argmax
  unsigned amask = 0;
#pragma unroll
  for (int i = 0; i < kDB; ++i)
    amask |= (i < nact && c0 + i >= g.dmin && c0 + i <= g.dmax) ? (1u << i) : 0u;

  ThreadGeom tg;
  tg.lplane = lplane;
  tg.rplane = rplane;
  tg.PP = g.PP;
  tg.p = u & 1;
  const int k = u >> 1;
  const int ru0 = u - c0;
  tg.q0 = ru0 & 1;
  const int m0 = ru0 >> 1;  // arithmetic shift: floor for negative ru0
  const int startA = g.PB + m0 - 10;
  const int startB = g.PB + (m0 - 1 + tg.q0) - 9;
  tg.wA = startA >> 2;
  tg.shA = (startA & 3) * 8;
  tg.wB = startB >> 2;
  tg.shB = (startB & 3) * 8;
  tg.Le = g.PB + k - 2;
  tg.Lo = g.PB + k - 3 + tg.p;

  int X[kDB], Y[kDB];
#pragma unroll
  for (int i = 0; i < kDB; ++i) X[i] = Y[i] = 0;

  if (active) {
    for (int dy = -h; dy <= h; ++dy) {
      const RowWords w = row_words(tg, v_begin + dy);
      warm_all(w, ((dy + h) & 1) == 1 /* dy even */, X, Y,
               std::make_integer_sequence<int, kDB>{});
    }
  }

  for (int v = v_begin; v < v_end; ++v) {
    if (v > v_begin && active) {
      const RowWords wo = row_words(tg, v - 6);
      const RowWords wn = row_words(tg, v + 5);
      step_all(wo, wn, X, Y, std::make_integer_sequence<int, kDB>{});
    }
    const int slot = (v - v_begin) & (kRB - 1);
    float* gs = s_g + (slot * NCB + j * kDB) * 32 + lane;  // staged g of this (row, block)
    float best = -INFINITY, second = -INFINITY;
    int arg = kNoArg;
    if (active) {
      const int sl = __ldg(&lstat[(long)v * W + u].x);
      const int2* rrow = rstat + (long)v * g.SP + g.SPAD + ru0;
      // Branch-free: every lane scores all kDB candidates (padded rstat keeps
      // the loads in bounds); amask selects those inside [d_min, d_max] and
      // the volume range, NaN (undefined) folds to -inf.
#pragma unroll
      for (int i = 0; i < kDB; ++i) {
        const int2 rs = __ldg(rrow - i);
        const int num = 61 * X[i] - sl * rs.x;
        const float gv = __int2float_rn(num) * __int_as_float(rs.y);
        gs[i * 32] = gv;
        const float gc = ((amask >> i) & 1) ? fmaxf(gv, -INFINITY) : -INFINITY;
        second = fmaxf(second, fminf(best, gc));
        arg = gc > best ? c0 + i : arg;
        best = fmaxf(best, gc);
      }
    }
    const int so = (slot * NB + j) * 32 + lane;
    s_best[so] = best;
    s_sec[so] = second;
    s_arg[so] = arg;
    if (slot == kRB - 1 || v == v_end - 1) {
      __syncthreads();
      for (int r = j; r <= slot; r += NB) {
        float B = -INFINITY, S = -INFINITY;
        int A = kNoArg;
        for (int jj = 0; jj < NB; ++jj) {
          const int o = (r * NB + jj) * 32 + lane;
          const int a = s_arg[o];
          if (a == kNoArg) continue;
          const float b = s_best[o], s2 = s_sec[o];
          if (b > B) {
            S = fmaxf(B, s2);
            B = b;
            A = a;
          } else {
            S = fmaxf(S, fmaxf(b, s2));
          }
        }
        if (u < W - h) {
          const int vv = v - slot + r;
          const long idx = (long)vv * W + u;
          const float rl = __int_as_float(__ldg(&lstat[idx].y));
          if (do_argmax) {
            float dout = 0.f;
            uint8_t vout = 0;
            if (A != kNoArg && !isnan(rl)) {
              const bool near_tie = S >= B - 4e-6f * fabsf(B);
              const float sc = B * rl;
              const bool amb = fabsf(sc - min_zncc_f) <= thr_tol;
              if (near_tie || amb) {
                flag_list[atomicAdd(flag_count, 1u)] = (int)idx;
              } else if (sc >= min_zncc_f) {
                dout = (float)A;
                vout = 1;
              }
            }
            disp[idx] = dout;
            valid[idx] = vout;
          }
          // Candidate window for the refinement: kWin consecutive scores
          // s = g * rl around the pick (or the caller's base map).
          const int anchor = base_map ? base_map[idx] : A;
          int wb = kNoWin;
          if (!isnan(rl) && anchor != kNoArg && anchor != kNoWin)
            wb = window_base(anchor, g.cmin, g.NC);
          const long bi = bt_index(W, vv, u);
          wbase[bi] = wb;
          if (wb != kNoWin) {
            const float* gr = s_g + r * NCB * 32 + lane;
            uint32_t w[kWin / 2];  // kWin fp16 match costs (m_code)
#pragma unroll
            for (int q = 0; q < kWin / 2; ++q) {
              const int ci = wb - g.cmin + 2 * q;
              const float s0 = ci < g.NC ? gr[ci * 32] * rl : __int_as_float(0x7fc00000);
              const float s1 = ci + 1 < g.NC ? gr[(ci + 1) * 32] * rl : __int_as_float(0x7fc00000);
              w[q] = pack_m2(s0, s1);
            }
            uint32_t* wq = reinterpret_cast<uint32_t*>(win) + win_word(W, vv, u, 0);
#pragma unroll
            for (int q = 0; q < kWin / 2; ++q) wq[(long)q * W * 32] = w[q];
          }
        }
      }
      __syncthreads();
    }
  }
}

void launch_wta11(const uint8_t* lplane, const uint8_t* rplane, const int2* lstat,
                  const int2* rstat, wscore_t* win, int* wbase, const int* base_map, float* disp,
                  uint8_t* valid, int* flag_list, unsigned int* flag_count, const Geom& g,
                  double min_zncc, int frames, long plane_stride, long lstat_stride,
                  long rstat_stride, long map_stride, long win_stride, int do_argmax,
                  cudaStream_t s) {
  const int h = 5;
  if (g.W - 2 * h <= 0 || g.H - 2 * h <= 0 || frames <= 0) return;
  const int NB = (g.NC + kDB - 1) / kDB;
  const int TH = 32;
  dim3 block(32, NB);
  dim3 grid((g.W - 2 * h + 31) / 32, (g.H - 2 * h + TH - 1) / TH, frames);
  const size_t smem = (size_t)kRB * NB * 32 * 12 + (size_t)kRB * NB * kDB * 32 * 4;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(k_wta11, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  const float mz = (float)min_zncc;
  const float tol = 4e-6f * fmaxf(1.f, fabsf(mz));
  k_wta11<<<grid, block, smem, s>>>(lplane, rplane, lstat, rstat, win, wbase, base_map, disp,
                                    valid, flag_list, flag_count, g, TH, mz, tol, do_argmax,
                                    plane_stride, lstat_stride, rstat_stride, map_stride,
                                    win_stride);
}

// ---- exact FP64 path: warp per pixel, lanes over d ----
__global__ void k_wta_exact(const uint8_t* __restrict__ lgray, const uint8_t* __restrict__ rgray,
                            const int* __restrict__ flag_list,
                            const unsigned int* __restrict__ flag_count, float* disp,
                            uint8_t* valid, Geom g, double min_zncc, long gray_stride,
                            long map_stride, long flag_stride, int mode_all,
                            unsigned long long* counters) {
  const long fr = blockIdx.y;
  if (!mode_all && counters && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(counters, (unsigned long long)flag_count[fr]);
  lgray += fr * gray_stride;
  rgray += fr * gray_stride;
  disp += fr * map_stride;
  valid += fr * map_stride;
  const int lane = threadIdx.x & 31;
  const int half = g.half;
  const int iw = g.W - 2 * half, ih = g.H - 2 * half;
  long total;
  if (mode_all) {
    total = (iw > 0 && ih > 0) ? (long)iw * ih : 0;
  } else {
    flag_list += fr * flag_stride;
    total = flag_count[fr];
  }
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  for (long item = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; item < total;
       item += nwarps) {
    int u, v;
    if (mode_all) {
      v = half + (int)(item / iw);
      u = half + (int)(item % iw);
    } else {
      const int idx = flag_list[item];
      v = idx / g.W;
      u = idx % g.W;
    }
    bool found = false;
    double best = 0.0;
    int bestd = 0;
    for (int d = g.dmin + lane; d <= g.dmax; d += 32) {
      const int ru = u - d;
      if (ru < half || ru >= g.W - half) continue;
      const ExactScore es = zncc_exact(lgray, rgray, g.W, u, v, ru, half, true);
      if (!es.defined) continue;
      if (!found || es.score > best) {
        found = true;
        best = es.score;
        bestd = d;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const int of = __shfl_down_sync(0xffffffffu, (int)found, off);
      const double ob = __shfl_down_sync(0xffffffffu, best, off);
      const int od = __shfl_down_sync(0xffffffffu, bestd, off);
      if (of && (!found || ob > best || (ob == best && od < bestd))) {
        found = true;
        best = ob;
        bestd = od;
      }
    }
    if (lane == 0) {
      const long idx = (long)v * g.W + u;
      const bool ok = found && best >= min_zncc;
      disp[idx] = ok ? (float)bestd : 0.f;
      valid[idx] = ok ? 1 : 0;
    }
  }
}

void launch_wta_resolve(const uint8_t* lgray, const uint8_t* rgray, const int* flag_list,
                        const unsigned int* flag_count, float* disp, uint8_t* valid,
                        const Geom& g, double min_zncc, int frames, long gray_stride,
                        long map_stride, long flag_stride, unsigned long long* counters,
                        cudaStream_t s) {
  if (frames <= 0) return;
  k_wta_exact<<<dim3(64, frames), 256, 0, s>>>(lgray, rgray, flag_list, flag_count, disp, valid,
                                               g, min_zncc, gray_stride, map_stride,
                                               flag_stride, 0, counters);
}

void launch_wta_generic(const uint8_t* lgray, const uint8_t* rgray, float* disp,
                        uint8_t* valid, const Geom& g, double min_zncc, int frames,
                        long gray_stride, long map_stride, cudaStream_t s) {
  if (frames <= 0) return;
  k_wta_exact<<<dim3(1184, frames), 256, 0, s>>>(lgray, rgray, nullptr, nullptr, disp, valid,
                                                 g, min_zncc, gray_stride, map_stride, 0, 1,
                                                 nullptr);
}

// ---- candidate windows for pixels the cleanup changed (post-cleanup) ----

// Pass 1: a valid pixel needs a window centred on its (possibly filled)
// disparity o0; if the sweep's window is centred elsewhere (the pixel was
// removed/filled, or its WTA pick was resolved in FP64) queue it.
__global__ void k_window_check(const float* __restrict__ disp, const uint8_t* __restrict__ valid,
                               const int2* __restrict__ lstat, int* __restrict__ wbase,
                               int* __restrict__ list, unsigned* __restrict__ count, Geom g,
                               long stride, long win_stride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= g.W || v >= g.H) return;
  const long pix = (long)v * g.W + u, i = f * stride + pix;
  if (!valid[i]) return;
  const int h = g.half;
  const bool fits = u >= h && u < g.W - h && v >= h && v < g.H - h;
  int* wb = wbase + f * win_stride + bt_index(g.W, v, u);
  if (!fits || isnan(__int_as_float(__ldg(&lstat[i].y)))) {
    *wb = kNoWin;
    return;
  }
  const int want = window_base((int)floor((double)disp[i]), g.cmin, g.NC);
  if (*wb != want) list[f * stride + atomicAdd(count + f, 1u)] = (int)pix;
}

// Pass 2: half a warp per queued pixel, lane q computes candidate wbase + q
// with the sweep's exact integer arithmetic (61-tap chessboard cross sum,
// num = 61 slr - sl sr, g = float(num) / sqrt(var_r), s = g / sqrt(var_l)),
// so the window is bit-identical to one the sweep would have written.
__global__ void k_window_build(const float* __restrict__ disp, const uint8_t* __restrict__ lgray,
                               const uint8_t* __restrict__ rgray, const int2* __restrict__ lstat,
                               const int2* __restrict__ rstat, wscore_t* __restrict__ win,
                               int* __restrict__ wbase, const int* __restrict__ list,
                               const unsigned* __restrict__ count, Geom g, long stride,
                               long rstat_stride, long win_stride) {
  const long f = blockIdx.y;
  const unsigned n = count[f];
  const int q = threadIdx.x & (kWin - 1);
  const unsigned groups = gridDim.x * (blockDim.x / kWin);
  const uint8_t* L = lgray + f * stride;
  const uint8_t* R = rgray + f * stride;
  const int W = g.W, h = g.half;
  for (unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) / kWin; t < n; t += groups) {
    const int pix = list[f * stride + t];
    const int u = pix % W, v = pix / W;
    const long i = f * stride + pix;
    const int wb = window_base((int)floor((double)disp[i]), g.cmin, g.NC);
    const int c = wb + q;
    const int ru = u - c;
    float s = __int_as_float(0x7fc00000);
    if (c < g.cmin + g.NC && ru >= h && ru < W - h) {
      const int2 ls = __ldg(&lstat[i]);
      const int2 rs = __ldg(&rstat[f * rstat_stride + (long)v * g.SP + g.SPAD + ru]);
      int slr = 0;
      for (int dv = -h; dv <= h; ++dv) {
        const uint8_t* lr = L + (long)(v + dv) * W + u;
        const uint8_t* rr = R + (long)(v + dv) * W + ru;
        for (int du = -h + ((dv + h) & 1); du <= h; du += 2) slr += (int)__ldg(lr + du) * __ldg(rr + du);
      }
      const int num = 61 * slr - ls.x * rs.x;
      s = (__int2float_rn(num) * __int_as_float(rs.y)) * __int_as_float(ls.y);
    }
    win[(f * win_stride * (kWin / 2) + win_word(W, v, u, q >> 1)) * 2 + (q & 1)] =
        __ushort_as_half(m_code(s));
    if (q == 0) wbase[f * win_stride + bt_index(W, v, u)] = wb;
  }
}

void launch_window_fix(const float* disp, const uint8_t* valid, const uint8_t* lgray,
                       const uint8_t* rgray, const int2* lstat, const int2* rstat, wscore_t* win,
                       int* wbase, int* list, unsigned* count, const Geom& g, int frames,
                       long stride, long rstat_stride, long win_stride, cudaStream_t s) {
  if (g.W <= 0 || g.H <= 0 || frames <= 0) return;
  cudaMemsetAsync(count, 0, sizeof(unsigned) * frames, s);
  dim3 b(32, 8);
  k_window_check<<<dim3((g.W + 31) / 32, (g.H + 7) / 8, frames), b, 0, s>>>(
      disp, valid, lstat, wbase, list, count, g, stride, win_stride);
  k_window_build<<<dim3(148, frames), 256, 0, s>>>(disp, lgray, rgray, lstat, rstat, win, wbase,
                                                   list, count, g, stride, rstat_stride,
                                                   win_stride);
}

}  // namespace ssb
