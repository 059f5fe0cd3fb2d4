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
//   goes to the cost volume (read back by the refinement re-pick) and feeds a
//   per-thread (best, second, arg) that NB warps merge through shared memory.
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

template <int I>
__device__ __forceinline__ void terms_i(uint32_t Lea, uint32_t Leb, uint32_t Loa, uint32_t Lob,
                                        const uint32_t (&SA)[4], const uint32_t (&SB)[4],
                                        uint32_t (&He)[kDB], uint32_t (&Ho)[kDB]) {
  constexpr int t = I >> 1;
  if constexpr ((I & 1) == 0) {
    He[I] = __dp4a(Lea, win<8 - t>(SA), __dp4a(Leb, win<12 - t>(SA), 0u));
    Ho[I] = __dp4a(Loa, win<7 - t>(SB), __dp4a(Lob, win<11 - t>(SB), 0u));
  } else {
    He[I] = __dp4a(Lea, win<7 - t>(SB), __dp4a(Leb, win<11 - t>(SB), 0u));
    Ho[I] = __dp4a(Loa, win<7 - t>(SA), __dp4a(Lob, win<11 - t>(SA), 0u));
  }
}

template <int... Is>
__device__ __forceinline__ void terms_all(uint32_t Lea, uint32_t Leb, uint32_t Loa,
                                          uint32_t Lob, const uint32_t (&SA)[4],
                                          const uint32_t (&SB)[4], uint32_t (&He)[kDB],
                                          uint32_t (&Ho)[kDB],
                                          std::integer_sequence<int, Is...>) {
  (terms_i<Is>(Lea, Leb, Loa, Lob, SA, SB, He, Ho), ...);
}

// He/Ho of image row y for the thread's kDB candidates.
__device__ __forceinline__ void row_terms(const ThreadGeom& tg, int y, uint32_t (&He)[kDB],
                                          uint32_t (&Ho)[kDB]) {
  const uint8_t* lre = tg.lplane + (long)(2 * y + tg.p) * tg.PP;
  const uint8_t* lro = tg.lplane + (long)(2 * y + 1 - tg.p) * tg.PP;
  const uint32_t Lea = ld_win(lre, tg.Le);
  const uint32_t Leb = ld_win(lre, tg.Le + 4) & 0xFFu;
  const uint32_t Loa = ld_win(lro, tg.Lo);
  const uint32_t Lob = ld_win(lro, tg.Lo + 4) & 0xFFFFu;
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
  uint32_t SA[4], SB[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    SA[t] = __funnelshift_r(a[t], a[t + 1], tg.shA);
    SB[t] = __funnelshift_r(b[t], b[t + 1], tg.shB);
  }
  terms_all(Lea, Leb, Loa, Lob, SA, SB, He, Ho, std::make_integer_sequence<int, kDB>{});
}

}  // namespace

__global__ void __launch_bounds__(512) k_wta11(
    const uint8_t* __restrict__ lplane, const uint8_t* __restrict__ rplane,
    const int2* __restrict__ lstat, const int2* __restrict__ rstat, float* __restrict__ vol,
    float* __restrict__ disp, uint8_t* __restrict__ valid, int* __restrict__ flag_list,
    unsigned int* __restrict__ flag_count, Geom g, int TH, float min_zncc_f, float thr_tol,
    int do_argmax, long plane_stride, long lstat_stride, long rstat_stride, long vol_stride,
    long map_stride) {
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x, j = threadIdx.y, NB = blockDim.y;
  float* s_best = reinterpret_cast<float*>(smem_raw);
  float* s_sec = s_best + kRB * NB * 32;
  int* s_arg = reinterpret_cast<int*>(s_sec + kRB * NB * 32);

  const long fr = blockIdx.z;
  lplane += fr * plane_stride;
  rplane += fr * plane_stride;
  lstat += fr * lstat_stride;
  rstat += fr * rstat_stride;
  vol += fr * vol_stride;
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
      uint32_t He[kDB], Ho[kDB];
      row_terms(tg, v_begin + dy, He, Ho);
      const bool even = ((dy + h) & 1) == 1;  // dy even <=> dy + 5 odd
#pragma unroll
      for (int i = 0; i < kDB; ++i) {
        X[i] += (int)(even ? He[i] : Ho[i]);
        Y[i] += (int)(even ? Ho[i] : He[i]);
      }
    }
  }

  for (int v = v_begin; v < v_end; ++v) {
    if (v > v_begin && active) {
      uint32_t Heo[kDB], Hoo[kDB], Hen[kDB], Hon[kDB];
      row_terms(tg, v - 6, Heo, Hoo);
      row_terms(tg, v + 5, Hen, Hon);
#pragma unroll
      for (int i = 0; i < kDB; ++i) {
        const int xn = Y[i] - (int)Heo[i] + (int)Hon[i];
        const int yn = X[i] + (int)Hen[i] - (int)Hoo[i];
        X[i] = xn;
        Y[i] = yn;
      }
    }
    float best = -INFINITY, second = -INFINITY;
    int arg = kNoArg;
    if (active) {
      const int sl = __ldg(&lstat[(long)v * W + u].x);
      const int2* rrow = rstat + (long)v * g.SP + g.SPAD + ru0;
      // pixel-major volume: this thread's kDB candidates are 64 contiguous bytes
      float4* vrow = reinterpret_cast<float4*>(vol + ((long)v * W + u) * g.NCP + j * kDB);
      float gvs[kDB];
#pragma unroll
      for (int i = 0; i < kDB; ++i) {
        gvs[i] = 0.f;
        if (i < nact) {
          const int2 rs = __ldg(rrow - i);
          const int num = 61 * X[i] - sl * rs.x;
          const float gv = __int2float_rn(num) * __int_as_float(rs.y);
          gvs[i] = gv;
          const int c = c0 + i;
          if (c >= g.dmin && c <= g.dmax) {
            if (gv > best) {
              second = best;
              best = gv;
              arg = c;
            } else {
              second = fmaxf(second, gv);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kDB / 4; ++q)
        if (4 * q < nact)  // NCP is a multiple of 4: the tail vector stays in this pixel
          __stcs(vrow + q, make_float4(gvs[4 * q], gvs[4 * q + 1], gvs[4 * q + 2], gvs[4 * q + 3]));
    }
    if (!do_argmax) continue;
    const int slot = (v - v_begin) & (kRB - 1);
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
      }
      __syncthreads();
    }
  }
}

void launch_wta11(const uint8_t* lplane, const uint8_t* rplane, const int2* lstat,
                  const int2* rstat, float* vol, float* disp, uint8_t* valid, int* flag_list,
                  unsigned int* flag_count, const Geom& g, double min_zncc, int frames,
                  long plane_stride, long lstat_stride, long rstat_stride, long vol_stride,
                  long map_stride, int do_argmax, cudaStream_t s) {
  const int h = 5;
  if (g.W - 2 * h <= 0 || g.H - 2 * h <= 0 || frames <= 0) return;
  const int NB = (g.NC + kDB - 1) / kDB;
  const int TH = 32;
  dim3 block(32, NB);
  dim3 grid((g.W - 2 * h + 31) / 32, (g.H - 2 * h + TH - 1) / TH, frames);
  const size_t smem = (size_t)kRB * NB * 32 * 12;
  const float mz = (float)min_zncc;
  const float tol = 4e-6f * fmaxf(1.f, fabsf(mz));
  k_wta11<<<grid, block, smem, s>>>(lplane, rplane, lstat, rstat, vol, disp, valid, flag_list,
                                    flag_count, g, TH, mz, tol, do_argmax, plane_stride,
                                    lstat_stride, rstat_stride, vol_stride, map_stride);
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

}  // namespace ssb
