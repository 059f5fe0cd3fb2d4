// ZNCC cost sweep + winner-take-all (compute_disparity, matcher.cpp:166-211).
//
// k_wta11 — the hot kernel, window 11 (the default and the paper's setting).
//   Block = 32 lanes (consecutive columns u) x NB warps (blocks of kDB = 16
//   consecutive candidates of the WTA range [d_min, d_max]) over a strip of
//   kTH rows. Thread 0 streams the strip's image rows into a shared-memory
//   ring (bulk copies on per-slot mbarriers, issued up to 16 rows ahead): per
//   row the block's left tap words (k_ltap), the right parity-split rows in 4
//   byte-shifted copies (k_rcopy: every 4-byte window is one aligned word plus
//   at most one funnel shift) and the right-window statistics. For every row y
//   entering or leaving the 11-row window a thread forms the two chessboard
//   half-sums of one image row
//       He(y) = sum_{du even} L(u+du, y) R(u-c+du, y)   (5 taps)
//       Ho(y) = sum_{du odd}  L(u+du, y) R(u-c+du, y)   (6 taps)
//   with 4 dp4a (u8 x u8 -> int32), and keeps two running sums per candidate
//   so that the exact integer cross sum slr(u, v, c) costs O(1) per row step
//   instead of 61 MACs:
//       X(v+1) = Y(v) - He(v-5) + Ho(v+6),   Y(v+1) = X(v) + He(v+6) - Ho(v-5)
//   where X(v) = sum_{dv even} He(v+dv) + sum_{dv odd} Ho(v+dv) = slr(v).
//   num = 61 slr - sl sr is exact; g = float(num) / sqrt(var_r) (FP32, <= 3 ulp)
//   feeds a per-thread (best, second, arg); every kRB rows the warps stage
//   them in shared memory and kRB warps merge one row each (named barriers:
//   the merge overlaps the other warps' next row). The staged g also give,
//   once a pixel's pick is known, the kWin = 16 scores around it: the
//   refinement's score window (32 B/pixel of fp16 match costs instead of a
//   (D+10) x 4 B cost volume). Windows reaching past [d_min, d_max] (the
//   re-pick's +-5 margin) are left to k_window_build.
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
#include "tma.cuh"

namespace ssb {

namespace {

constexpr int kRB = 1;  // output rows per shared-memory reduction chunk
constexpr int kTH = 64;  // rows per block strip (11-row warm-up amortised over 64)
constexpr int kNoArg = INT_MIN;  // "no defined candidate" (disparities may be negative)

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
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

// One image row as the thread's kDB candidates need it (read from the row
// ring): the left tap words (k_ltap) and 16 aligned bytes of each right
// parity stream (k_rcopy):
// stream A = plane (u - c0) & 1 from plane byte m0 - 10, stream B = the other
// plane from m0 - 10 + q0 (m0 = (u - c0) >> 1).
struct RowWords {
  uint4 L;
  uint32_t A[4], B[4];
};

// He (even-offset taps, 5) and Ho (odd-offset taps, 6) of candidate I = 2i + e:
// e = 0: even taps from A at byte 8 - i, odd taps from B at 7 - i;
// e = 1: even taps from B at 7 - i, odd taps from A at 7 - i.
template <int I>
__device__ __forceinline__ uint32_t term_e(const RowWords& w) {
  constexpr int t = I >> 1;
  if constexpr ((I & 1) == 0) return __dp4a(w.L.x, win<8 - t>(w.A), __dp4a(w.L.y, win<12 - t>(w.A), 0u));
  else return __dp4a(w.L.x, win<7 - t>(w.B), __dp4a(w.L.y, win<11 - t>(w.B), 0u));
}
template <int I>
__device__ __forceinline__ uint32_t term_o(const RowWords& w) {
  constexpr int t = I >> 1;
  if constexpr ((I & 1) == 0) return __dp4a(w.L.z, win<7 - t>(w.B), __dp4a(w.L.w, win<11 - t>(w.B), 0u));
  else return __dp4a(w.L.z, win<7 - t>(w.A), __dp4a(w.L.w, win<11 - t>(w.A), 0u));
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

// Score candidate I: g = float(61 slr - sl sr) / sqrt(var_r) (NaN when
// undefined), staged for the window; (best, second, arg) kept NaN-safe:
// second' = min(best, max(second, g)) is the runner-up for any g order.
template <bool MASKED, int I>
__device__ __forceinline__ void score_i(const int (&X)[kDB], const int2* rrow, int sl,
                                        unsigned amask, float* gs, float& best, float& second,
                                        int& arg) {
  const int2 rs = rrow[-I];  // shared-memory row ring
  const int num = 61 * X[I] - sl * rs.x;
  float gv = __int2float_rn(num) * __int_as_float(rs.y);
  gs[I * 32] = gv;
  if constexpr (MASKED) gv = ((amask >> I) & 1) ? gv : __int_as_float(0x7fc00000);
  second = fminf(best, fmaxf(second, gv));
  arg = gv > best ? I : arg;
  best = fmaxf(best, gv);
}
template <bool MASKED, int... Is>
__device__ __forceinline__ void score_all(const int (&X)[kDB], const int2* rrow, int sl,
                                          unsigned amask, float* gs, float& best, float& second,
                                          int& arg, std::integer_sequence<int, Is...>) {
  (score_i<MASKED, Is>(X, rrow, sl, amask, gs, best, second, arg), ...);
}

}  // namespace

// Shared-memory row ring of the staged sweep. Slot of image row y:
//   [0, 512)                 ltap[y][u0 .. u0+31]
//   [512, 512 + 32 RW)       rcopy[y][par][s][wlo .. wlo+RW) (8 sub-rows)
//   [512 + 32 RW, +8 RSN)    rstat[y][e_lo .. e_lo+RSN) (int2)
// filled by one thread with bulk copies completing on the slot's mbarrier.
// Rows in flight: 12 live rows (v - 6 .. v + 5) + kRB rows of the next chunk
// + prefetch depth; a power of two so slot indices are masks.
constexpr int kNSlots = 16;
static_assert(kNSlots >= 11 + 2 * kRB + 1, "row ring too small");
struct RingGeom {
  int RW, RSN, slot_bytes;
};
__host__ __device__ inline RingGeom ring_geom(int NB) {
  RingGeom r;
  const int span_m = (31 + kDB * (NB - 1)) / 2 + 2;  // m0 range of a block (+ slack)
  r.RW = ((span_m + 3) / 4 + 9 + 3) / 4 * 4;            // words per sub-row, 16 B multiple
  r.RSN = (kDB * NB + 31 + 2 + 1) / 2 * 2;              // rstat elements, 16 B multiple
  r.slot_bytes = (512 + 32 * r.RW + 8 * r.RSN + 127) / 128 * 128;
  return r;
}

__global__ void __launch_bounds__(512) k_wta11(
    const uint4* __restrict__ ltap, const uint32_t* __restrict__ rcopy,
    const int2* __restrict__ lstat, const int2* __restrict__ rstat, wscore_t* __restrict__ win,
    int* __restrict__ wbase, const int* __restrict__ base_map, float* __restrict__ disp,
    uint8_t* __restrict__ valid, int* __restrict__ flag_list,
    unsigned int* __restrict__ flag_count, Geom g, float min_zncc_f, float thr_tol,
    int do_argmax, long tap_stride, long copy_stride, long lstat_stride, long rstat_stride,
    long map_stride, long win_stride) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // warps 0 .. NB-1 sweep (one block of kDB candidates each); warp NB merges
  const int lane = threadIdx.x, j = threadIdx.y, NB = blockDim.y - 1;
  const bool merger = j == NB;
  const int NCB = NB * kDB;  // staged candidates per pixel
  const RingGeom rg = ring_geom(NB);
  unsigned char* ring = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kNSlots * rg.slot_bytes);
  // staging, double-buffered by chunk parity: partials [2][kRB][NB][32],
  // scores [2][kRB][NCB][32]
  float* s_best0 = reinterpret_cast<float*>(bars + kNSlots);
  float* s_sec0 = s_best0 + 2 * kRB * NB * 32;
  int* s_arg0 = reinterpret_cast<int*>(s_sec0 + 2 * kRB * NB * 32);
  float* s_g0 = reinterpret_cast<float*>(s_arg0 + 2 * kRB * NB * 32);

  const long fr = blockIdx.z;
  ltap += fr * tap_stride;
  rcopy += fr * copy_stride;
  lstat += fr * lstat_stride;
  if (win) {
    win += fr * win_stride * kWin;
    wbase += fr * win_stride;
  }
  if (base_map) base_map += fr * map_stride;
  disp += fr * map_stride;
  valid += fr * map_stride;
  flag_list += fr * map_stride;
  flag_count += fr;

  constexpr int h = 5;
  const int W = g.W, H = g.H;
  const int u0 = h + blockIdx.x * 32;
  const int u = u0 + lane;
  const int v_begin = h + blockIdx.y * kTH;
  const int v_end = min(v_begin + kTH, H - h);
  if (v_begin >= v_end) return;  // uniform over the block
  // The sweep covers exactly the WTA range [d_min, d_max]; window entries
  // outside it (the refinement's +-5 margin) come from k_window_build.
  const int ND = g.dmax - g.dmin + 1;
  const int c0 = g.dmin + j * kDB;
  const int nact = merger ? 0 : min(kDB, ND - j * kDB);
  const bool active = (u < W - h) && (nact > 0);
  unsigned amask = 0;
#pragma unroll
  for (int i = 0; i < kDB; ++i)
    amask |= i < nact ? (1u << i) : 0u;
  // warps whose candidates all take part in the WTA argmax skip the mask
  const bool full = __all_sync(0xffffffffu, amask == 0xFFFFu || !active);

  // ---- block-uniform copy geometry ----
  const int PW = g.PP / 4;
  const int c0_last = g.dmin + kDB * (NB - 1);
  const int m0_min = (u0 - c0_last) >> 1;
  const int wlo = ((g.PB + m0_min - 10) >> 2) & ~3;
  const int ru_lo = u0 - c0_last - (kDB - 1);  // lowest right column any thread scores
  const long rs_base = fr * rstat_stride + g.SPAD + ru_lo;  // + y * SP: element of ru_lo
  // ---- per-thread stream offsets (words into a slot's rcopy area) ----
  const int ru0 = u - c0;
  const int q0 = ru0 & 1;
  const int m0 = ru0 >> 1;  // arithmetic shift: floor for negative ru0
  const int stA = g.PB + m0 - 10, stB = stA + q0;
  const int offA = (q0 * 4 + (stA & 3)) * rg.RW + (stA >> 2) - wlo;
  const int offB = ((1 - q0) * 4 + (stB & 3)) * rg.RW + (stB >> 2) - wlo;
  const int offR = ru0 - ru_lo;  // + (row parity of rs_base + y SP) -> rstat element

  const int y_first = v_begin - h, y_last = v_end + h - 1;  // rows this strip reads
  const int tid = j * 32 + lane;
  auto issue = [&](int y) {  // thread 0 only
    const int k = (y - y_first) & (kNSlots - 1);
    unsigned char* sl = ring + (size_t)k * rg.slot_bytes;
    uint64_t* bar = bars + k;
    const long rsg = rs_base + (long)y * g.SP;
    const long rse = rsg & ~1L;
    mbar_expect_tx(bar, 512u + 32u * rg.RW + 8u * rg.RSN);
    bulk_g2s(sl, ltap + (long)y * W + u0, 512u, bar);
    const uint32_t* rrow = rcopy + (long)y * 8 * PW + wlo;
#pragma unroll 1
    for (int r = 0; r < 8; ++r)
      bulk_g2s(sl + 512 + r * rg.RW * 4, rrow + (long)r * PW, rg.RW * 4u, bar);
    bulk_g2s(sl + 512 + 32 * rg.RW, rstat + rse, 8u * rg.RSN, bar);
  };
  auto slot_of = [&](int y) {
    return ring + (size_t)((y - y_first) & (kNSlots - 1)) * rg.slot_bytes;
  };
  auto wait_row = [&](int y) {
    const int n = y - y_first;
    mbar_wait(bars + (n & (kNSlots - 1)), (unsigned)(n / kNSlots) & 1u);
  };
  int issued = y_first - 1;  // last row issued
  if (tid == 0) {
    for (int k = 0; k < kNSlots; ++k) mbar_init(bars + k, 1);
    mbar_fence_init();
    for (int y = y_first; y <= min(y_last, y_first + kNSlots - 1); ++y) issue(y);
  }
  issued = min(y_last, y_first + kNSlots - 1);
  __syncthreads();

  auto words = [&](int y) {
    const unsigned char* sl = slot_of(y);
    RowWords w;
    w.L = reinterpret_cast<const uint4*>(sl)[lane];
    const uint32_t* rc = reinterpret_cast<const uint32_t*>(sl + 512);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      w.A[t] = rc[offA + t];
      w.B[t] = rc[offB + t];
    }
    return w;
  };

  const int nrows = v_end - v_begin;
  const int nchunks = (nrows + kRB - 1) / kRB;
  // Named barriers: FULL(b) = 1 + b (sweep warps arrive, the merger waits),
  // EMPTY(b) = 3 + b (the merger arrives, sweep warps wait before reusing
  // staging buffer b two chunks later).
  const int nthr = (NB + 1) * 32;

  if (merger) {
    static_assert(kRB == 1, "the merge warp prefetches one row's 1/sqrt(var_l) ahead");
    // 1/sqrt(var_l) of the next row, loaded before waiting for its partials
    // (a global load off the merge warp's critical path)
    const bool in_img = u < W - h;
    float rl_next = in_img ? __int_as_float(__ldg(&lstat[(long)v_begin * W + u].y)) : 0.f;
    for (int k = 0; k < nchunks; ++k) {
      const int b = k & 1;
      const float rl_cur = rl_next;
      if (in_img && k + 1 < nchunks)
        rl_next = __int_as_float(__ldg(&lstat[(long)(v_begin + k + 1) * W + u].y));
      bar_sync(1 + b, nthr);
      const int vk0 = v_begin + k * kRB, rows = min(kRB, v_end - vk0);
      const int vlast = vk0 + rows - 1;
      // every sweep warp is past step vlast: rows <= vlast - 6 are dead
      if (lane == 0) {
        const int hi = min(y_last, vlast - 6 + kNSlots);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int y = issued + 1; y <= hi; ++y) issue(y);
      }
      issued = min(y_last, max(issued, vlast - 6 + kNSlots));
      const float* s_best = s_best0 + b * kRB * NB * 32;
      const float* s_sec = s_sec0 + b * kRB * NB * 32;
      const int* s_arg = s_arg0 + b * kRB * NB * 32;
      const float* s_g = s_g0 + b * kRB * NCB * 32;
      for (int r = 0; r < rows; ++r) {
        float B = -INFINITY, S = -INFINITY;
        int A = kNoArg;
        for (int jj = 0; jj < NB; ++jj) {
          const int o = (r * NB + jj) * 32 + lane;
          const int a = s_arg[o];
          if (a == kNoArg) continue;
          const float bb = s_best[o], s2 = s_sec[o];
          if (bb > B) {
            S = fmaxf(B, s2);
            B = bb;
            A = a;
          } else {
            S = fmaxf(S, fmaxf(bb, s2));
          }
        }
        if (u >= W - h) continue;
        const int vv = vk0 + r;
        const long idx = (long)vv * W + u;
        const float rl = rl_cur;
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
        if (!win) continue;  // argmax only (right view of the LR check)
        const int anchor = base_map ? base_map[idx] : A;
        int wb = kNoWin;
        if (!isnan(rl) && anchor != kNoArg && anchor != kNoWin)
          wb = window_base(anchor, g.cmin, g.NC);
        // A window reaching past [d_min, d_max] is left for k_window_build
        // (wbase kNoWin never matches the post-cleanup check's target).
        if (wb != kNoWin && (wb < g.dmin || wb + kWin - 1 > g.dmax)) wb = kNoWin;
        const long bi = bt_index(W, vv, u);
        wbase[bi] = wb;
        if (wb != kNoWin) {
          const float* gr = s_g + (r * NCB + wb - g.dmin) * 32 + lane;
          uint32_t w[kWin / 2];  // kWin fp16 match costs (m_code)
#pragma unroll
          for (int q = 0; q < kWin / 2; ++q)
            w[q] = pack_m2(gr[(2 * q) * 32] * rl, gr[(2 * q + 1) * 32] * rl);
          uint32_t* wq = reinterpret_cast<uint32_t*>(win) + win_word(W, vv, u, 0);
#pragma unroll
          for (int q = 0; q < kWin / 2; ++q) wq[(long)q * W * 32] = w[q];
        }
      }
      __syncwarp();
      bar_arrive(3 + b, nthr);
    }
    return;
  }

  int X[kDB], Y[kDB];
#pragma unroll
  for (int i = 0; i < kDB; ++i) X[i] = Y[i] = 0;

#pragma unroll 1
  for (int dy = -h; dy <= h; ++dy) {
    const int y = v_begin + dy;
    wait_row(y);
    if (active) {
      const RowWords w = words(y);
      warm_all(w, ((dy + h) & 1) == 1 /* dy even */, X, Y, std::make_integer_sequence<int, kDB>{});
    }
  }

  for (int v = v_begin; v < v_end; ++v) {
    if (v > v_begin) {
      wait_row(v + 5);
      if (active) {
        const RowWords wo = words(v - 6);
        const RowWords wn = words(v + 5);
        step_all(wo, wn, X, Y, std::make_integer_sequence<int, kDB>{});
      }
    }
    const int k = (v - v_begin) / kRB, slot = (v - v_begin) - k * kRB, b = k & 1;
    // staging buffer b was merged (chunk k - 2) before it is rewritten
    if (slot == 0 && k >= 2) bar_sync(3 + b, nthr);
    float* gs = s_g0 + ((b * kRB + slot) * NCB + j * kDB) * 32 + lane;
    float best = -INFINITY, second = -INFINITY;
    int arg = kNoArg;
    if (active) {
      const int sl = __ldg(&lstat[(long)v * W + u].x);
      const int2* rrow = reinterpret_cast<const int2*>(slot_of(v) + 512 + 32 * rg.RW) + offR +
                         (int)((rs_base + (long)v * g.SP) & 1);
      int ai = -1;
      if (full)
        score_all<false>(X, rrow, sl, amask, gs, best, second, ai,
                         std::make_integer_sequence<int, kDB>{});
      else
        score_all<true>(X, rrow, sl, amask, gs, best, second, ai,
                        std::make_integer_sequence<int, kDB>{});
      arg = ai >= 0 ? c0 + ai : kNoArg;
    }
    const int so = ((b * kRB + slot) * NB + j) * 32 + lane;
    s_best0[so] = best;
    s_sec0[so] = second;
    s_arg0[so] = arg;
    if (slot == kRB - 1 || v == v_end - 1) bar_arrive(1 + b, nthr);  // chunk k staged
  }
}

void launch_wta11(const uint4* ltap, const uint32_t* rcopy, const int2* lstat, const int2* rstat,
                  wscore_t* win, int* wbase, const int* base_map, float* disp, uint8_t* valid,
                  int* flag_list, unsigned int* flag_count, const Geom& g, double min_zncc,
                  int frames, long tap_stride, long copy_stride, long lstat_stride,
                  long rstat_stride, long map_stride, long win_stride, int do_argmax,
                  cudaStream_t s) {
  const int h = 5;
  if (g.W - 2 * h <= 0 || g.H - 2 * h <= 0 || frames <= 0) return;
  const int NB = (g.dmax - g.dmin + 1 + kDB - 1) / kDB;
  const RingGeom rg = ring_geom(NB);
  dim3 block(32, NB + 1);
  dim3 grid((g.W - 2 * h + 31) / 32, (g.H - 2 * h + kTH - 1) / kTH, frames);
  const size_t smem = (size_t)kNSlots * rg.slot_bytes + 8 * kNSlots +
                      2 * ((size_t)kRB * NB * 32 * 12 + (size_t)kRB * NB * kDB * 32 * 4);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(k_wta11, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  const float mz = (float)min_zncc;
  const float tol = 4e-6f * fmaxf(1.f, fabsf(mz));
  k_wta11<<<grid, block, smem, s>>>(ltap, rcopy, lstat, rstat, win, wbase, base_map, disp, valid,
                                    flag_list, flag_count, g, mz, tol, do_argmax, tap_stride,
                                    copy_stride, lstat_stride, rstat_stride, map_stride,
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

// Pixels queued by the window check in k_refine_init (a valid pixel whose
// sweep window is not centred on its possibly filled disparity): half a warp
// per queued pixel, lane q computes candidate wbase + q
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

void launch_window_build(const float* disp, const uint8_t* lgray, const uint8_t* rgray,
                         const int2* lstat, const int2* rstat, wscore_t* win, int* wbase,
                         const int* list, const unsigned* count, const Geom& g, int frames,
                         long stride, long rstat_stride, long win_stride, cudaStream_t s) {
  if (g.W <= 0 || g.H <= 0 || frames <= 0) return;
  k_window_build<<<dim3(148, frames), 256, 0, s>>>(disp, lgray, rgray, lstat, rstat, win, wbase,
                                                   list, count, g, stride, rstat_stride,
                                                   win_stride);
}

}  // namespace ssb
