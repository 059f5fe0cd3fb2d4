// Frame preparation kernels: luma, tap words / parity planes, chessboard window stats.
//
//   k_to_gray   to_gray, matcher.cpp:21-30 (FP64, no FMA, lround)
//   k_ltap      left tap words and k_rcopy byte-shifted right parity planes
//               for the dp4a cross-correlation (layout in ss_internal.cuh)
//   k_stats     patch_stats, matcher.cpp:112-137, plus the float reciprocal
//               sqrt of the variance used by the FP32 filter of the WTA sweep
//
// All three are HBM/latency-trivial next to the WTA sweep (a few bytes and a
// few dozen integer ops per pixel); they are written for coalescing only.
#include "ss_internal.cuh"

namespace ssb {

__global__ void k_to_gray(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ gray,
                          long n, long in_stride, long out_stride) {
  const long f = blockIdx.y;
  rgb += f * in_stride;
  gray += f * out_stride;
  // (0.299 R + 0.587 G) + 0.114 B, each product rounded, no contraction;
  // lround: half away from 0
  auto luma = [](uint32_t r, uint32_t g, uint32_t b) -> uint32_t {
    const double x = __dadd_rn(__dadd_rn(__dmul_rn(0.299, (double)r), __dmul_rn(0.587, (double)g)),
                               __dmul_rn(0.114, (double)b));
    return (uint32_t)round(x);
  };
  const long step = (long)gridDim.x * blockDim.x;
  const long t0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long i0 = 0;
  if (((reinterpret_cast<uintptr_t>(rgb) | reinterpret_cast<uintptr_t>(gray)) & 3) == 0) {
    // four pixels per thread: three 32-bit loads, one 32-bit store
    const long nq = n / 4;
    for (long q = t0; q < nq; q += step) {
      const uint32_t* s = reinterpret_cast<const uint32_t*>(rgb) + 3 * q;
      const uint32_t w0 = __ldg(s), w1 = __ldg(s + 1), w2 = __ldg(s + 2);
      const uint32_t g0 = luma(w0 & 0xFF, (w0 >> 8) & 0xFF, (w0 >> 16) & 0xFF);
      const uint32_t g1 = luma(w0 >> 24, w1 & 0xFF, (w1 >> 8) & 0xFF);
      const uint32_t g2 = luma((w1 >> 16) & 0xFF, w1 >> 24, w2 & 0xFF);
      const uint32_t g3 = luma((w2 >> 8) & 0xFF, (w2 >> 16) & 0xFF, w2 >> 24);
      reinterpret_cast<uint32_t*>(gray)[q] = g0 | g1 << 8 | g2 << 16 | g3 << 24;
    }
    i0 = nq * 4;
  }
  for (long i = i0 + t0; i < n; i += step)
    gray[i] = (uint8_t)luma(rgb[3 * i + 0], rgb[3 * i + 1], rgb[3 * i + 2]);
}

void launch_to_gray(const uint8_t* rgb, uint8_t* gray, long n, int frames, long in_stride,
                    long out_stride, cudaStream_t s) {
  if (n <= 0 || frames <= 0) return;
  const int threads = 256;
  long blocks = (n / 4 + threads - 1) / threads;  // four pixels per thread
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  k_to_gray<<<dim3((unsigned)blocks, frames), threads, 0, s>>>(rgb, gray, n, in_stride,
                                                              out_stride);
}

// Left tap words, one uint4 per pixel (u, y) (ss_internal.cuh):
//   x = L(u-4) L(u-2) L(u) L(u+2)   y = L(u+4) 0 0 0
//   z = L(u-5) L(u-3) L(u-1) L(u+1) w = L(u+3) L(u+5) 0 0
// byte 0 lowest; bytes outside the row are 0 (such pixels never score).
__global__ void __launch_bounds__(128)
    k_ltap(const uint8_t* __restrict__ gray, uint4* __restrict__ ltap, int W, long gray_stride,
           long tap_stride) {
  // the block's row segment u0 - 5 .. u0 + 132 staged once (coalesced), each
  // thread then packs its 11 taps from shared memory
  __shared__ uint8_t seg[128 + 16];
  const long f = blockIdx.z;
  const int u0 = blockIdx.x * 128;
  const int u = u0 + threadIdx.x;
  const int y = blockIdx.y;
  const uint8_t* row = gray + f * gray_stride + (long)y * W;
  for (int k = threadIdx.x; k < 128 + 10; k += 128) {
    const int x = u0 - 5 + k;
    seg[k] = (x >= 0 && x < W) ? __ldg(row + x) : 0;
  }
  __syncthreads();
  if (u >= W) return;
  auto at = [&](int dx) -> uint32_t { return seg[threadIdx.x + 5 + dx]; };
  uint4 t;
  t.x = at(-4) | at(-2) << 8 | at(0) << 16 | at(2) << 24;
  t.y = at(4);
  t.z = at(-5) | at(-3) << 8 | at(-1) << 16 | at(1) << 24;
  t.w = at(3) | at(5) << 8;
  ltap[f * tap_stride + (long)y * W + u] = t;
}

__global__ void k_rcopy(const uint8_t* __restrict__ gray, uint32_t* __restrict__ rcopy, int W,
                        int PB, int PP, long gray_stride, long copy_stride) {
  // one thread: word wi of the four byte-shifted copies s = 0..3 of plane
  // `par` of image row y (sub-rows (y * 2 + par) * 4 + s): plane bytes
  // j0 .. j0 + 6, j0 = 4 wi - PB, loaded once and funnel-shifted per s
  const long f = blockIdx.z;
  const int words = PP / 4;
  const int wi = blockIdx.x * blockDim.x + threadIdx.x;
  const int yp = blockIdx.y;  // y * 2 + par
  if (wi >= words) return;
  const int par = yp & 1, y = yp >> 1;
  const int half_w = (W + 1) / 2;
  const uint8_t* src = gray + f * gray_stride + (long)y * W;
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int b = 0; b < 7; ++b) {
    const int j = wi * 4 + b - PB;  // plane index
    const int x = 2 * j + par;
    const uint32_t val = (j >= 0 && j < half_w && x < W) ? (uint32_t)__ldg(src + x) : 0u;
    if (b < 4) lo |= val << (8 * b);
    else hi |= val << (8 * (b - 4));
  }
  uint32_t* dst = rcopy + f * copy_stride + (long)yp * 4 * words + wi;
#pragma unroll
  for (int s = 0; s < 4; ++s) dst[(long)s * words] = __funnelshift_r(lo, hi, 8 * s);
}

void launch_ltap(const uint8_t* gray, uint4* ltap, const Geom& g, int frames, long gray_stride,
                 long tap_stride, cudaStream_t s) {
  if (g.W <= 0 || g.H <= 0 || frames <= 0) return;
  k_ltap<<<dim3((g.W + 127) / 128, g.H, frames), 128, 0, s>>>(gray, ltap, g.W, gray_stride,
                                                              tap_stride);
}

void launch_rcopy(const uint8_t* gray, uint32_t* rcopy, const Geom& g, int frames,
                  long gray_stride, long copy_stride, cudaStream_t s) {
  if (g.W <= 0 || g.H <= 0 || frames <= 0) return;
  const int words = g.PP / 4;
  k_rcopy<<<dim3((words + 127) / 128, 2 * g.H, frames), 128, 0, s>>>(
      gray, rcopy, g.W, g.PB, g.PP, gray_stride, copy_stride);
}

// Chessboard window statistics of one image. out[i] = {sum, bits(1/sqrt(var))}
// with NaN when the window leaves the image or var == 0 (undefined ZNCC).
// Right-image rows are padded by SPAD entries each side ({0, NaN}).
// Any window (int64 sums); window 11 runs k_stats_col below.
__global__ void k_stats(const uint8_t* __restrict__ gray, int2* __restrict__ out, int W,
                        int H, int half, int pitch, int pad, long gray_stride,
                        long stat_stride) {
  const long f = blockIdx.z;
  gray += f * gray_stride;
  out += f * stat_stride;
  const int v = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < pitch;
       x += gridDim.x * blockDim.x) {
    const int u = x - pad;
    int2 r = make_int2(0, __float_as_int(__int_as_float(0x7fc00000)));
    if (u >= half && u < W - half && v >= half && v < H - half) {
      int64_t n = 0, s = 0, sq = 0;
      for (int dv = -half; dv <= half; ++dv) {
        const uint8_t* row = gray + (long)(v + dv) * W + u;
        for (int du = -half + ((dv + half) & 1); du <= half; du += 2) {
          const int64_t a = row[du];
          n += 1;
          s += a;
          sq += a * a;
        }
      }
      // patch_stats stores int32 (matcher.cpp:132-133); windows >= 27 wrap.
      const int32_t var = (int32_t)(n * sq - s * s);
      r.x = (int32_t)s;
      if (var != 0) r.y = __float_as_int((float)(1.0 / sqrt((double)var)));
    }
    out[(long)v * pitch + x] = r;
  }
}

// Window 11 (the default): one thread walks one column down a strip of
// kStatRows output rows with running sums, so each image row is read once per
// column (11 byte loads) instead of once per output pixel (61). For output v
// the chessboard taps are: rows v + odd k use the row's odd-offset taps
// (du = +-1, +-3, +-5: "Ho"), rows v + even k its even-offset taps (du = 0,
// +-2, +-4: "He"). With P(r) = Ho(r) | He(r) << 16 (each half <= 6 * 255, so
// sums of 6 rows never carry) and
//   PO(v) = sum_{k odd} P(v + k),   PE(v) = sum_{k even} P(v + k),
// the window sum is lo16(PO) + hi16(PE), and one row down
//   PO(v + 1) = PE(v) + P(v + 6),   PE(v + 1) = PO(v) - P(v - 5);
// the squares run the same recurrences on separate Ho / He accumulators.
// Integer sums: bit-identical to the direct 61-tap loop of k_stats.
constexpr int kStatRows = 32;
constexpr int kStatCols = 128;

__global__ void __launch_bounds__(kStatCols)
    k_stats_col(const uint8_t* __restrict__ gray, int2* __restrict__ out, int W, int H,
                int pitch, int pad, long gray_stride, long stat_stride) {
  constexpr int HALF = 5;
  __shared__ int3 ring[12][kStatCols];  // P, Qo, Qe of the column's last 12 rows
  const long f = blockIdx.z;
  gray += f * gray_stride;
  out += f * stat_stride;
  const int x = blockIdx.x * kStatCols + threadIdx.x;
  if (x >= pitch) return;
  const int u = x - pad;
  const int v0 = blockIdx.y * kStatRows, v1 = min(v0 + kStatRows, H);
  const int2 undef = make_int2(0, 0x7fc00000);
  const bool col_ok = u >= HALF && u < W - HALF;
  const int vs = max(v0, HALF), ve = min(v1, H - HALF);  // rows with a fitting window
  for (int v = v0; v < (col_ok ? min(vs, v1) : v1); ++v) out[(long)v * pitch + x] = undef;
  if (!col_ok || vs >= ve) {
    if (col_ok)
      for (int v = max(vs, ve); v < v1; ++v) out[(long)v * pitch + x] = undef;
    return;
  }
  int3* rc = &ring[0][threadIdx.x];
  auto row_sums = [&](int r) {  // P, Qo, Qe of image row r at column u
    const uint8_t* p = gray + (long)r * W + u;
    int P = 0, qo = 0, qe = 0;
#pragma unroll
    for (int du = -HALF; du <= HALF; ++du) {
      const int a = __ldg(p + du);
      if (du & 1) {
        P += a;
        qo += a * a;
      } else {
        P += a << 16;
        qe += a * a;
      }
    }
    return make_int3(P, qo, qe);
  };
  // warm-up: rows vs - 5 .. vs + 5 by parity of k = r - vs
  int PO = 0, PE = 0, QOo = 0, QEo = 0, QOe = 0, QEe = 0;
#pragma unroll 1
  for (int k = -HALF; k <= HALF; ++k) {
    const int3 s = row_sums(vs + k);
    rc[((vs + k) % 12) * kStatCols] = s;
    if (k & 1) {
      PO += s.x;
      QOo += s.y;
      QOe += s.z;
    } else {
      PE += s.x;
      QEo += s.y;
      QEe += s.z;
    }
  }
#pragma unroll 1
  for (int v = vs;; ++v) {
    const int sum = (PO & 0xFFFF) + (int)((unsigned)PE >> 16);
    const int sq = QOo + QEe;
    // patch_stats stores int32 (matcher.cpp:132-133)
    const int32_t var = 61 * sq - sum * sum;
    int2 r = make_int2(sum, 0x7fc00000);
    if (var != 0) r.y = __float_as_int((float)(1.0 / sqrt((double)var)));
    out[(long)v * pitch + x] = r;
    if (v + 1 >= ve) break;
    const int3 nw = row_sums(v + HALF + 1);
    const int3 od = rc[((v - HALF) % 12) * kStatCols];
    rc[((v + HALF + 1) % 12) * kStatCols] = nw;
    const int po = PO, qoo = QOo, qoe = QOe;
    PO = PE + nw.x;
    QOo = QEo + nw.y;
    QOe = QEe + nw.z;
    PE = po - od.x;
    QEo = qoo - od.y;
    QEe = qoe - od.z;
  }
  for (int v = ve; v < v1; ++v) out[(long)v * pitch + x] = undef;
}

void launch_stats(const uint8_t* gray, int2* lstat, int2* rstat, int is_right, const Geom& g,
                  int frames, long gray_stride, long stat_stride, cudaStream_t s) {
  if (g.W <= 0 || g.H <= 0 || frames <= 0) return;
  const int pitch = is_right ? g.SP : g.W;
  const int pad = is_right ? g.SPAD : 0;
  const int threads = 128;
  dim3 grid((pitch + threads - 1) / threads, g.H, frames);
  if (g.half == 5) {
    dim3 gc((pitch + kStatCols - 1) / kStatCols, (g.H + kStatRows - 1) / kStatRows, frames);
    k_stats_col<<<gc, kStatCols, 0, s>>>(gray, is_right ? rstat : lstat, g.W, g.H, pitch, pad,
                                         gray_stride, stat_stride);
  } else
    k_stats<<<grid, threads, 0, s>>>(gray, is_right ? rstat : lstat, g.W, g.H, g.half, pitch,
                                        pad, gray_stride, stat_stride);
}

}  // namespace ssb
