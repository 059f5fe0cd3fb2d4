// Outlier removal and hole filling (cleanup.cpp:12-123).
//
// Every pass reads an input map and writes a full output map (the reference
// copies the map first: cleanup.cpp:13,46), so stale disparities under an
// invalid mask propagate exactly as in the reference.
//
//   k_remove_outliers  cleanup.cpp:12-42 — 8 rays, early exit on the first
//                      smooth ray; |cur - prev| compared in double.
//   k_fill_radial      cleanup.cpp:54-68 — nearest valid hit per ray <= R,
//                      IDW w = 1/(step * {1, sqrt2}), double sums in direction
//                      order 0..7 (the reference's order, so bit-exact).
//   k_disc_select /    cleanup.cpp:69-84 — support of every invalid pixel from
//   k_disc_sum         per-row prefix counts (exact integers); only pixels that
//                      will be filled enter a compacted list, and one thread
//                      per listed pixel accumulates all valid pixels of the
//                      radius-R disc in raster order in FP64, w = 1/sqrt(dd)
//                      from a table built with the same IEEE ops on the host.
// All maps of a frame stay L2-resident (5 B/pixel); these passes are a few
// percent of the frame and latency-, not bandwidth-bound.
#include <math.h>

#include <algorithm>

#include "ss_internal.cuh"

namespace ssb {


__constant__ int c_dirU[8] = {1, -1, 0, 0, 1, 1, -1, -1};
__constant__ int c_dirV[8] = {0, 0, 1, -1, 1, -1, 1, -1};

// Outlier rays as bit-parallel runs over smooth-edge bitmaps. A ray from a
// valid pixel p in direction e passes iff its far end is inside the image and
// every step q -> q + e (q = p, p + e, ...) joins two valid pixels with
// |d(q+e) - d(q)| <= thr (the reference's double comparison). That edge
// predicate is symmetric, so four edge maps hold it for all eight directions:
// E_h (q -> q+(1,0)), E_v ((0,1)), E_d1 ((1,1)) and E_d2 ((1,-1)), each
// row-major with bit u of word u/32 for pixel (u, v), plus the validity map.
// k_edge_words builds them (a warp walks a strip of rows of one 32-pixel word
// column: one coalesced load per pixel, neighbours by shuffles, one ballot per
// map and row); k_outlier_words decides 32 pixels per thread: a ray test is
// an AND over its r edges of one shifted word per step, horizontal runs by
// shift doubling, and a word stops as soon as all its valid pixels passed.
namespace {
constexpr int kEdgeMaps = 5;  // V, E_h, E_v, E_d1, E_d2
constexpr int kEdgeStrip = 8;  // rows per warp in k_edge_words (all loads in flight)
struct EdgeWords {
  const uint32_t* m[kEdgeMaps];
  int ww;  // words per row
  __device__ __forceinline__ uint32_t word(int map, int v, int q) const {
    return (q >= 0 && q < ww) ? __ldg(m[map] + (long)v * ww + q) : 0u;
  }
  // the 32 bits of row v of `map` starting at bit position `pos` (zero outside the row)
  __device__ __forceinline__ uint32_t bits(int map, int v, int pos) const {
    const int q = pos >> 5;  // floor (arithmetic shift)
    return __funnelshift_r(word(map, v, q), word(map, v, q + 1), pos & 31);
  }
};
__host__ __device__ inline int edge_ww(int W) { return (W + 31) / 32; }
}  // namespace

__global__ void __launch_bounds__(128)
    k_edge_words(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                 uint32_t* __restrict__ emap, int W, int H, double thr, long stride, long fw,
                 float* __restrict__ dcopy, float* __restrict__ dcopy2) {
  constexpr int KS = kEdgeStrip, NR = KS + 2;  // rows v0 - 1 .. v0 + KS
  const long f = blockIdx.z;
  const int lane = threadIdx.x;
  const int w = blockIdx.x * 4 + threadIdx.y, ww = edge_ww(W);
  if (w >= ww) return;
  const int v0 = blockIdx.y * KS;
  const int u = w * 32 + lane;
  const bool inx = u < W, inx1 = lane == 31 && u + 1 < W;
  // every load of the strip in flight at once: pixel (u, v) per lane, and
  // lane 31 also the right neighbour (u + 1, v)
  float x[NR], x1[NR];
  uint32_t ok = 0u, ok1 = 0u;  // bit j: row v0 - 1 + j valid at u / at u + 1 (lane 31)
  const long base = f * stride + (long)(v0 - 1) * W + u;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int v = v0 - 1 + j;
    x[j] = 0.f;
    x1[j] = 0.f;
    if (v >= 0 && v < H) {
      const long i = base + (long)j * W;
      if (inx) {
        x[j] = din[i];
        ok |= (vin[i] != 0 ? 1u : 0u) << j;
      }
      if (inx1) {
        x1[j] = din[i + 1];
        ok1 |= (vin[i + 1] != 0 ? 1u : 0u) << j;
      }
    }
  }
  if (inx) {
#pragma unroll
    for (int j = 1; j <= KS; ++j) {
      if (v0 - 1 + j < H) {
        if (dcopy) dcopy[base + (long)j * W] = x[j];
        if (dcopy2) dcopy2[base + (long)j * W] = x[j];
      }
    }
  }
  // right neighbours: from lane + 1, lane 31 from its own extra loads
  const uint32_t okn_all = __shfl_down_sync(0xFFFFFFFFu, ok, 1);
  const uint32_t okn = lane == 31 ? ok1 : okn_all;
  double d[NR], dn[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const float s = __shfl_down_sync(0xFFFFFFFFu, x[j], 1);
    d[j] = (double)x[j];
    dn[j] = (double)(lane == 31 ? x1[j] : s);
  }
  // smooth edge: both ends valid and |b - a| <= thr in double (cleanup.cpp:25-31)
  auto sm = [thr](double a, double b) { return !(fabs(b - a) > thr); };
  const long plane = (long)H * ww;
  uint32_t* out = emap + f * fw + (long)v0 * ww + w;
#pragma unroll
  for (int j = 1; j <= KS; ++j) {
    if (v0 - 1 + j >= H) break;
    const bool oc = (ok >> j) & 1u;
    const unsigned bv = __ballot_sync(0xFFFFFFFFu, oc);
    const unsigned bh = __ballot_sync(0xFFFFFFFFu, oc && ((okn >> j) & 1u) && sm(d[j], dn[j]));
    const unsigned bvv = __ballot_sync(0xFFFFFFFFu, oc && ((ok >> (j + 1)) & 1u) && sm(d[j], d[j + 1]));
    const unsigned bd1 =
        __ballot_sync(0xFFFFFFFFu, oc && ((okn >> (j + 1)) & 1u) && sm(d[j], dn[j + 1]));
    const unsigned bd2 =
        __ballot_sync(0xFFFFFFFFu, oc && ((okn >> (j - 1)) & 1u) && sm(d[j], dn[j - 1]));
    if (lane == 0) {
      uint32_t* o = out + (long)(j - 1) * ww;
      o[0] = bv;
      o[plane] = bh;
      o[2 * plane] = bvv;
      o[3 * plane] = bd1;
      o[4 * plane] = bd2;
    }
  }
}

// keep bits of the 32 pixels of word w of row v, for rays of r steps
// (r > 0). The early exit only skips rays whose pixels already passed.
__device__ __forceinline__ uint32_t outlier_keep(const EdgeWords& E, int W, int H, int v, int w,
                                                 int r) {
  const uint32_t valid = E.word(0, v, w);
  if (!valid) return 0u;
  uint32_t keep = 0u;
  const int u0 = w * 32;
  // horizontal: runs of r set bits of E_h, starting at u (1,0) or ending at u - 1 (-1,0)
  if (r <= 32) {
    // 64-bit windows over columns u0 - 32 .. u0 + 31 (lo) and u0 .. u0 + 63 (hi)
    const uint64_t a = ((uint64_t)E.word(1, v, w + 1) << 32) | E.word(1, v, w);
    const uint64_t b = ((uint64_t)E.word(1, v, w) << 32) | E.word(1, v, w - 1);
    // run-of-r masks by doubling: bit j of R set iff bits j .. j + r - 1 all set
    auto runs = [r](uint64_t x) {
      uint64_t acc = ~0ull, p = x;
      int off = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {  // p = runs of 2^k
        if ((r >> k) & 1) {
          acc &= p >> off;
          off += 1 << k;
        }
        if ((2 << k) > r) break;
        p &= p >> (1 << k);
      }
      return acc;
    };
    keep |= (uint32_t)runs(a);                 // bits u .. u + r - 1
    keep |= (uint32_t)(runs(b) >> (32 - r));   // bits u - r .. u - 1
  } else {
    uint32_t p = ~0u, m = ~0u;
    for (int k = 0; k < r && (p | m); ++k) {
      p &= E.bits(1, v, u0 + k);
      m &= E.bits(1, v, u0 - 1 - k);
    }
    keep |= p | m;
  }
  keep &= valid;
  if (keep == valid) return keep;
  // vertical and diagonal rays: one word per step; the far end must be in the image
  if (v + r <= H - 1) {
    uint32_t a = ~0u, d1 = ~0u, d2 = ~0u;
#pragma unroll 4
    for (int k = 0; k < r; ++k) {
      a &= E.word(2, v + k, w);                   // (0, 1): E_v rows v .. v + r - 1
      d1 &= E.bits(3, v + k, u0 + k);             // (1, 1): E_d1 row v + k, bit u + k
      d2 &= E.bits(4, v + k + 1, u0 - 1 - k);     // (-1, 1): E_d2 row v + k + 1, bit u - k - 1
      if (!((a | d1 | d2) & valid & ~keep)) break;
    }
    keep |= (a | d1 | d2) & valid;
    if (keep == valid) return keep;
  }
  if (v - r >= 0) {
    uint32_t a = ~0u, d1 = ~0u, d2 = ~0u;
#pragma unroll 4
    for (int k = 0; k < r; ++k) {
      a &= E.word(2, v - 1 - k, w);               // (0, -1): E_v rows v - 1 .. v - r
      d1 &= E.bits(3, v - 1 - k, u0 - 1 - k);     // (-1, -1): E_d1 row v - k - 1, bit u - k - 1
      d2 &= E.bits(4, v - k, u0 + k);             // (1, -1): E_d2 row v - k, bit u + k
      if (!((a | d1 | d2) & valid & ~keep)) break;
    }
    keep |= (a | d1 | d2) & valid;
  }
  (void)W;
  return keep;
}

// dout2/vout2 (optional): a second copy of the result (the radial fill's
// output buffer, so that fill only writes the pixels it fills; the disparity
// copies are written by k_edge_words); list/count (optional): per-frame list
// of the invalid output pixels (one atomic per warp, ~5% of the pixels).
// vout may alias the input validity (the maps hold it).
__global__ void __launch_bounds__(128)
    k_outlier_words(uint32_t* __restrict__ emap, uint8_t* vout, uint8_t* __restrict__ vout2,
                    int W, int H, int r, long stride, long fw, int* __restrict__ list,
                    unsigned* __restrict__ count) {
  const long f = blockIdx.z;
  const int ww = edge_ww(W);
  const int w = blockIdx.x * 32 + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  const bool act = w < ww && v < H;
  EdgeWords E;
  const long plane = (long)H * ww;
#pragma unroll
  for (int k = 0; k < kEdgeMaps; ++k) E.m[k] = emap + f * fw + k * plane;  // read only
  E.ww = ww;
  uint32_t keep = 0u, inimg = 0u;
  if (act) {
    keep = r > 0 ? outlier_keep(E, W, H, v, w, r) : E.word(0, v, w);  // r <= 0: no steps
    emap[f * fw + kEdgeMaps * plane + (long)v * ww + w] = keep;  // result plane (radial fill)
    const int n = min(32, W - w * 32);
    inimg = n == 32 ? ~0u : (1u << n) - 1u;
    const long i0 = f * stride + (long)v * W + w * 32;
    if (n == 32 && ((i0 & 15) == 0)) {
      uint4 q[2];
      uint32_t* qw = reinterpret_cast<uint32_t*>(q);
#pragma unroll
      for (int k = 0; k < 8; ++k)  // 4 bits -> 4 bytes of 0/1
        qw[k] = (((keep >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u;
      reinterpret_cast<uint4*>(vout + i0)[0] = q[0];
      reinterpret_cast<uint4*>(vout + i0)[1] = q[1];
      if (vout2) {
        reinterpret_cast<uint4*>(vout2 + i0)[0] = q[0];
        reinterpret_cast<uint4*>(vout2 + i0)[1] = q[1];
      }
    } else {
      for (int k = 0; k < n; ++k) {
        const uint8_t b = (keep >> k) & 1u;
        vout[i0 + k] = b;
        if (vout2) vout2[i0 + k] = b;
      }
    }
  }
  if (list) {
    // invalid output pixels, raster order within a thread's word
    const uint32_t bad = inimg & ~keep;
    const int c = __popc(bad);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if ((int)threadIdx.x >= o) incl += t;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (total) {
      unsigned base = 0;
      if (threadIdx.x == 31) base = atomicAdd(count + f, (unsigned)total);
      base = __shfl_sync(0xFFFFFFFFu, base, 31) + (unsigned)(incl - c);
      int* lf = list + f * stride;
      for (uint32_t m = bad; m; m &= m - 1) lf[base++] = v * W + w * 32 + (__ffs(m) - 1);
    }
  }
}
// Radial fill of one invalid pixel (cleanup.cpp:54-68): writes dout/vout
// only when the pixel is filled.
__device__ __forceinline__ void radial_fill_pixel(const float* __restrict__ din,
                                                  const uint8_t* __restrict__ vin,
                                                  float* __restrict__ dout,
                                                  uint8_t* __restrict__ vout, int W, int H,
                                                  int u, int v, int radius, int min_support) {
  const long i = (long)v * W + u;
  {
    double wsum = 0.0, vsum = 0.0;
    int support = 0;
    for (int dir = 0; dir < 8; ++dir) {
      const double len = dir < 4 ? 1.0 : 1.41421356237309504880;  // M_SQRT2
      const int du = c_dirU[dir], dv = c_dirV[dir];
      // first valid pixel at step 1..radius, stopping at the image border;
      // four steps' validity loads in flight at a time
      int hit = 0;
      for (int s0 = 1; s0 <= radius && hit == 0; s0 += 4) {
        uint8_t ok[4];
        bool in[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int step = s0 + k, nu = u + du * step, nv = v + dv * step;
          in[k] = step <= radius && nu >= 0 && nu < W && nv >= 0 && nv < H;
          ok[k] = in[k] ? __ldg(vin + (long)nv * W + nu) : 0;
        }
        bool stop = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (stop || hit) continue;
          if (!in[k]) stop = true;
          else if (ok[k]) hit = s0 + k;
        }
        if (stop) break;
      }
      if (hit) {
        const long ni = (long)(v + dv * hit) * W + (u + du * hit);
        const double w = __ddiv_rn(1.0, __dmul_rn((double)hit, len));
        wsum = __dadd_rn(wsum, w);
        vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(din + ni)));
        ++support;
      }
    }
    if (support >= min_support && wsum > 0.0) {
      dout[i] = (float)__ddiv_rn(vsum, wsum);
      vout[i] = 1;
    }
  }
}

__global__ void k_fill_radial(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                              float* __restrict__ dout, uint8_t* __restrict__ vout, int W, int H,
                              int radius, int min_support, long stride) {
  const long f = blockIdx.z;
  din += f * stride;
  vin += f * stride;
  dout += f * stride;
  vout += f * stride;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = (long)v * W + u;
  dout[i] = din[i];
  vout[i] = vin[i];
  if (!vin[i]) radial_fill_pixel(din, vin, dout, vout, W, H, u, v, radius, min_support);
}

// The outlier pass's result by columns and by diagonals (for the radial
// fill's ray searches): one warp per (32-row block, word column w), lane =
// row; each transposed word is one ballot over the lanes' row words. Lines:
// column u (position v); d1 = u - v + H - 1 (position v); d2 = u + v
// (position v); ceil(H/32) words per line. Word columns -1 .. ww cover the
// diagonals that cross a row block's first row outside the image.
namespace {
struct ValidLines {
  uint32_t *col, *d1, *d2;
  int hw;
};
__host__ __device__ inline ValidLines valid_lines(uint32_t* frame, int W, int H) {
  const int ww = edge_ww(W), hw = (H + 31) / 32;
  ValidLines L;
  L.col = frame + 6L * H * ww;
  L.d1 = L.col + (long)W * hw;
  L.d2 = L.d1 + (long)(W + H - 1) * hw;
  L.hw = hw;
  return L;
}
}  // namespace

__global__ void __launch_bounds__(128)
    k_valid_bits(uint32_t* __restrict__ emap, int W, int H, long fw) {
  const long f = blockIdx.z;
  const int lane = threadIdx.x;
  const int w = (int)(blockIdx.x * blockDim.y + threadIdx.y) - 1;  // -1 .. ww
  const int ww = edge_ww(W);
  if (w > ww) return;
  const int rb = blockIdx.y, v = rb * 32 + lane;
  uint32_t* fr = emap + f * fw;
  const uint32_t* K = fr + kEdgeMaps * (long)H * ww;
  auto kw = [&](int q) { return (v < H && q >= 0 && q < ww) ? K[(long)v * ww + q] : 0u; };
  const uint32_t km = kw(w - 1), k0 = kw(w), kp = kw(w + 1);
  const uint64_t a1 = ((uint64_t)kp << 32) | k0;  // columns 32w .. 32w + 63
  const uint64_t a2 = ((uint64_t)k0 << 32) | km;  // columns 32w - 32 .. 32w + 31
  const ValidLines L = valid_lines(fr, W, H);
  uint32_t mc = 0, m1 = 0, m2 = 0;
#pragma unroll 4
  for (int d = 0; d < 32; ++d) {
    // column 32w + d; d1 line through (32w + d, 32 rb); d2 line through it
    const uint32_t c = __ballot_sync(0xFFFFFFFFu, (k0 >> d) & 1u);
    const uint32_t x1 = __ballot_sync(0xFFFFFFFFu, (uint32_t)(a1 >> (d + lane)) & 1u);
    const uint32_t x2 = __ballot_sync(0xFFFFFFFFu, (uint32_t)(a2 >> (32 + d - lane)) & 1u);
    if (lane == d) {
      mc = c;
      m1 = x1;
      m2 = x2;
    }
  }
  const int u = 32 * w + lane;
  if (w >= 0 && u < W) L.col[(long)u * L.hw + rb] = mc;
  const long i1 = (long)u - rb * 32 + H - 1, i2 = (long)u + rb * 32;
  if (w < ww && i1 >= 0 && i1 < W + H - 1) L.d1[i1 * L.hw + rb] = m1;
  if (w >= 0 && i2 >= 0 && i2 < W + H - 1) L.d2[i2 * L.hw + rb] = m2;
}

namespace {
// first / last set position of a bit line in [a, b] (a <= b), or -1
__device__ __forceinline__ int first_set(const uint32_t* __restrict__ line, int a, int b) {
  for (int q = a >> 5; q <= (b >> 5); ++q) {
    uint32_t x = __ldg(line + q);
    if (q == (a >> 5)) x &= ~0u << (a & 31);
    if (q == (b >> 5)) x &= ~0u >> (31 - (b & 31));
    if (x) return q * 32 + __ffs(x) - 1;
  }
  return -1;
}
__device__ __forceinline__ int last_set(const uint32_t* __restrict__ line, int a, int b) {
  for (int q = b >> 5; q >= (a >> 5); --q) {
    uint32_t x = __ldg(line + q);
    if (q == (a >> 5)) x &= ~0u << (a & 31);
    if (q == (b >> 5)) x &= ~0u >> (31 - (b & 31));
    if (x) return q * 32 + 31 - __clz(x);
  }
  return -1;
}
}  // namespace

// Chain variant: dout/vout already hold the input map (the outlier pass's
// second copy); one thread per listed invalid pixel. The nearest valid pixel
// of each ray is a bit search on the outlier result's row, column or
// diagonal line (the reference's per-step walk, cleanup.cpp:57-66, stops at
// the first valid pixel within the radius and at the image border; the
// search range is clipped to both). Sums in direction order 0..7, as there.
__global__ void k_fill_radial_list(const float* __restrict__ din, float* __restrict__ dout,
                                   uint8_t* __restrict__ vout, int W, int H, int radius,
                                   int min_support, long stride, const int* __restrict__ list,
                                   const unsigned* __restrict__ count,
                                   const uint32_t* __restrict__ emap, long fw) {
  const long f = blockIdx.y;
  const unsigned n = count[f];
  const int ww = edge_ww(W);
  const uint32_t* fr = emap + f * fw;
  const uint32_t* K = fr + kEdgeMaps * (long)H * ww;
  const ValidLines L = valid_lines(const_cast<uint32_t*>(fr), W, H);
  const float* dr = din + f * stride;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int pix = list[f * stride + t];
    const int u = pix % W, v = pix / W;
    const int r = radius;
    const int rr = min(r, W - 1 - u), rl = min(r, u), rd = min(r, H - 1 - v), ru = min(r, v);
    const uint32_t* row = K + (long)v * ww;
    const uint32_t* col = L.col + (long)u * L.hw;
    const uint32_t* d1 = L.d1 + ((long)u - v + H - 1) * L.hw;
    const uint32_t* d2 = L.d2 + ((long)u + v) * L.hw;
    int step[8];
    int p;
    p = rr > 0 ? first_set(row, u + 1, u + rr) : -1;
    step[0] = p < 0 ? 0 : p - u;                                          // (1, 0)
    p = rl > 0 ? last_set(row, u - rl, u - 1) : -1;
    step[1] = p < 0 ? 0 : u - p;                                          // (-1, 0)
    p = rd > 0 ? first_set(col, v + 1, v + rd) : -1;
    step[2] = p < 0 ? 0 : p - v;                                          // (0, 1)
    p = ru > 0 ? last_set(col, v - ru, v - 1) : -1;
    step[3] = p < 0 ? 0 : v - p;                                          // (0, -1)
    int m = min(rr, rd);
    p = m > 0 ? first_set(d1, v + 1, v + m) : -1;
    step[4] = p < 0 ? 0 : p - v;                                          // (1, 1)
    m = min(rr, ru);
    p = m > 0 ? last_set(d2, v - m, v - 1) : -1;
    step[5] = p < 0 ? 0 : v - p;                                          // (1, -1)
    m = min(rl, rd);
    p = m > 0 ? first_set(d2, v + 1, v + m) : -1;
    step[6] = p < 0 ? 0 : p - v;                                          // (-1, 1)
    m = min(rl, ru);
    p = m > 0 ? last_set(d1, v - m, v - 1) : -1;
    step[7] = p < 0 ? 0 : v - p;                                          // (-1, -1)
    double wsum = 0.0, vsum = 0.0;
    int support = 0;
#pragma unroll
    for (int dir = 0; dir < 8; ++dir) {
      const int hit = step[dir];
      if (!hit) continue;
      const double len = dir < 4 ? 1.0 : 1.41421356237309504880;  // M_SQRT2
      const long ni = (long)(v + c_dirV[dir] * hit) * W + (u + c_dirU[dir] * hit);
      const double w = __ddiv_rn(1.0, __dmul_rn((double)hit, len));
      wsum = __dadd_rn(wsum, w);
      vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(dr + ni)));
      ++support;
    }
    if (support >= min_support && wsum > 0.0) {
      dout[f * stride + pix] = (float)__ddiv_rn(vsum, wsum);
      vout[f * stride + pix] = 1;
    }
  }
}

// fx (pass 1) holds the disc pass's input as floats: a valid disparity as is,
// an invalid neighbour as a NaN payload that valid disparities are re-coded
// away from (half the tap-load bytes of a double map; measured 5% faster).
constexpr uint32_t kFxInvalid = 0xFFBADBADu;
using fx_t = float;
__device__ __forceinline__ fx_t fx_code(bool ok, float d) {
  return ok ? (__float_as_uint(d) == kFxInvalid ? __uint_as_float(0x7FFFFFFFu) : d)
            : __uint_as_float(kFxInvalid);
}

// Disc fill, pass 1: copy the map through and, for invalid pixels, count the
// valid disc neighbours from per-row prefix counts (exact integers, 2 loads
// per disc row). Pixels that will be filled go to a per-frame list.
__global__ void k_disc_select(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                              float* __restrict__ dout, uint8_t* __restrict__ vout,
                              const int* __restrict__ pcnt, const int* __restrict__ span,
                              int* __restrict__ list, unsigned* __restrict__ count,
                              double* __restrict__ fx, int W, int H, int radius, int min_support,
                              long stride, long pstride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = f * stride + (long)v * W + u;
  const float od = din[i];
  const uint8_t ov = vin[i];
  dout[i] = od;
  vout[i] = ov;
  reinterpret_cast<fx_t*>(fx)[i] = fx_code(ov != 0, od);  // invalid neighbour: marker
  bool listed = false;
  if (!ov && radius > 0) {
    const int* pc = pcnt + f * pstride;
    const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
    int support = 0;
    for (int dv = v0; dv <= v1; ++dv) {
      const int sx = __ldg(span + (dv < 0 ? -dv : dv));
      const int* row = pc + (long)(v + dv) * (W + 1);
      support += __ldg(row + min(W - 1, u + sx) + 1) - __ldg(row + max(0, u - sx));
    }
    // The centre is invalid, so it never contributes (cleanup.cpp:74 skips dd == 0).
    listed = support >= min_support && support > 0;
  }
  warp_append(list + f * stride, count + f, listed, v * W + u);
}

// Disc fill, pass 2: one thread per listed pixel, the reference's raster-order
// double accumulation (cleanup.cpp:71-83) with w = 1/sqrt(dd) from a host
// table ((2R+1)^2 doubles, staged in shared memory). The neighbours come from
// fx = valid ? d : marker (written by pass 1): one 4-byte load per disc pixel
// gives both, an invalid one adds +0.0 to both sums, the loads
// of a row are issued together and only the two FP64 add chains are serial.
__device__ __forceinline__ void disc_acc(double& wsum, double& vsum, double w, float xf) {
  // invalid: x = 0 and w_eff = 0 add +0.0 to both sums, which leaves them
  // bit-identical (neither is ever -0.0: both start at +0.0 and an
  // exactly-zero round-to-nearest sum is +0.0)
  const bool ok = __float_as_uint(xf) != kFxInvalid;
  wsum = __dadd_rn(wsum, ok ? w : 0.0);
  vsum = __dadd_rn(vsum, __dmul_rn(w, (double)(ok ? xf : 0.f)));
}

template <bool SMEM>
__global__ void __launch_bounds__(256)
    k_disc_sum(const fx_t* __restrict__ fx, float* __restrict__ dout, uint8_t* __restrict__ vout,
               const int* __restrict__ list, const unsigned* __restrict__ count,
               const int* __restrict__ span, const double* __restrict__ wtab, int W, int H,
               int radius, long stride, unsigned long long* __restrict__ ctr) {
  extern __shared__ double s_w[];
  const int D = 2 * radius + 1;
  if (SMEM) {
    for (int k = threadIdx.x; k < D * D; k += blockDim.x) s_w[k] = __ldg(wtab + k);
    __syncthreads();
  }
  const long f = blockIdx.y;
  const unsigned n = count[f];
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctr) atomicAdd(ctr + 4, (unsigned long long)n);
  const fx_t* xf = fx + f * stride;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int idx = list[f * stride + t];
    const int v = idx / W, u = idx % W;
    const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
    double wsum = 0.0, vsum = 0.0;
    for (int dv = v0; dv <= v1; ++dv) {
      const int sx = __ldg(span + (dv < 0 ? -dv : dv));
      const int a = max(-sx, -u), b = min(sx, W - 1 - u);
      const fx_t* xr = xf + (long)(v + dv) * W + u;
      const int wo = (dv + radius) * D + radius;
      int du = a;
      for (; du + 3 <= b; du += 4) {
        fx_t x[4];
        double w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          x[k] = __ldg(xr + du + k);
          w[k] = SMEM ? s_w[wo + du + k] : __ldg(wtab + wo + du + k);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) disc_acc(wsum, vsum, w[k], x[k]);
      }
      for (; du <= b; ++du)
        disc_acc(wsum, vsum, SMEM ? s_w[wo + du] : __ldg(wtab + wo + du), __ldg(xr + du));
    }
    if (wsum > 0.0) {
      dout[f * stride + idx] = (float)__ddiv_rn(vsum, wsum);
      vout[f * stride + idx] = 1;
    }
  }
}

static dim3 map_grid(int W, int H, int frames, dim3 b) {
  return dim3((W + b.x - 1) / b.x, (H + b.y - 1) / b.y, frames);
}

void launch_remove_outliers(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                            int W, int H, int radius, double thr, uint32_t* emap, int frames,
                            long stride, cudaStream_t s, float* dout2, uint8_t* vout2, int* list,
                            unsigned* count) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const long fw = edge_map_words(W, H);
  const int ww = edge_ww(W);
  k_edge_words<<<dim3((ww + 3) / 4, (H + kEdgeStrip - 1) / kEdgeStrip, frames), dim3(32, 4), 0,
                 s>>>(din, vin, emap, W, H, thr, stride, fw, dout, dout2);
  k_outlier_words<<<dim3((ww + 31) / 32, (H + 3) / 4, frames), dim3(32, 4), 0, s>>>(
      emap, vout, vout2, W, H, radius, stride, fw, list, count);
}

void launch_fill_radial_list(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                             int W, int H, int radius, int min_support, const int* list,
                             const unsigned* count, const uint32_t* emap, int frames, long stride,
                             cudaStream_t s) {
  (void)vin;  // the validity comes from the outlier pass's bit planes in emap
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const long fw = edge_map_words(W, H);
  const int ww = edge_ww(W);
  k_valid_bits<<<dim3((ww + 2 + 3) / 4, (H + 31) / 32, frames), dim3(32, 4), 0, s>>>(
      const_cast<uint32_t*>(emap), W, H, fw);
  k_fill_radial_list<<<dim3(96, frames), 128, 0, s>>>(din, dout, vout, W, H, radius, min_support,
                                                      stride, list, count, emap, fw);
}

void launch_fill_radial(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                        int W, int H, int radius, int min_support, int frames, long stride,
                        cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  k_fill_radial<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                        min_support, stride);
}

void launch_fill_disc(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                      int W, int H, int radius, int min_support, const double* wtab,
                      const int* span, int* pcnt, int* list, unsigned* count, double* fx,
                      unsigned long long* ctr, int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const long pstride = (long)H * (W + 1);
  launch_row_count(vin, pcnt, W, H, frames, stride, pstride, s);
  cudaMemsetAsync(count, 0, sizeof(unsigned) * frames, s);
  dim3 b(32, 8);
  k_disc_select<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, pcnt, span, list,
                                                        count, fx, W, H, radius, min_support,
                                                        stride, pstride);
  const size_t wbytes = sizeof(double) * (2 * (size_t)radius + 1) * (2 * (size_t)radius + 1);
  if (wbytes <= 40 * 1024)
    k_disc_sum<true><<<dim3(96, frames), 256, wbytes, s>>>(
        reinterpret_cast<const fx_t*>(fx), dout, vout, list, count, span, wtab, W, H, radius,
        stride, ctr);
  else
    k_disc_sum<false><<<dim3(96, frames), 256, 0, s>>>(
        reinterpret_cast<const fx_t*>(fx), dout, vout, list, count, span, wtab, W, H, radius,
        stride, ctr);
}

}  // namespace ssb
