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
//   k_disc_sum_cert    per-row prefix counts (exact integers); only pixels that
//                      will be filled enter a compacted list; 8 lanes per
//                      listed pixel sum the radius-R disc in FP64 (w = 1/sqrt(dd)
//                      from a table built with the same IEEE ops on the host)
//                      and certify that the result rounds to the reference's
//                      float, else recompute it in the reference's raster order.
// All maps of a frame stay L2-resident (5 B/pixel); these passes are a few
// percent of the frame and latency-, not bandwidth-bound.
#include <math.h>

#include <algorithm>

#include "ss_internal.cuh"

namespace ssb {


__constant__ int c_dirU[8] = {1, -1, 0, 0, 1, 1, -1, -1};
__constant__ int c_dirV[8] = {0, 0, 1, -1, 1, -1, 1, -1};

// Outlier rays via smooth-edge bitmaps. A ray from a valid pixel p in
// direction e passes iff its far end is inside the image and every step q ->
// q + e (q = p, p + e, ...) joins two valid pixels with |d(q+e) - d(q)| <= thr
// (the reference's double comparison). That edge predicate is symmetric, so
// four bitmaps hold it for all eight directions — E_h (q -> q+(1,0)) by rows,
// E_v ((0,1)) by columns, E_d1 ((1,1)) and E_d2 ((1,-1)) by diagonals — laid
// out so that every ray is a run of consecutive bits, and the ray test is
// "r consecutive ones" on one or two words.
namespace {
struct EdgeMaps {
  uint32_t *bh, *bv, *bd1, *bd2;
  int lw, lh;  // words per row line (E_h) / per column or diagonal line
};
__host__ __device__ inline EdgeMaps edge_maps(uint32_t* base, int W, int H) {
  EdgeMaps m;
  m.lw = (W + 31) / 32 + 1;  // +1: a two-word read never leaves the line
  m.lh = (H + 31) / 32 + 1;
  m.bh = base;
  m.bv = m.bh + (long)H * m.lw;
  m.bd1 = m.bv + (long)W * m.lh;
  m.bd2 = m.bd1 + (long)(W + H - 1) * m.lh;
  return m;
}
// bits [p, p + r) of a line all set
__device__ __forceinline__ bool run_ok(const uint32_t* __restrict__ line, int p, int r) {
  while (r > 0) {
    const int wi = p >> 5, b = p & 31;
    const uint32_t x = __funnelshift_r(__ldg(line + wi), __ldg(line + wi + 1), b);
    const int n = r < 32 ? r : 32;
    const uint32_t m = n == 32 ? 0xFFFFFFFFu : (1u << n) - 1u;
    if ((x & m) != m) return false;
    p += n;
    r -= n;
  }
  return true;
}
}  // namespace

__global__ void __launch_bounds__(256)
    k_edge_bits(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                uint32_t* __restrict__ emap, int W, int H, double thr, long stride, long fw) {
  __shared__ double td[34][33];    // rows v0-1 .. v0+32, columns u0 .. u0+32 (widened once)
  __shared__ uint32_t tv[34][33];  // validity (words: no byte bank conflicts)
  __shared__ uint32_t eb[32][34];  // per pixel: bit0 E_h, bit1 E_v, bit2 E_d1, bit3 E_d2
  const long f = blockIdx.z;
  const int u0 = blockIdx.x * 32, v0 = blockIdx.y * 32;
  const int lane = threadIdx.x, wy = threadIdx.y;
  // cells (r, c): c = lane for r = wy + 8k (k < 5), plus column 32 for the
  // threads 0..33 — every load issued before the first store
  constexpr int kCells = 6;
  float xs[kCells];
  uint8_t ms[kCells];
#pragma unroll
  for (int k = 0; k < kCells; ++k) {
    const int tid = wy * 32 + lane;
    const int r = k < 5 ? wy + 8 * k : tid, c = k < 5 ? lane : 32;
    const int v = v0 - 1 + r, u = u0 + c;
    xs[k] = 0.f;
    ms[k] = 0;
    if (r < 34 && v >= 0 && v < H && u < W) {
      const long i = f * stride + (long)v * W + u;
      ms[k] = vin[i];
      xs[k] = din[i];
    }
  }
#pragma unroll
  for (int k = 0; k < kCells; ++k) {
    const int tid = wy * 32 + lane;
    const int r = k < 5 ? wy + 8 * k : tid, c = k < 5 ? lane : 32;
    if (r < 34) {
      td[r][c] = (double)xs[k];
      tv[r][c] = ms[k] ? 1u : 0u;
    }
  }
  __syncthreads();
  // smooth edge from cell (r, c) to (r2, c2): both valid, |d2 - d| <= thr in
  // double (cleanup.cpp:29-30; NaN compares false, as there)
  auto E = [&](int r, int c, int r2, int c2) -> unsigned {
    return (tv[r][c] & tv[r2][c2]) && !(fabs(td[r2][c2] - td[r][c]) > thr)
               ? 1u
               : 0u;
  };
  for (int l = wy; l < 32; l += 8) {
    const int r = l + 1, c = lane;
    eb[l][lane] = E(r, c, r, c + 1) | (E(r, c, r + 1, c) << 1) | (E(r, c, r + 1, c + 1) << 2) |
                  (E(r, c, r - 1, c + 1) << 3);
  }
  __syncthreads();
  const EdgeMaps M = edge_maps(emap + f * fw, W, H);
  for (int l = wy; l < 32; l += 8) {  // E_h: lanes = columns, one word per row
    const unsigned m = __ballot_sync(0xFFFFFFFFu, eb[l][lane] & 1u);
    if (lane == 0 && v0 + l < H) M.bh[(long)(v0 + l) * M.lw + (u0 >> 5)] = m;
  }
  for (int c = wy; c < 32; c += 8) {  // E_v: lanes = rows, one word per column
    const unsigned m = __ballot_sync(0xFFFFFFFFu, (eb[lane][c] >> 1) & 1u);
    if (lane == 0 && u0 + c < W) M.bv[(long)(u0 + c) * M.lh + (v0 >> 5)] = m;
  }
  // diagonals: lanes = rows; a tile holds a partial word of 63 diagonals of
  // each kind, OR-ed into the (zeroed) maps.
  for (int dd = wy; dd < 63; dd += 8) {
    {  // E_d1 (1,1): diagonal u - v = const, column c = lane + delta
      const int delta = dd - 31, c = lane + delta;
      const bool e = c >= 0 && c < 32 && ((eb[lane][c] >> 2) & 1u);
      const unsigned m = __ballot_sync(0xFFFFFFFFu, e);
      if (lane == 0 && m) atomicOr(M.bd1 + ((long)(u0 - v0 + delta) + H - 1) * M.lh + (v0 >> 5), m);
    }
    {  // E_d2 (1,-1): diagonal u + v = const, column c = dd - lane
      const int c = dd - lane;
      const bool e = c >= 0 && c < 32 && ((eb[lane][c] >> 3) & 1u);
      const unsigned m = __ballot_sync(0xFFFFFFFFu, e);
      if (lane == 0 && m) atomicOr(M.bd2 + ((long)u0 + v0 + dd) * M.lh + (v0 >> 5), m);
    }
  }
}

// dout2/vout2 (optional): a second copy of the result (the radial fill's
// output buffer, so that fill only writes the pixels it fills); list/count
// (optional): per-frame list of the invalid output pixels (warp-aggregated
// appends: ~5% of the pixels, one counter per frame).
// In place allowed (vout == vin, dout == NULL: each thread reads only its own
// pixel of din / vin, before writing it), hence no __restrict__ on those.
__global__ void k_remove_outliers(const float* din, const uint8_t* vin, float* dout,
                                  uint8_t* vout, int W, int H, int r,
                                  const uint32_t* __restrict__ emap, long stride, long fw,
                                  float* __restrict__ dout2, uint8_t* __restrict__ vout2,
                                  int* __restrict__ list, unsigned* __restrict__ count) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = f * stride + (long)v * W + u;
  const float d0 = din[i];
  if (dout) dout[i] = d0;
  if (dout2) dout2[i] = d0;
  bool keep = false;
  if (vin[i]) {
    const EdgeMaps M = edge_maps(const_cast<uint32_t*>(emap) + f * fw, W, H);
    keep = r <= 0;  // no steps: every ray is smooth (cleanup.cpp:21-33)
    const uint32_t* row = M.bh + (long)v * M.lw;
    const uint32_t* col = M.bv + (long)u * M.lh;
    const uint32_t* d1 = M.bd1 + ((long)u - v + H - 1) * M.lh;
    const uint32_t* d2 = M.bd2 + ((long)u + v) * M.lh;
    if (!keep && u + r < W) keep = run_ok(row, u, r);                      // (1, 0)
    if (!keep && u - r >= 0) keep = run_ok(row, u - r, r);                 // (-1, 0)
    if (!keep && v + r < H) keep = run_ok(col, v, r);                      // (0, 1)
    if (!keep && v - r >= 0) keep = run_ok(col, v - r, r);                 // (0, -1)
    if (!keep && u + r < W && v + r < H) keep = run_ok(d1, v, r);          // (1, 1)
    if (!keep && u + r < W && v - r >= 0) keep = run_ok(d2, v - r + 1, r); // (1, -1)
    if (!keep && u - r >= 0 && v + r < H) keep = run_ok(d2, v + 1, r);     // (-1, 1)
    if (!keep && u - r >= 0 && v - r >= 0) keep = run_ok(d1, v - r, r);   // (-1, -1)
  }
  vout[i] = keep ? 1 : 0;
  if (vout2) vout2[i] = keep ? 1 : 0;
  if (list) warp_append(list + f * stride, count + f, !keep, v * W + u);
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

// Chain variant: dout/vout already hold the input map (k_remove_outliers'
// second copy); one thread per listed invalid pixel, no idle lanes.
__global__ void k_fill_radial_list(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                                   float* __restrict__ dout, uint8_t* __restrict__ vout, int W,
                                   int H, int radius, int min_support, long stride,
                                   const int* __restrict__ list,
                                   const unsigned* __restrict__ count) {
  const long f = blockIdx.y;
  const unsigned n = count[f];
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int pix = list[f * stride + t];
    radial_fill_pixel(din + f * stride, vin + f * stride, dout + f * stride, vout + f * stride,
                      W, H, pix % W, pix / W, radius, min_support);
  }
}

// Disc fill, pass 1: copy the map through and, for invalid pixels, count the
// valid disc neighbours from per-row prefix counts (exact integers, 2 loads
// per disc row). Pixels that will be filled go to a per-frame list. fx gets
// the map as doubles in a layout padded by R on every side, invalid pixels
// and the padding holding the marker -0.0 (so w * x adds -0.0, which leaves a
// sum unchanged, and every disc tap of every pixel is in bounds); meta[2f+1]
// = 1 if a valid pixel holds a value whose high word is the marker's (only
// -0.0 converts to one: that frame then takes the exact path throughout; the
// chain never produces one).
constexpr int kMarkHi = (int)0x80000000;  // high word of -0.0

__host__ __device__ inline long disc_pitch(int W, int R) { return (long)W + 2 * R; }
__host__ __device__ inline long disc_frame(int W, int H, int R) {
  return disc_pitch(W, R) * ((long)H + 2 * R);
}

__global__ void __launch_bounds__(256)
    k_disc_select(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                  float* __restrict__ dout, uint8_t* __restrict__ vout,
                  const int* __restrict__ pcnt, const int* __restrict__ span,
                  int* __restrict__ list, unsigned* __restrict__ count, double* __restrict__ fx,
                  unsigned* __restrict__ meta, int W, int H, int radius, int min_support,
                  long stride, long pstride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  const long P = disc_pitch(W, radius);
  double* xf = fx + f * disc_frame(W, H, radius) + (long)radius * P + radius;
  unsigned clash = 0;
  bool listed = false;
  if (u < W && v < H) {
    const long i = f * stride + (long)v * W + u;
    const float od = din[i];
    const uint8_t ov = vin[i];
    dout[i] = od;
    vout[i] = ov;
    const double xd = (double)od;
    xf[(long)v * P + u] = ov ? xd : -0.0;
    if (ov) {
      clash = __double2hiint(xd) == kMarkHi;
    } else if (radius > 0) {
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
  }
  warp_append(list + f * stride, count + f, listed, v * W + u);
  if (__any_sync(0xFFFFFFFFu, clash) && (threadIdx.x & 31) == 0) atomicOr(meta + 2 * f + 1, 1u);
}

// The reference's raster-order double accumulation (cleanup.cpp:71-83) for
// one pixel, from the input map itself: the exact path.
__device__ double disc_fill_exact(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                                  const int* __restrict__ span, const double* __restrict__ wtab,
                                  int W, int H, int u, int v, int radius, double& wsum) {
  const int D = 2 * radius + 1;
  const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
  double vsum = 0.0;
  wsum = 0.0;
  for (int dv = v0; dv <= v1; ++dv) {
    const int sx = __ldg(span + (dv < 0 ? -dv : dv));
    const int a = max(-sx, -u), b = min(sx, W - 1 - u);
    const long r = (long)(v + dv) * W + u;
    const double* wr = wtab + (dv + radius) * D + radius;
    for (int du = a; du <= b; ++du) {
      if (du == 0 && dv == 0) continue;
      if (!__ldg(vin + r + du)) continue;
      const double w = __ldg(wr + du);
      wsum = __dadd_rn(wsum, w);
      vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(din + r + du)));
    }
  }
  return vsum;
}

// Disc fill, pass 2 (certified, parallel): one warp per listed pixel. The
// disc's taps (centre excluded) are a table in raster order in shared memory
// (padded-layout offset, weight); lane l sums taps l, l + 32, ..., so a warp
// load reads consecutive pixels of one or two rows, and the 32 partial sums
// are combined by shuffles. This reassociates the reference's raster-order
// sums (cleanup.cpp:71-83). Both add the SAME terms — table weights w and
// products fl(w x) — so each is within gamma_{n-1} sum|term| of the exact
// sum and they differ by at most 4 n u sum|term| <= 4 n u wsum max|d|
// (n = taps, u = 2^-53). The reference's fl(vsum / wsum) therefore lies in
// [q_lo, q_hi], computed with directed rounding; when both ends round to the
// same float — the output type — that float is the reference's result.
// Otherwise (~1 pixel per frame), and in a frame where a valid pixel holds
// the marker, lane 0 recomputes the pixel in the reference's exact order. The
// weight sum is fma(w, m, wsum) with m in {0, 1}: w m is exact, so it equals
// the masked add.
constexpr int kDiscMaxR = 31;  // (2R+1)^2 <= 3969 taps in shared memory
__host__ __device__ inline int disc_tab_cap(int R) { return ((2 * R + 1) * (2 * R + 1) + 31) & ~31; }

__global__ void __launch_bounds__(256, 4)
    k_disc_sum_cert(const double* __restrict__ fx, const float* __restrict__ din,
                    const uint8_t* __restrict__ vin, float* __restrict__ dout,
                    uint8_t* __restrict__ vout, const int* __restrict__ list,
                    const unsigned* __restrict__ count, const unsigned* __restrict__ meta,
                    const int* __restrict__ span, const double* __restrict__ wtab, int W, int H,
                    int radius, long stride, unsigned long long* __restrict__ ctr) {
  extern __shared__ double s_tw[];  // [cap] weights, then [cap] byte offsets
  const int D = 2 * radius + 1;
  const long P = disc_pitch(W, radius);
  int* s_off = reinterpret_cast<int*>(s_tw + disc_tab_cap(radius));
  __shared__ int s_row0[2 * kDiscMaxR + 2];
  if (threadIdx.x == 0) {
    int n = 0;
    for (int dv = -radius; dv <= radius; ++dv) {
      s_row0[dv + radius] = n;
      n += 2 * __ldg(span + (dv < 0 ? -dv : dv)) + 1 - (dv == 0 ? 1 : 0);
    }
    s_row0[D] = n;
  }
  __syncthreads();
  const int taps = s_row0[D];
  const int taps32 = (taps + 31) & ~31;  // padded to whole warp passes: w = 0, offset 0
  // raster-order tap table (dv, then du ascending), centre excluded; byte
  // offsets into the padded map
  for (int k = threadIdx.x; k < D * D; k += blockDim.x) {
    const int dv = k / D - radius, du = k % D - radius;
    const int sx = __ldg(span + (dv < 0 ? -dv : dv));
    if ((du < 0 ? -du : du) > sx || (du == 0 && dv == 0)) continue;
    const int t = s_row0[dv + radius] + du + sx - (dv == 0 && du > 0 ? 1 : 0);
    s_tw[t] = __ldg(wtab + k);
    s_off[t] = (int)((dv * P + du) * (long)sizeof(double));
  }
  for (int t = taps + threadIdx.x; t < taps32; t += blockDim.x) {
    s_tw[t] = 0.0;
    s_off[t] = 0;  // the (invalid) centre: adds w * -0.0 and 0 weight
  }
  __syncthreads();
  const long f = blockIdx.y;
  const unsigned n = count[f];
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctr) atomicAdd(ctr + 4, (unsigned long long)n);
  const bool exact_all = meta[2 * f + 1] != 0;
  const int lane = threadIdx.x & 31;
  const unsigned wpb = blockDim.x >> 5;
  const double c4nu = 4.0 * (double)taps * 0x1p-53;
  const double* xf = fx + f * disc_frame(W, H, radius) + (long)radius * P + radius;
  for (unsigned t = blockIdx.x * wpb + (threadIdx.x >> 5); t < n; t += gridDim.x * wpb) {
    const int idx = list[f * stride + t];
    const int v = idx / W, u = idx % W;
    bool done = false;
    float out = 0.f;
    if (!exact_all) {
      const char* xc = reinterpret_cast<const char*>(xf + (long)v * P + u);
      double ws = 0.0, vs = 0.0, as = 0.0;
      // batches of 8 taps per lane: all 8 loads in flight before the first use
      for (int k0 = lane; k0 < taps32; k0 += 8 * 32) {
        double xs[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = k0 + 32 * j;
          xs[j] = k < taps32 ? __ldg(reinterpret_cast<const double*>(xc + s_off[k])) : -0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = k0 + 32 * j;
          const double w = k < taps32 ? s_tw[k] : 0.0;
          const double p = __dmul_rn(w, xs[j]);
          ws = __fma_rn(w, __double2hiint(xs[j]) != kMarkHi ? 1.0 : 0.0, ws);
          vs = __dadd_rn(vs, p);
          as = __dadd_rn(as, fabs(p));
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ws = __dadd_rn(ws, __shfl_xor_sync(0xFFFFFFFFu, ws, off));
        vs = __dadd_rn(vs, __shfl_xor_sync(0xFFFFFFFFu, vs, off));
        as = __dadd_rn(as, __shfl_xor_sync(0xFFFFFFFFu, as, off));
      }
      // both sums are within gamma_{n-1} * sum|p| of exact; the computed
      // sum|p| (as) is within gamma_n of its own exact value: 2.02 n u as
      // bounds the difference, 4 n u as with margin
      const double ev = __dmul_ru(c4nu, as);
      const double ew = __dmul_ru(c4nu, ws);
      const double nlo = __dsub_rd(vs, ev), nhi = __dadd_ru(vs, ev);
      const double dlo = __dsub_rd(ws, ew), dhi = __dadd_ru(ws, ew);
      if (dlo > 0.0) {
        const double qlo = __ddiv_rd(nlo, nlo >= 0.0 ? dhi : dlo);
        const double qhi = __ddiv_ru(nhi, nhi >= 0.0 ? dlo : dhi);
        const float flo = __double2float_rn(qlo), fhi = __double2float_rn(qhi);
        if (__float_as_uint(flo) == __float_as_uint(fhi) && !isnan(flo)) {
          done = true;
          out = flo;
        }
      }
    }
    if (lane == 0) {
      if (!done) {
        double ws;
        const double vs = disc_fill_exact(din + f * stride, vin + f * stride, span, wtab, W, H,
                                          u, v, radius, ws);
        if (ctr) atomicAdd(ctr + 3, 1ull);
        done = ws > 0.0;
        out = (float)__ddiv_rn(vs, ws);
      }
      if (done) {
        dout[f * stride + idx] = out;
        vout[f * stride + idx] = 1;
      }
    }
  }
}

// Generic disc fill pass 2 (weights table too large for shared memory): one
// thread per listed pixel in the exact order.
__global__ void __launch_bounds__(256)
    k_disc_sum_serial(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                      float* __restrict__ dout, uint8_t* __restrict__ vout,
                      const int* __restrict__ list, const unsigned* __restrict__ count,
                      const int* __restrict__ span, const double* __restrict__ wtab, int W, int H,
                      int radius, long stride) {
  const long f = blockIdx.y;
  const unsigned n = count[f];
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int idx = list[f * stride + t];
    double ws;
    const double vs = disc_fill_exact(din + f * stride, vin + f * stride, span, wtab, W, H,
                                      idx % W, idx / W, radius, ws);
    if (ws > 0.0) {
      dout[f * stride + idx] = (float)__ddiv_rn(vs, ws);
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
  if (radius > 0) {
    cudaMemsetAsync(emap, 0, sizeof(uint32_t) * fw * frames, s);
    k_edge_bits<<<dim3((W + 31) / 32, (H + 31) / 32, frames), dim3(32, 8), 0, s>>>(
        din, vin, emap, W, H, thr, stride, fw);
  }
  dim3 b(32, 8);
  k_remove_outliers<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                            emap, stride, fw, dout2, vout2, list,
                                                            count);
}

void launch_fill_radial_list(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                             int W, int H, int radius, int min_support, const int* list,
                             const unsigned* count, int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_fill_radial_list<<<dim3(96, frames), 128, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                      min_support, stride, list, count);
}

void launch_fill_radial(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                        int W, int H, int radius, int min_support, int frames, long stride,
                        cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  k_fill_radial<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                        min_support, stride);
}

// The R-wide frame of fx around the image: the marker (a disc tap there adds
// nothing), written per call (fx is shared by every geometry of the ctx).
__global__ void __launch_bounds__(256) k_disc_pad(double* __restrict__ fx, int W, int H, int R) {
  const long P = disc_pitch(W, R);
  const long top = (long)R * P;                 // rows -R..-1 (and H..H+R-1 below)
  const long side = (long)H * 2 * R;            // R columns left and right of each row
  long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double* xf = fx + blockIdx.y * disc_frame(W, H, R);
  long y, x;
  if (k < top) {
    y = k / P;
    x = k % P;
  } else if ((k -= top) < top) {
    y = R + H + k / P;
    x = k % P;
  } else if ((k -= top) < side) {
    y = R + k / (2 * R);
    x = k % (2 * R);
    if (x >= R) x += W;
  } else {
    return;
  }
  xf[y * P + x] = -0.0;
}

long disc_fx_elems(int W, int H, int radius) { return disc_frame(W, H, std::max(radius, 0)); }

void launch_fill_disc(const float* din, const uint8_t* vin, float* dout, uint8_t* vout,
                      int W, int H, int radius, int min_support, const double* wtab,
                      const int* span, int* pcnt, int* list, unsigned* count, double* fx,
                      unsigned* meta, unsigned long long* ctr, int frames, long stride,
                      int n_sm, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const long pstride = (long)H * (W + 1);
  launch_row_count(vin, pcnt, W, H, frames, stride, pstride, s);
  cudaMemsetAsync(count, 0, sizeof(unsigned) * frames, s);
  cudaMemsetAsync(meta, 0, sizeof(unsigned) * 2 * frames, s);
  dim3 b(32, 8);
  k_disc_select<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, pcnt, span, list,
                                                        count, fx, meta, W, H, std::max(radius, 0),
                                                        min_support, stride, pstride);
  // persistent grid: ~4 blocks per SM over all frames; each block's warps
  // stride through their frame's device-side list
  const int gx = std::max(1, 4 * n_sm / frames);
  const long D = 2L * std::max(radius, 0) + 1;
  if (radius <= kDiscMaxR) {
    k_disc_pad<<<dim3((unsigned)((disc_frame(W, H, radius) - (long)W * H + 255) / 256), frames), 256,
                 0, s>>>(fx, W, H, std::max(radius, 0));
    const size_t smem = disc_tab_cap(std::max(radius, 0)) * (sizeof(double) + sizeof(int));
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_disc_sum_cert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_disc_sum_cert<<<dim3(gx, frames), 256, smem, s>>>(fx, din, vin, dout, vout, list, count,
                                                         meta, span, wtab, W, H,
                                                         std::max(radius, 0), stride, ctr);
  } else {
    k_disc_sum_serial<<<dim3(gx, frames), 256, 0, s>>>(din, vin, dout, vout, list, count, span,
                                                       wtab, W, H, radius, stride);
  }
}

}  // namespace ssb
