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

// Invalid-neighbour marker in fx: the smallest denormal (low word 1) — a double
// converted from a float always has its low 29 mantissa bits zero, so no
// disparity (not even NaN/inf) carries it, and 0 * marker = +0.
constexpr int kInvalidLo = 1;

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
  fx[i] = ov ? (double)od : __hiloint2double(0, kInvalidLo);  // invalid neighbour
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
// fx = valid ? double(d) : marker (written by pass 1): one load per disc pixel
// gives both, an invalid one adds +0.0 to both sums, the loads
// of a row are issued together and only the two FP64 add chains are serial.
__device__ __forceinline__ void disc_acc(double& wsum, double& vsum, double w, double x) {
  // invalid: w_eff = 0 adds +0.0 to both sums, which leaves them bit-identical
  // (neither is ever -0.0: both start at +0.0 and an exactly-zero
  // round-to-nearest sum is +0.0)
  const double we = __double2loint(x) != kInvalidLo ? w : 0.0;
  wsum = __dadd_rn(wsum, we);
  vsum = __dadd_rn(vsum, __dmul_rn(we, x));
}

template <bool SMEM>
__global__ void __launch_bounds__(256)
    k_disc_sum(const double* __restrict__ fx, float* __restrict__ dout, uint8_t* __restrict__ vout,
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
  const double* xf = fx + f * stride;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int idx = list[f * stride + t];
    const int v = idx / W, u = idx % W;
    const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
    double wsum = 0.0, vsum = 0.0;
    for (int dv = v0; dv <= v1; ++dv) {
      const int sx = __ldg(span + (dv < 0 ? -dv : dv));
      const int a = max(-sx, -u), b = min(sx, W - 1 - u);
      const double* xr = xf + (long)(v + dv) * W + u;
      const int wo = (dv + radius) * D + radius;
      int du = a;
      for (; du + 3 <= b; du += 4) {
        double x[4], w[4];
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
    k_disc_sum<true><<<dim3(96, frames), 256, wbytes, s>>>(fx, dout, vout, list, count, span, wtab,
                                                         W, H, radius, stride, ctr);
  else
    k_disc_sum<false><<<dim3(96, frames), 256, 0, s>>>(fx, dout, vout, list, count, span, wtab, W,
                                                     H, radius, stride, ctr);
}

}  // namespace ssb
