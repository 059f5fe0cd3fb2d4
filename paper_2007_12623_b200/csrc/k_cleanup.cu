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

#include "ss_internal.cuh"

namespace ssb {

__constant__ int c_dirU[8] = {1, -1, 0, 0, 1, 1, -1, -1};
__constant__ int c_dirV[8] = {0, 0, 1, -1, 1, -1, 1, -1};

__global__ void k_remove_outliers(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                                  float* __restrict__ dout, uint8_t* __restrict__ vout, int W,
                                  int H, int radius, double thr, long stride) {
  const long f = blockIdx.z;
  din += f * stride;
  vin += f * stride;
  dout += f * stride;
  vout += f * stride;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = (long)v * W + u;
  const float cd = din[i];
  const uint8_t cv = vin[i];
  dout[i] = cd;
  if (!cv) {
    vout[i] = 0;
    return;
  }
  bool keep = false;
  for (int dir = 0; dir < 8 && !keep; ++dir) {
    const int du = c_dirU[dir], dv = c_dirV[dir];
    // Rays that leave the image never qualify: check the far end first.
    const int eu = u + du * radius, ev = v + dv * radius;
    if (eu < 0 || eu >= W || ev < 0 || ev >= H) continue;
    double prev = cd;
    bool ok = true;
    for (int step = 1; step <= radius; ++step) {
      const long ni = (long)(v + dv * step) * W + (u + du * step);
      if (!__ldg(vin + ni)) {
        ok = false;
        break;
      }
      const double cur = __ldg(din + ni);
      if (fabs(cur - prev) > thr) {
        ok = false;
        break;
      }
      prev = cur;
    }
    keep = ok;
  }
  vout[i] = keep ? 1 : 0;
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
  float od = din[i];
  uint8_t ov = vin[i];
  if (!ov) {
    double wsum = 0.0, vsum = 0.0;
    int support = 0;
    for (int dir = 0; dir < 8; ++dir) {
      const double len = dir < 4 ? 1.0 : 1.41421356237309504880;  // M_SQRT2
      const int du = c_dirU[dir], dv = c_dirV[dir];
      for (int step = 1; step <= radius; ++step) {
        const int nu = u + du * step, nv = v + dv * step;
        if (nu < 0 || nu >= W || nv < 0 || nv >= H) break;
        const long ni = (long)nv * W + nu;
        if (!__ldg(vin + ni)) continue;
        const double w = __ddiv_rn(1.0, __dmul_rn((double)step, len));
        wsum = __dadd_rn(wsum, w);
        vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(din + ni)));
        ++support;
        break;
      }
    }
    if (support >= min_support && wsum > 0.0) {
      od = (float)__ddiv_rn(vsum, wsum);
      ov = 1;
    }
  }
  dout[i] = od;
  vout[i] = ov;
}

// Disc fill, pass 1: copy the map through and, for invalid pixels, count the
// valid disc neighbours from per-row prefix counts (exact integers, 2 loads
// per disc row). Pixels that will be filled go to a per-frame list.
__global__ void k_disc_select(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                              float* __restrict__ dout, uint8_t* __restrict__ vout,
                              const int* __restrict__ pcnt, const int* __restrict__ span,
                              int* __restrict__ list, unsigned* __restrict__ count, int W, int H,
                              int radius, int min_support, long stride, long pstride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = f * stride + (long)v * W + u;
  const float od = din[i];
  const uint8_t ov = vin[i];
  dout[i] = od;
  vout[i] = ov;
  if (ov || radius <= 0) return;
  const int* pc = pcnt + f * pstride;
  const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
  int support = 0;
  for (int dv = v0; dv <= v1; ++dv) {
    const int sx = __ldg(span + (dv < 0 ? -dv : dv));
    const int* row = pc + (long)(v + dv) * (W + 1);
    support += __ldg(row + min(W - 1, u + sx) + 1) - __ldg(row + max(0, u - sx));
  }
  // The centre is invalid, so it never contributes (cleanup.cpp:74 skips dd == 0).
  if (support >= min_support && support > 0)
    list[f * stride + atomicAdd(count + f, 1u)] = (int)((long)v * W + u);
}

// Disc fill, pass 2: one thread per listed pixel, the reference's raster-order
// double accumulation (cleanup.cpp:71-83), w = 1/sqrt(dd) from a host table.
__global__ void k_disc_sum(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                           float* __restrict__ dout, uint8_t* __restrict__ vout,
                           const int* __restrict__ list, const unsigned* __restrict__ count,
                           const int* __restrict__ span, const double* __restrict__ wtab, int W,
                           int H, int radius, long stride) {
  const long f = blockIdx.y;
  const unsigned n = count[f];
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int idx = list[f * stride + t];
    const int v = idx / W, u = idx % W;
    const uint8_t* vf = vin + f * stride;
    const float* df = din + f * stride;
    const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
    double wsum = 0.0, vsum = 0.0;
    for (int dv = v0; dv <= v1; ++dv) {
      const int sx = __ldg(span + (dv < 0 ? -dv : dv));
      const int a = max(-sx, -u), b = min(sx, W - 1 - u);
      const uint8_t* row = vf + (long)(v + dv) * W + u;
      const float* drow = df + (long)(v + dv) * W + u;
      const int dv2 = dv * dv;
      for (int du = a; du <= b; ++du) {
        if (!__ldg(row + du)) continue;
        const double w = __ldg(wtab + du * du + dv2);
        wsum = __dadd_rn(wsum, w);
        vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(drow + du)));
      }
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
                            int W, int H, int radius, double thr, int frames, long stride,
                            cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  k_remove_outliers<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                            thr, stride);
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
                      const int* span, int* pcnt, int* list, unsigned* count, int frames,
                      long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const long pstride = (long)H * (W + 1);
  launch_row_count(vin, pcnt, W, H, frames, stride, pstride, s);
  cudaMemsetAsync(count, 0, sizeof(unsigned) * frames, s);
  dim3 b(32, 8);
  k_disc_select<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, pcnt, span, list,
                                                        count, W, H, radius, min_support, stride,
                                                        pstride);
  k_disc_sum<<<dim3(96, frames), 256, 0, s>>>(din, vin, dout, vout, list, count, span, wtab, W,
                                             H, radius, stride);
}

}  // namespace ssb
