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
//   k_fill_disc        cleanup.cpp:69-84 — all valid pixels of the radius-R
//                      disc in raster order, w = 1/sqrt(dd) from a table built
//                      with the same IEEE double ops on the host. The support
//                      count (integer) is taken first; the FP64 sums run only
//                      for pixels that will be filled.
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

__global__ void k_fill_disc(const float* __restrict__ din, const uint8_t* __restrict__ vin,
                            float* __restrict__ dout, uint8_t* __restrict__ vout, int W, int H,
                            int radius, int min_support, const double* __restrict__ wtab,
                            long stride) {
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
    const int r2 = radius * radius;
    const int v0 = max(-radius, -v), v1 = min(radius, H - 1 - v);
    // Pass 1: integer support count (decides whether a fill happens).
    int support = 0;
    for (int dv = v0; dv <= v1; ++dv) {
      const int span = (int)floor(sqrt((double)(r2 - dv * dv)));
      const int a = max(-span, -u), b = min(span, W - 1 - u);
      const uint8_t* row = vin + (long)(v + dv) * W + u;
      for (int du = a; du <= b; ++du) support += __ldg(row + du);
    }
    support -= 0;  // the centre is invalid, so it never counted
    if (support >= min_support && support > 0) {
      // Pass 2: reference-order double sums (raster dv, du).
      double wsum = 0.0, vsum = 0.0;
      for (int dv = v0; dv <= v1; ++dv) {
        const int span = (int)floor(sqrt((double)(r2 - dv * dv)));
        const int a = max(-span, -u), b = min(span, W - 1 - u);
        const uint8_t* row = vin + (long)(v + dv) * W + u;
        const float* drow = din + (long)(v + dv) * W + u;
        for (int du = a; du <= b; ++du) {
          if (!__ldg(row + du)) continue;
          const double w = wtab[du * du + dv * dv];
          wsum = __dadd_rn(wsum, w);
          vsum = __dadd_rn(vsum, __dmul_rn(w, (double)__ldg(drow + du)));
        }
      }
      if (wsum > 0.0) {
        od = (float)__ddiv_rn(vsum, wsum);
        ov = 1;
      }
    }
  }
  dout[i] = od;
  vout[i] = ov;
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
                      int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  k_fill_disc<<<map_grid(W, H, frames, b), b, 0, s>>>(din, vin, dout, vout, W, H, radius,
                                                      min_support, wtab, stride);
}

}  // namespace ssb
