// Disparity -> oriented point cloud (disparity_to_cloud, cloud.cpp:14-94).
//
//   k_cloud_count / k_cloud_offsets / k_cloud_index
//       deterministic raster-order compaction (cloud.cpp:23-39): a point per
//       valid pixel with d > 1e-6, numbered in raster order — block counts,
//       a per-frame scan of the block counts, then a ballot/popc scan inside
//       each block. Bit-identical to the serial loop.
//   k_cloud_points
//       z = (fx b) / d, x = (z (u - cx)) / fx, y = (z (v - cy)) / fy in FP64,
//       the reference's association order -> bit-identical points; colour
//       from the left RGB image when (u, v) is inside it.
//   k_cloud_normals
//       7x7 neighbourhood (kNormalWindowHalf = 3) of existing points, mean and
//       covariance accumulated in raster order in FP64, closed-form symmetric
//       3x3 eigen-decomposition (trigonometric eigenvalues, cross-product
//       eigenvector) instead of Eigen's SelfAdjointEigenSolver (cloud.cpp:78):
//       agreement is within tolerance, not bitwise. Same
//       acceptance rule (lambda1 > 1e-9 max(1, lambda2)), same -p/|p|
//       fallback and camera-facing flip (cloud.cpp:81-89).
#include <math.h>

#include "ss_internal.cuh"

namespace ssb {

constexpr int kCloudBlock = 1024;

__device__ __forceinline__ bool has_point(const float* disp, const uint8_t* valid, long i) {
  return valid[i] && ((double)disp[i] > 1e-6);
}

__global__ void k_cloud_count(const float* __restrict__ disp, const uint8_t* __restrict__ valid,
                              int* __restrict__ block_sums, long n, int nblocks, long stride) {
  const long f = blockIdx.y;
  disp += f * stride;
  valid += f * stride;
  const long i = (long)blockIdx.x * kCloudBlock + threadIdx.x;
  const bool p = i < n && has_point(disp, valid, i);
  const int wc = __popc(__ballot_sync(0xffffffffu, p));
  __shared__ int ws[kCloudBlock / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = wc;
  __syncthreads();
  if (threadIdx.x < 32) {
    int x = ws[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (threadIdx.x == 0) block_sums[f * nblocks + blockIdx.x] = x;
  }
}

// One block per frame: exclusive scan of the block counts, total -> n_points.
__global__ void k_cloud_offsets(int* __restrict__ block_sums, int* __restrict__ n_points,
                                int nblocks) {
  const long f = blockIdx.x;
  int* bs = block_sums + f * nblocks;
  __shared__ int carry;
  __shared__ int ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += blockDim.x) {
    const int k = base + threadIdx.x;
    const int x = k < nblocks ? bs[k] : 0;
    // inclusive warp scan
    int s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) >= o) s += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
      int t = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (threadIdx.x >= o) t += y;
      }
      ws[threadIdx.x] = t;
    }
    __syncthreads();
    const int warp_prefix = (threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0;
    const int excl = carry + warp_prefix + s - x;
    if (k < nblocks) bs[k] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) n_points[f] = carry;
}

__global__ void k_cloud_index(const float* __restrict__ disp, const uint8_t* __restrict__ valid,
                              const int* __restrict__ block_offsets, int* __restrict__ index,
                              long n, int nblocks, long stride) {
  const long f = blockIdx.y;
  disp += f * stride;
  valid += f * stride;
  index += f * stride;
  const long i = (long)blockIdx.x * kCloudBlock + threadIdx.x;
  const bool p = i < n && has_point(disp, valid, i);
  const unsigned ballot = __ballot_sync(0xffffffffu, p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int ws[kCloudBlock / 32];
  if (lane == 0) ws[warp] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x < 32) {
    int t = ws[threadIdx.x];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (threadIdx.x >= o) t += y;
    }
    ws[threadIdx.x] = t;  // inclusive
  }
  __syncthreads();
  const int before = (warp ? ws[warp - 1] : 0) + __popc(ballot & ((1u << lane) - 1u));
  if (i < n) index[i] = p ? block_offsets[f * nblocks + blockIdx.x] + before : -1;
}

void launch_cloud_index(const float* disp, const uint8_t* valid, int* index, int* block_sums,
                        int* n_points, int W, int H, int frames, long stride, cudaStream_t s) {
  const long n = (long)W * H;
  if (frames <= 0) return;
  const int nblocks = (int)((n + kCloudBlock - 1) / kCloudBlock);
  if (nblocks == 0) {
    cudaMemsetAsync(n_points, 0, sizeof(int) * frames, s);
    return;
  }
  k_cloud_count<<<dim3(nblocks, frames), kCloudBlock, 0, s>>>(disp, valid, block_sums, n,
                                                             nblocks, stride);
  k_cloud_offsets<<<frames, 1024, 0, s>>>(block_sums, n_points, nblocks);
  k_cloud_index<<<dim3(nblocks, frames), kCloudBlock, 0, s>>>(disp, valid, block_sums, index,
                                                             n, nblocks, stride);
}

__device__ __forceinline__ void point_of(const CloudArgs& c, int u, int v, double d,
                                         double* p) {
  const double z = __ddiv_rn(__dmul_rn(c.fx, c.baseline), d);
  p[0] = __ddiv_rn(__dmul_rn(z, __dsub_rn((double)u, c.cx)), c.fx);
  p[1] = __ddiv_rn(__dmul_rn(z, __dsub_rn((double)v, c.cy)), c.fy);
  p[2] = z;
}

__global__ void k_cloud_points(const float* __restrict__ disp, const int* __restrict__ index,
                               const uint8_t* __restrict__ rgb, int cw, int ch, int W, int H,
                               CloudArgs c, double* __restrict__ pts_d, float* __restrict__ pts_f,
                               uint8_t* __restrict__ colors, int* __restrict__ pixels,
                               long stride, long rgb_stride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = (long)v * W + u;
  const int k = index[f * stride + i];
  if (k < 0) return;
  double p[3];
  point_of(c, u, v, (double)disp[f * stride + i], p);
  const long o = f * stride * 3 + 3l * k;
  if (pts_d) {
    pts_d[o + 0] = p[0];
    pts_d[o + 1] = p[1];
    pts_d[o + 2] = p[2];
  }
  if (pts_f) {
    pts_f[o + 0] = (float)p[0];
    pts_f[o + 1] = (float)p[1];
    pts_f[o + 2] = (float)p[2];
  }
  if (colors) {
    uint8_t r = 0, g = 0, b = 0;
    if (rgb && u < cw && v < ch) {
      const uint8_t* px = rgb + f * rgb_stride + ((long)v * cw + u) * 3;
      r = px[0];
      g = px[1];
      b = px[2];
    }
    colors[o + 0] = r;
    colors[o + 1] = g;
    colors[o + 2] = b;
  }
  if (pixels) {
    pixels[f * stride * 2 + 2l * k + 0] = u;
    pixels[f * stride * 2 + 2l * k + 1] = v;
  }
}

void launch_cloud_points(const float* disp, const int* index, const uint8_t* rgb, int cw,
                         int ch, int W, int H, const CloudArgs& c, double* pts_d,
                         float* pts_f, uint8_t* colors, int* pixels, int frames, long stride,
                         long rgb_stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  dim3 grid((W + 31) / 32, (H + 7) / 8, frames);
  k_cloud_points<<<grid, b, 0, s>>>(disp, index, rgb, cw, ch, W, H, c, pts_d, pts_f, colors,
                                    pixels, stride, rgb_stride);
}

// Smallest-eigenvalue eigenvector of a symmetric 3x3 (a00 a01 a02 a11 a12 a22).
__device__ void sym3_smallest(const double a[6], double ev[3], double n[3]) {
  const double a00 = a[0], a01 = a[1], a02 = a[2], a11 = a[3], a12 = a[4], a22 = a[5];
  const double p1 = a01 * a01 + a02 * a02 + a12 * a12;
  if (p1 == 0.0) {
    // Diagonal: eigenvalues are the diagonal entries, eigenvectors the axes.
    double d[3] = {a00, a11, a22};
    int id[3] = {0, 1, 2};
    for (int x = 0; x < 3; ++x)
      for (int y = x + 1; y < 3; ++y)
        if (d[id[y]] < d[id[x]]) {
          const int t = id[x];
          id[x] = id[y];
          id[y] = t;
        }
    for (int x = 0; x < 3; ++x) ev[x] = d[id[x]];
    n[0] = id[0] == 0 ? 1.0 : 0.0;
    n[1] = id[0] == 1 ? 1.0 : 0.0;
    n[2] = id[0] == 2 ? 1.0 : 0.0;
    return;
  }
  const double q = (a00 + a11 + a22) / 3.0;
  const double b00 = a00 - q, b11 = a11 - q, b22 = a22 - q;
  const double p2 = b00 * b00 + b11 * b11 + b22 * b22 + 2.0 * p1;
  const double p = sqrt(p2 / 6.0);
  const double det = b00 * (b11 * b22 - a12 * a12) - a01 * (a01 * b22 - a12 * a02) +
                     a02 * (a01 * a12 - b11 * a02);
  double r = det / (2.0 * p * p * p);
  r = r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r);
  const double phi = acos(r) / 3.0;
  const double e2 = q + 2.0 * p * cos(phi);
  const double e0 = q + 2.0 * p * cos(phi + 2.0943951023931954923);  // + 2 pi / 3
  const double e1 = 3.0 * q - e0 - e2;
  ev[0] = e0;
  ev[1] = e1;
  ev[2] = e2;
  const double r0[3] = {a00 - e0, a01, a02};
  const double r1[3] = {a01, a11 - e0, a12};
  const double r2[3] = {a02, a12, a22 - e0};
  double c[3][3];
  c[0][0] = r0[1] * r1[2] - r0[2] * r1[1];
  c[0][1] = r0[2] * r1[0] - r0[0] * r1[2];
  c[0][2] = r0[0] * r1[1] - r0[1] * r1[0];
  c[1][0] = r0[1] * r2[2] - r0[2] * r2[1];
  c[1][1] = r0[2] * r2[0] - r0[0] * r2[2];
  c[1][2] = r0[0] * r2[1] - r0[1] * r2[0];
  c[2][0] = r1[1] * r2[2] - r1[2] * r2[1];
  c[2][1] = r1[2] * r2[0] - r1[0] * r2[2];
  c[2][2] = r1[0] * r2[1] - r1[1] * r2[0];
  int bi = 0;
  double bn = -1.0;
  for (int k = 0; k < 3; ++k) {
    const double m = c[k][0] * c[k][0] + c[k][1] * c[k][1] + c[k][2] * c[k][2];
    if (m > bn) {
      bn = m;
      bi = k;
    }
  }
  const double inv = 1.0 / sqrt(bn);
  n[0] = c[bi][0] * inv;
  n[1] = c[bi][1] * inv;
  n[2] = c[bi][2] * inv;
}

__global__ void k_cloud_normals(const float* __restrict__ disp, const int* __restrict__ index,
                                int W, int H, CloudArgs c, double* __restrict__ nrm_d,
                                float* __restrict__ nrm_f, long stride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  disp += f * stride;
  index += f * stride;
  const int k = index[(long)v * W + u];
  if (k < 0) return;
  double p[3];
  point_of(c, u, v, (double)disp[(long)v * W + u], p);
  double mean[3] = {0.0, 0.0, 0.0};
  int count = 0;
  for (int dv = -3; dv <= 3; ++dv) {
    const int nv = v + dv;
    if (nv < 0 || nv >= H) continue;
    for (int du = -3; du <= 3; ++du) {
      const int nu = u + du;
      if (nu < 0 || nu >= W) continue;
      const long ni = (long)nv * W + nu;
      if (__ldg(index + ni) < 0) continue;
      double q[3];
      point_of(c, nu, nv, (double)__ldg(disp + ni), q);
      mean[0] += q[0];
      mean[1] += q[1];
      mean[2] += q[2];
      ++count;
    }
  }
  double n[3] = {0.0, 0.0, -1.0};
  bool fitted = false;
  if (count >= 3) {
    mean[0] /= count;
    mean[1] /= count;
    mean[2] /= count;
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int dv = -3; dv <= 3; ++dv) {
      const int nv = v + dv;
      if (nv < 0 || nv >= H) continue;
      for (int du = -3; du <= 3; ++du) {
        const int nu = u + du;
        if (nu < 0 || nu >= W) continue;
        const long ni = (long)nv * W + nu;
        if (__ldg(index + ni) < 0) continue;
        double q[3];
        point_of(c, nu, nv, (double)__ldg(disp + ni), q);
        q[0] -= mean[0];
        q[1] -= mean[1];
        q[2] -= mean[2];
        a[0] += q[0] * q[0];
        a[1] += q[0] * q[1];
        a[2] += q[0] * q[2];
        a[3] += q[1] * q[1];
        a[4] += q[1] * q[2];
        a[5] += q[2] * q[2];
      }
    }
    double ev[3], e[3];
    sym3_smallest(a, ev, e);
    if (ev[1] > 1e-9 * fmax(1.0, ev[2])) {
      n[0] = e[0];
      n[1] = e[1];
      n[2] = e[2];
      fitted = true;
    }
  }
  if (!fitted) {
    const double len = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    n[0] = -p[0] / len;
    n[1] = -p[1] / len;
    n[2] = -p[2] / len;
  }
  if (n[0] * p[0] + n[1] * p[1] + n[2] * p[2] > 0.0) {
    n[0] = -n[0];
    n[1] = -n[1];
    n[2] = -n[2];
  }
  const long o = f * stride * 3 + 3l * k;
  if (nrm_d) {
    nrm_d[o + 0] = n[0];
    nrm_d[o + 1] = n[1];
    nrm_d[o + 2] = n[2];
  }
  if (nrm_f) {
    nrm_f[o + 0] = (float)n[0];
    nrm_f[o + 1] = (float)n[1];
    nrm_f[o + 2] = (float)n[2];
  }
}

void launch_cloud_normals(const float* disp, const int* index, const CloudArgs& c,
                          double* nrm_d, float* nrm_f, int W, int H, int frames, long stride,
                          cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  dim3 grid((W + 31) / 32, (H + 7) / 8, frames);
  k_cloud_normals<<<grid, b, 0, s>>>(disp, index, W, H, c, nrm_d, nrm_f, stride);
}

}  // namespace ssb
