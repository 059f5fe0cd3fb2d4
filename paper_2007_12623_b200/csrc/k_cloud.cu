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
//       7x7 neighbourhood (kNormalWindowHalf = 3) of existing points: window
//       moments as FP64 box sums over a 32 x 8 tile, covariance, closed-form
//       FP32 eigenvalues with an FP64 inverse-iteration eigenvector; the fast
//       path only claims "fitted" when lambda1 > 2e-3 max(1, lambda2), ten
//       times its measured error. Below that the pixel runs the reference's
//       computation on the device: mean and covariance of the FP64 points in
//       its neighbour order and a restatement of Eigen 3.4.0's
//       SelfAdjointEigenSolver (cloud.cpp:78, eg::eigen3_sym below) with its
//       acceptance rule lambda1 > 1e-9 max(1, lambda2) (cloud.cpp:81).
//       Normals agree within a tolerance, not bitwise; the
//       fit/fallback decision and the -p/|p| fallback and camera-facing flip
//       (cloud.cpp:81-89) are the reference's.
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
                               float4* __restrict__ pts4, uint8_t* __restrict__ colors,
                               int* __restrict__ pixels, long stride, long rgb_stride) {
  const long f = blockIdx.z;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  const long i = (long)v * W + u;
  const int k = index[f * stride + i];
  if (k < 0) {
    pts4[f * stride + i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  double p[3];
  point_of(c, u, v, (double)disp[f * stride + i], p);
  // pixel-indexed copy for the normal fit (w = 1 marks a point)
  pts4[f * stride + i] = make_float4((float)p[0], (float)p[1], (float)p[2], 1.f);
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
                         float* pts_f, float4* pts4, uint8_t* colors, int* pixels, int frames,
                         long stride, long rgb_stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(32, 8);
  dim3 grid((W + 31) / 32, (H + 7) / 8, frames);
  k_cloud_points<<<grid, b, 0, s>>>(disp, index, rgb, cw, ch, W, H, c, pts_d, pts_f, pts4,
                                    colors, pixels, stride, rgb_stride);
}

// ---- The reference's eigensolver on the device (cloud.cpp:78) ----
// Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d>::compute, restated operation
// for operation (scale by the largest |lower-triangle| entry, 3x3 Householder
// tridiagonalisation, implicit symmetric QR with Wilkinson shifts and
// makeGivens rotations, ascending sort). Every operation is an
// explicit IEEE round-to-nearest intrinsic (this translation unit is built
// with FMA contraction), so for the same covariance the eigenvalues, and the
// fit/fallback test on them, are the test restatement's.
// Used for the near-degenerate neighbourhoods, where the fast closed-form
// solver cannot decide the 1e-9 test.
namespace eg {
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

__device__ double hypot_pos(double x, double y) {  // positive_real_hypot(|x|, |y|)
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  const double p = x > y ? x : y;
  if (p == 0.0) return 0.0;
  const double qp = dvd(y < x ? y : x, p);
  return mul(p, __dsqrt_rn(add(1.0, mul(qp, qp))));
}

__device__ void givens(double p, double q, double& c, double& s) {
  if (q == 0.0) {
    c = p < 0.0 ? -1.0 : 1.0;
    s = 0.0;
  } else if (p == 0.0) {
    c = 0.0;
    s = q < 0.0 ? 1.0 : -1.0;
  } else if (fabs(p) > fabs(q)) {
    const double t = dvd(q, p);
    double u = __dsqrt_rn(add(1.0, mul(t, t)));
    if (p < 0.0) u = -u;
    c = dvd(1.0, u);
    s = mul(-t, c);
  } else {
    const double t = dvd(p, q);
    double u = __dsqrt_rn(add(1.0, mul(t, t)));
    if (q < 0.0) u = -u;
    s = dvd(-1.0, u);
    c = mul(-t, s);
  }
}

__device__ void qr_step(double* diag, double* sub_, int start, int end, double (&Q)[3][3]) {
  const double td = mul(sub(diag[end - 1], diag[end]), 0.5);
  const double e = sub_[end - 1];
  double mu = diag[end];
  if (td == 0.0) {
    mu = sub(mu, fabs(e));
  } else if (e != 0.0) {
    const double e2 = mul(e, e);
    const double h = hypot_pos(td, e);
    const double den = add(td, td > 0.0 ? h : -h);
    if (e2 == 0.0) mu = sub(mu, dvd(e, dvd(den, e)));
    else mu = sub(mu, dvd(e2, den));
  }
  double x = sub(diag[start], mu);
  double z = sub_[start];
  for (int k = start; k < end && z != 0.0; ++k) {
    double c, s;
    givens(x, z, c, s);
    const double sdk = add(mul(s, diag[k]), mul(c, sub_[k]));
    const double dkp1 = add(mul(s, sub_[k]), mul(c, diag[k + 1]));
    diag[k] = sub(mul(c, sub(mul(c, diag[k]), mul(s, sub_[k]))),
                  mul(s, sub(mul(c, sub_[k]), mul(s, diag[k + 1]))));
    diag[k + 1] = add(mul(s, sdk), mul(c, dkp1));
    sub_[k] = sub(mul(c, sdk), mul(s, dkp1));
    if (k > start) sub_[k - 1] = sub(mul(c, sub_[k - 1]), mul(s, z));
    x = sub_[k];
    if (k < end - 1) {
      z = mul(-s, sub_[k + 1]);
      sub_[k + 1] = mul(c, sub_[k + 1]);
    }
    for (int i = 0; i < 3; ++i) {  // Q = Q G: columns k, k+1 by (c, -s)
      const double xi = Q[i][k], yi = Q[i][k + 1];
      Q[i][k] = add(mul(c, xi), mul(-s, yi));
      Q[i][k + 1] = add(mul(s, xi), mul(c, yi));
    }
  }
}

// A: lower triangle {a00, a10, a11, a20, a21, a22}; ev ascending, V columns.
__device__ void eigen3_sym(const double A[6], double ev[3], double (&V)[3][3]) {
  double m00 = A[0], m10 = A[1], m11 = A[2], m20 = A[3], m21 = A[4], m22 = A[5];
  double scale = fmax(fmax(fmax(fabs(m00), fabs(m10)), fmax(fabs(m11), fabs(m20))),
                      fmax(fabs(m21), fabs(m22)));
  if (scale == 0.0) scale = 1.0;
  m00 = dvd(m00, scale);
  m10 = dvd(m10, scale);
  m11 = dvd(m11, scale);
  m20 = dvd(m20, scale);
  m21 = dvd(m21, scale);
  m22 = dvd(m22, scale);
  double diag[3], sb[2];
  diag[0] = m00;
  const double v1norm2 = mul(m20, m20);
  if (v1norm2 <= 2.2250738585072014e-308) {
    diag[1] = m11;
    diag[2] = m22;
    sb[0] = m10;
    sb[1] = m21;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) V[r][c] = r == c ? 1.0 : 0.0;
  } else {
    const double beta = __dsqrt_rn(add(mul(m10, m10), v1norm2));
    const double inv = dvd(1.0, beta);
    const double m01 = mul(m10, inv), m02 = mul(m20, inv);
    const double q = add(mul(mul(2.0, m01), m21), mul(m02, sub(m22, m11)));
    diag[1] = add(m11, mul(m02, q));
    diag[2] = sub(m22, mul(m02, q));
    sb[0] = beta;
    sb[1] = sub(m21, mul(m01, q));
    V[0][0] = 1.0; V[0][1] = 0.0; V[0][2] = 0.0;
    V[1][0] = 0.0; V[1][1] = m01; V[1][2] = m02;
    V[2][0] = 0.0; V[2][1] = m02; V[2][2] = -m01;
  }
  const double precision_inv = 4503599627370496.0;  // 1 / DBL_EPSILON
  int end = 2, start = 0, iter = 0;
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (fabs(sb[i]) < 2.2250738585072014e-308) {
        sb[i] = 0.0;
      } else {
        const double sc = mul(precision_inv, sb[i]);
        if (mul(sc, sc) <= add(fabs(diag[i]), fabs(diag[i + 1]))) sb[i] = 0.0;
      }
    }
    while (end > 0 && sb[end - 1] == 0.0) end--;
    if (end <= 0) break;
    if (++iter > 90) break;
    start = end - 1;
    while (start > 0 && sb[start - 1] != 0.0) start--;
    qr_step(diag, sb, start, end, V);
  }
  if (iter <= 90) {
    for (int i = 0; i < 2; ++i) {
      int k = 0;
      for (int j = 1; j < 3 - i; ++j)
        if (diag[i + j] < diag[i + k]) k = j;
      if (k > 0) {
        const double t = diag[i];
        diag[i] = diag[k + i];
        diag[k + i] = t;
        for (int r = 0; r < 3; ++r) {
          const double tv = V[r][i];
          V[r][i] = V[r][k + i];
          V[r][k + i] = tv;
        }
      }
    }
  }
  for (int k = 0; k < 3; ++k) ev[k] = mul(diag[k], scale);
}
}  // namespace eg

// Smallest eigenpair of a symmetric 3x3 (a00 a01 a02 a11 a12 a22):
// trigonometric eigenvalues, eigenvector from the best-conditioned cross
// product of two rows of (A - l0 I). T = float on the fast path, double for
// the near-degenerate re-check.
__device__ __forceinline__ void sincos_t(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_t(double x, double* s, double* c) { sincos(x, s, c); }

template <typename T>
__device__ void sym3_smallest(const T a[6], T ev[3], T n[3]) {
  const T a00 = a[0], a01 = a[1], a02 = a[2], a11 = a[3], a12 = a[4], a22 = a[5];
  const T p1 = a01 * a01 + a02 * a02 + a12 * a12;
  if (p1 == T(0)) {
    T d[3] = {a00, a11, a22};
    int id[3] = {0, 1, 2};
    for (int x = 0; x < 3; ++x)
      for (int y = x + 1; y < 3; ++y)
        if (d[id[y]] < d[id[x]]) {
          const int t = id[x];
          id[x] = id[y];
          id[y] = t;
        }
    for (int x = 0; x < 3; ++x) ev[x] = d[id[x]];
    n[0] = id[0] == 0 ? T(1) : T(0);
    n[1] = id[0] == 1 ? T(1) : T(0);
    n[2] = id[0] == 2 ? T(1) : T(0);
    return;
  }
  const T q = (a00 + a11 + a22) / T(3);
  const T b00 = a00 - q, b11 = a11 - q, b22 = a22 - q;
  const T p2 = b00 * b00 + b11 * b11 + b22 * b22 + T(2) * p1;
  const T p = sqrt(p2 / T(6));
  const T det = b00 * (b11 * b22 - a12 * a12) - a01 * (a01 * b22 - a12 * a02) +
                a02 * (a01 * a12 - b11 * a02);
  T r = det / (T(2) * p * p * p);
  r = r < T(-1) ? T(-1) : (r > T(1) ? T(1) : r);
  const T phi = acos(r) / T(3);
  T sp, cp;
  sincos_t(phi, &sp, &cp);
  const T e2 = q + T(2) * p * cp;
  // cos(phi + 2 pi / 3) = -(cos phi + sqrt(3) sin phi) / 2
  const T e0 = q - p * (cp + T(1.7320508075688772935) * sp);
  const T e1 = T(3) * q - e0 - e2;
  ev[0] = e0;
  ev[1] = e1;
  ev[2] = e2;
  const T r0[3] = {a00 - e0, a01, a02};
  const T r1[3] = {a01, a11 - e0, a12};
  const T r2[3] = {a02, a12, a22 - e0};
  T cr[3][3];
  cr[0][0] = r0[1] * r1[2] - r0[2] * r1[1];
  cr[0][1] = r0[2] * r1[0] - r0[0] * r1[2];
  cr[0][2] = r0[0] * r1[1] - r0[1] * r1[0];
  cr[1][0] = r0[1] * r2[2] - r0[2] * r2[1];
  cr[1][1] = r0[2] * r2[0] - r0[0] * r2[2];
  cr[1][2] = r0[0] * r2[1] - r0[1] * r2[0];
  cr[2][0] = r1[1] * r2[2] - r1[2] * r2[1];
  cr[2][1] = r1[2] * r2[0] - r1[0] * r2[2];
  cr[2][2] = r1[0] * r2[1] - r1[1] * r2[0];
  int bi = 0;
  T bn = T(-1);
  for (int k = 0; k < 3; ++k) {
    const T m = cr[k][0] * cr[k][0] + cr[k][1] * cr[k][1] + cr[k][2] * cr[k][2];
    if (m > bn) {
      bn = m;
      bi = k;
    }
  }
  const T inv = T(1) / sqrt(bn);
  n[0] = cr[bi][0] * inv;
  n[1] = cr[bi][1] * inv;
  n[2] = cr[bi][2] * inv;
}

constexpr int kNW = 3;              // kNormalWindowHalf (cloud.cpp:10)
constexpr int kNTX = 32, kNTY = 8;  // output tile
constexpr int kNIX = kNTX + 2 * kNW, kNIY = kNTY + 2 * kNW;  // input tile (38 x 14)
constexpr int kNQ = 10;             // window moments: n, sx, sy, sz, sxx, sxy, sxz, syy, syz, szz
constexpr int kNSeg = 2;            // output columns per horizontal running-sum task

constexpr int kNVSeg = 4;           // output rows per vertical running-sum task

struct NormalSmem {
  double p[4][kNIY][kNIX];    // per input pixel: point flag (1/0), x, y, z (0 where no point)
  double h[kNQ][kNIY][kNTX];  // 7-wide horizontal window sums of the kNQ quantities
  double m[kNQ][kNTY][kNTX];  // 7x7 window sums (vertical running sums of h)
};

// Normals from 7x7 window moments (cloud.cpp:41-90). The window's point count,
// coordinate sums and second-moment sums are box sums of per-point
// quantities, computed in FP64 for a whole 32 x 8 tile at once (7-wide
// horizontal running sums of the per-point products, 7-high vertical sums), so a pixel
// costs ~10 products + ~65 adds instead of two 49-point passes. The
// covariance sum (q - mean)(q - mean)^T = S_qq - S_q S_q^T / n is formed in
// FP64 (point magnitudes <= 1e4 mm keep the cancellation error ~1e-7 of the
// entries) and solved in FP32 (closed-form eigenpairs); windows whose middle
// eigenvalue is within 1e-4 of degenerate are re-fitted from FP64 points so
// the reference's 1e-9 acceptance test (cloud.cpp:81) decides them.
__global__ void __launch_bounds__(kNTX * kNTY, 3)
    k_cloud_normals(const float4* __restrict__ pts4, const float* __restrict__ disp, int W,
                    int H, CloudArgs cargs, double* __restrict__ nrm_d,
                    float* __restrict__ nrm_f, short2* __restrict__ nrm_o,
                    uint8_t* __restrict__ fitted_out, const int* __restrict__ index,
                    long stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  NormalSmem& S = *reinterpret_cast<NormalSmem*>(smem_raw);
  const long f = blockIdx.z;
  pts4 += f * stride;
  const int bx = blockIdx.x * kNTX, by = blockIdx.y * kNTY;
  const int tid = threadIdx.y * kNTX + threadIdx.x;
  // all of a thread's tile loads are issued before the first store
  constexpr int kLoads = (kNIY * kNIX + kNTX * kNTY - 1) / (kNTX * kNTY);
  float4 pl[kLoads];
#pragma unroll
  for (int j = 0; j < kLoads; ++j) {
    const int t = tid + j * kNTX * kNTY;
    const int ty = t / kNIX, tx = t - ty * kNIX;
    const int gx = bx + tx - kNW, gy = by + ty - kNW;
    pl[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < kNIY * kNIX && gx >= 0 && gx < W && gy >= 0 && gy < H)
      pl[j] = pts4[(long)gy * W + gx];
  }
#pragma unroll
  for (int j = 0; j < kLoads; ++j) {
    const int t = tid + j * kNTX * kNTY;
    if (t >= kNIY * kNIX) break;
    const int ty = t / kNIX, tx = t - ty * kNIX;
    S.p[0][ty][tx] = pl[j].w != 0.f ? 1.0 : 0.0;
    S.p[1][ty][tx] = pl[j].x;
    S.p[2][ty][tx] = pl[j].y;
    S.p[3][ty][tx] = pl[j].z;
  }
  __syncthreads();
  // horizontal: task = (input row, kNSeg output columns); the 10 quantities of
  // the segment's kNSeg + 6 points are formed on the fly (products of floats
  // are exact in FP64) and slid across the segment.
  constexpr int kSegs = kNTX / kNSeg;
  for (int t = tid; t < kNIY * kSegs; t += kNTX * kNTY) {
    const int r = t / kSegs, c0 = (t % kSegs) * kNSeg;
    auto quant = [&](int c, double (&q)[kNQ]) {
      const double w = S.p[0][r][c], x = S.p[1][r][c], y = S.p[2][r][c], z = S.p[3][r][c];
      q[0] = w;
      q[1] = x;
      q[2] = y;
      q[3] = z;
      q[4] = x * x;
      q[5] = x * y;
      q[6] = x * z;
      q[7] = y * y;
      q[8] = y * z;
      q[9] = z * z;
    };
    double acc[kNQ], q[kNQ];
#pragma unroll
    for (int k = 0; k < kNQ; ++k) acc[k] = 0.0;
#pragma unroll
    for (int du = 0; du <= 2 * kNW; ++du) {
      quant(c0 + du, q);
#pragma unroll
      for (int k = 0; k < kNQ; ++k) acc[k] += q[k];
    }
#pragma unroll
    for (int k = 0; k < kNQ; ++k) S.h[k][r][c0] = acc[k];
#pragma unroll
    for (int j = 1; j < kNSeg; ++j) {
      double qo[kNQ];
      quant(c0 + j + 2 * kNW, q);
      quant(c0 + j - 1, qo);
#pragma unroll
      for (int k = 0; k < kNQ; ++k) {
        acc[k] += q[k] - qo[k];
        S.h[k][r][c0 + j] = acc[k];
      }
    }
  }
  __syncthreads();
  // vertical: task = (quantity, column, kNVSeg output rows), a 7-high running sum
  constexpr int kVSegs = kNTY / kNVSeg;
  for (int t = tid; t < kNQ * kNTX * kVSegs; t += kNTX * kNTY) {
    const int col = t % kNTX, qs = t / kNTX, q = qs / kVSegs, r0 = (qs % kVSegs) * kNVSeg;
    double acc = 0.0;
#pragma unroll
    for (int dv = 0; dv <= 2 * kNW; ++dv) acc += S.h[q][r0 + dv][col];
    S.m[q][r0][col] = acc;
#pragma unroll
    for (int j = 1; j < kNVSeg; ++j) {
      acc += S.h[q][r0 + j + 2 * kNW][col] - S.h[q][r0 + j - 1][col];
      S.m[q][r0 + j][col] = acc;
    }
  }
  __syncthreads();
  const int u = bx + threadIdx.x, v = by + threadIdx.y;
  if (u >= W || v >= H) return;
  const int cy = threadIdx.y + kNW, cx = threadIdx.x + kNW;
  if (S.p[0][cy][cx] == 0.0) return;
  const int k = index[f * stride + (long)v * W + u];
  double m[kNQ];
#pragma unroll
  for (int q = 0; q < kNQ; ++q) m[q] = S.m[q][threadIdx.y][threadIdx.x];
  const int count = (int)m[0];
  float n[3] = {0.f, 0.f, -1.f};
  bool fitted = false;
  if (count >= 3) {
    const double inv = 1.0 / m[0];
    const double ad[6] = {m[4] - m[1] * m[1] * inv, m[5] - m[1] * m[2] * inv,
                          m[6] - m[1] * m[3] * inv, m[7] - m[2] * m[2] * inv,
                          m[8] - m[2] * m[3] * inv, m[9] - m[3] * m[3] * inv};
    const float a[6] = {(float)ad[0], (float)ad[1], (float)ad[2],
                        (float)ad[3], (float)ad[4], (float)ad[5]};
    float ev[3], e[3];
    sym3_smallest<float>(a, ev, e);
    const float scale = fmaxf(1.f, ev[2]);
    // the closed-form FP32 eigenvalues of a near-degenerate neighbourhood
    // are only ~sqrt(eps) accurate (|l1 error| <= 2e-4 max(1, l2) measured
    // over rank-1 neighbourhoods): above 2e-3 the reference's 1e-9 test
    // certainly passes; below, the reference's own solver decides (refit)
    if (ev[1] > 2e-3f * scale) {
      // One FP64 inverse-iteration step, x = adj(A - mu I) e: the FP32
      // eigenvector's error shrinks by |lambda0 - mu| / |lambda1 - mu|, so
      // small eigen gaps (1e-3 of lambda2) still give ~1e-7 rad normals.
      const double mu = ev[0];
      const double b00 = ad[0] - mu, b11 = ad[3] - mu, b22 = ad[5] - mu;
      const double b01 = ad[1], b02 = ad[2], b12 = ad[4];
      const double c00 = b11 * b22 - b12 * b12, c01 = b02 * b12 - b01 * b22,
                   c02 = b01 * b12 - b02 * b11, c11 = b00 * b22 - b02 * b02,
                   c12 = b01 * b02 - b00 * b12, c22 = b00 * b11 - b01 * b01;
      const double x0 = c00 * e[0] + c01 * e[1] + c02 * e[2];
      const double x1 = c01 * e[0] + c11 * e[1] + c12 * e[2];
      const double x2 = c02 * e[0] + c12 * e[1] + c22 * e[2];
      const double len2 = x0 * x0 + x1 * x1 + x2 * x2;
      if (len2 > 0.0 && isfinite(len2)) {
        const double rl = rsqrt(len2);  // the normal is stored in FP32
        n[0] = (float)(x0 * rl);
        n[1] = (float)(x1 * rl);
        n[2] = (float)(x2 * rl);
      } else {
        n[0] = e[0];
        n[1] = e[1];
        n[2] = e[2];
      }
      fitted = true;
    } else {
      // Near-degenerate neighbourhood: the reference's computation
      // (cloud.cpp:49-85): mean and covariance of the FP64 points in its
      // neighbour order, then its eigensolver and 1e-9 test.
      double pd[3];
      double mean[3] = {0.0, 0.0, 0.0};
      for (int dv = -kNW; dv <= kNW; ++dv)
        for (int du = -kNW; du <= kNW; ++du) {
          if (S.p[0][threadIdx.y + kNW + dv][threadIdx.x + kNW + du] == 0.0) continue;
          point_of(cargs, u + du, v + dv, (double)disp[f * stride + (long)(v + dv) * W + u + du], pd);
          mean[0] = __dadd_rn(mean[0], pd[0]);
          mean[1] = __dadd_rn(mean[1], pd[1]);
          mean[2] = __dadd_rn(mean[2], pd[2]);
        }
      mean[0] = __ddiv_rn(mean[0], (double)count);
      mean[1] = __ddiv_rn(mean[1], (double)count);
      mean[2] = __ddiv_rn(mean[2], (double)count);
      double cv[6] = {0, 0, 0, 0, 0, 0};  // lower triangle: 00, 10, 11, 20, 21, 22
      for (int dv = -kNW; dv <= kNW; ++dv)
        for (int du = -kNW; du <= kNW; ++du) {
          if (S.p[0][threadIdx.y + kNW + dv][threadIdx.x + kNW + du] == 0.0) continue;
          point_of(cargs, u + du, v + dv, (double)disp[f * stride + (long)(v + dv) * W + u + du], pd);
          const double x = __dsub_rn(pd[0], mean[0]), y = __dsub_rn(pd[1], mean[1]),
                       z = __dsub_rn(pd[2], mean[2]);
          cv[0] = __dadd_rn(cv[0], __dmul_rn(x, x));
          cv[1] = __dadd_rn(cv[1], __dmul_rn(y, x));
          cv[2] = __dadd_rn(cv[2], __dmul_rn(y, y));
          cv[3] = __dadd_rn(cv[3], __dmul_rn(z, x));
          cv[4] = __dadd_rn(cv[4], __dmul_rn(z, y));
          cv[5] = __dadd_rn(cv[5], __dmul_rn(z, z));
        }
      double evd[3], V[3][3];
      eg::eigen3_sym(cv, evd, V);
      if (evd[1] > __dmul_rn(1e-9, fmax(1.0, evd[2]))) {  // cloud.cpp:81
        n[0] = (float)V[0][0];
        n[1] = (float)V[1][0];
        n[2] = (float)V[2][0];
        fitted = true;
      }
    }
  }
  double nd[3] = {n[0], n[1], n[2]};
  const double pc[3] = {S.p[1][cy][cx], S.p[2][cy][cx], S.p[3][cy][cx]};
  if (!fitted) {
    const double len = sqrt(pc[0] * pc[0] + pc[1] * pc[1] + pc[2] * pc[2]);
    nd[0] = -pc[0] / len;
    nd[1] = -pc[1] / len;
    nd[2] = -pc[2] / len;
  }
  if (nd[0] * pc[0] + nd[1] * pc[1] + nd[2] * pc[2] > 0.0) {
    nd[0] = -nd[0];
    nd[1] = -nd[1];
    nd[2] = -nd[2];
  }
  const long o = f * stride * 3 + 3l * k;
  if (nrm_d) {
    nrm_d[o + 0] = nd[0];
    nrm_d[o + 1] = nd[1];
    nrm_d[o + 2] = nd[2];
  }
  if (nrm_f) {
    nrm_f[o + 0] = (float)nd[0];
    nrm_f[o + 1] = (float)nd[1];
    nrm_f[o + 2] = (float)nd[2];
  }
  if (fitted_out) fitted_out[f * stride + k] = fitted ? 1 : 0;
  if (nrm_o) {
    // octahedral map of the unit normal, snorm16 (decoded by ss_oct_decode)
    const float a = fabsf((float)nd[0]) + fabsf((float)nd[1]) + fabsf((float)nd[2]);
    float x = (float)nd[0] / a, y = (float)nd[1] / a;
    if (nd[2] < 0.0) {
      const float ox = x;
      x = (1.f - fabsf(y)) * (ox < 0.f ? -1.f : 1.f);
      y = (1.f - fabsf(ox)) * (y < 0.f ? -1.f : 1.f);
    }
    nrm_o[f * stride + k] = make_short2((short)__float2int_rn(fminf(fmaxf(x, -1.f), 1.f) * 32767.f),
                                        (short)__float2int_rn(fminf(fmaxf(y, -1.f), 1.f) * 32767.f));
  }
}

void launch_cloud_normals(const float4* pts4, const float* disp, const int* index,
                          const CloudArgs& c, double* nrm_d, float* nrm_f, short2* nrm_o,
                          uint8_t* fitted, int W, int H, int frames, long stride,
                          cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  dim3 b(kNTX, kNTY);
  dim3 grid((W + kNTX - 1) / kNTX, (H + kNTY - 1) / kNTY, frames);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_cloud_normals, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(NormalSmem));
    configured = true;
  }
  k_cloud_normals<<<grid, b, sizeof(NormalSmem), s>>>(pts4, disp, W, H, c, nrm_d, nrm_f, nrm_o,
                                                      fitted, index, stride);
}

}  // namespace ssb
