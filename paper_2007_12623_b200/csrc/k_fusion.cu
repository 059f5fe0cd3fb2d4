// Fusion consumer on the GPU (SPEC.md:440-476 [MODULE]
// fusion): projective association of a keyframe's stereo cloud with the
// surfel model, weighted-average merging and new-point insertion, keeping the
// clouds on the device instead of gathering them to the host. The reference
// has no source for this module (SPEC only); the test oracle restates the
// SPEC's rules with the conventions below, and the kernels reproduce it
// operation for operation (FP64, no contraction).
//
//   pose    row-major [R | t] (world -> camera), X_cam = R X_world + t
//   k_raster_depth / k_raster_id   z-buffer: surfels with X_cam.z > 0 land on
//           pixel (floor(fx x/z + cx + 0.5), floor(fy y/z + cy + 0.5)); the
//           smallest depth wins (atomicMin on the IEEE bits of a positive
//           double, monotone), then the smaller surfel id (second pass)
//   k_fuse_pixels   per stereo pixel with a point: associate with the raster's
//           surfel when |z - z_s| <= gate (each surfel owns at most one pixel,
//           so updates never race) — increment clamped to trunc, weight
//           average, normal re-normalised, colour averaged with the edge-decay
//           weight omega(u, v) — otherwise mark the pixel new; new pixels are
//           appended in raster order (block counts -> scan -> scatter).
#include <limits.h>

#include "ss_internal.cuh"

namespace ssb {

namespace {

struct Pose {
  double m[12];
};

__device__ __forceinline__ void apply(const Pose& P, const double x[3], double y[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    y[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(P.m[4 * r], x[0]), __dmul_rn(P.m[4 * r + 1], x[1])),
                               __dmul_rn(P.m[4 * r + 2], x[2])),
                     P.m[4 * r + 3]);
}
__device__ __forceinline__ void rot_inv(const Pose& P, const double y[3], double x[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
    x[c] = __dadd_rn(__dadd_rn(__dmul_rn(P.m[c], y[0]), __dmul_rn(P.m[4 + c], y[1])),
                     __dmul_rn(P.m[8 + c], y[2]));
}

struct Cam {
  double fx, fy, cx, cy;
  int w, h;
};

// pixel index of a camera-frame point, or -1
__device__ __forceinline__ long project(const Cam& k, const double q[3]) {
  if (!(q[2] > 0.0)) return -1;
  const double u = __dadd_rn(__ddiv_rn(__dmul_rn(k.fx, q[0]), q[2]), k.cx);
  const double v = __dadd_rn(__ddiv_rn(__dmul_rn(k.fy, q[1]), q[2]), k.cy);
  const double fu = floor(__dadd_rn(u, 0.5)), fv = floor(__dadd_rn(v, 0.5));
  if (!(fu >= 0.0 && fu < (double)k.w && fv >= 0.0 && fv < (double)k.h)) return -1;
  return (long)fv * k.w + (long)fu;
}

__device__ __forceinline__ double omega(int u, int v, int w, int h, double omega_min) {
  const double cu = __dmul_rn(0.5, (double)(w - 1)), cv = __dmul_rn(0.5, (double)(h - 1));
  const double du = __dsub_rn((double)u, cu), dv = __dsub_rn((double)v, cv);
  const double r = __dsqrt_rn(__dadd_rn(__dmul_rn(du, du), __dmul_rn(dv, dv)));
  const double R = __dsqrt_rn(__dadd_rn(__dmul_rn(cu, cu), __dmul_rn(cv, cv)));
  double o = R > 0.0 ? __dsub_rn(1.0, __ddiv_rn(r, R)) : 1.0;
  o = o < omega_min ? omega_min : o;
  return o > 1.0 ? 1.0 : o;
}

}  // namespace

struct FusionModel {  // device SoA
  double *pos, *nrm, *col, *w, *cw;
};

__global__ void k_raster_depth(const double* __restrict__ pos, int n, Pose P, Cam k,
                               unsigned long long* __restrict__ zbits) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double x[3] = {pos[3L * s], pos[3L * s + 1], pos[3L * s + 2]};
  double q[3];
  apply(P, x, q);
  const long px = project(k, q);
  if (px >= 0) atomicMin(zbits + px, (unsigned long long)__double_as_longlong(q[2]));
}

__global__ void k_raster_id(const double* __restrict__ pos, int n, Pose P, Cam k,
                            const unsigned long long* __restrict__ zbits, int* __restrict__ ids) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double x[3] = {pos[3L * s], pos[3L * s + 1], pos[3L * s + 2]};
  double q[3];
  apply(P, x, q);
  const long px = project(k, q);
  if (px >= 0 && zbits[px] == (unsigned long long)__double_as_longlong(q[2]))
    atomicMin(ids + px, s);
}

__global__ void k_raster_reset(unsigned long long* __restrict__ zbits, int* __restrict__ ids,
                               long npx) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < npx;
       i += (long)gridDim.x * blockDim.x) {
    zbits[i] = ~0ull;
    ids[i] = INT_MAX;
  }
}

// Points of the stereo cloud: double xyz (per-stage input) or float xyz
// (the ctx's device-resident cloud), one of the two non-null.
struct CloudIn {
  const int* index;
  const double* pd;
  const double* nd;
  const float* pf;
  const float* nf;
  const uint8_t* col;
};
__device__ __forceinline__ void cloud_point(const CloudIn& c, int p, double x[3], double nv[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    x[i] = c.pd ? c.pd[3L * p + i] : (double)c.pf[3L * p + i];
    nv[i] = c.nd ? c.nd[3L * p + i] : (double)c.nf[3L * p + i];
  }
}

// Pass 1: associate + update, or flag new; per-block new counts.
__global__ void k_fuse_pixels(FusionModel M, CloudIn C, Pose P, Cam k,
                              const unsigned long long* __restrict__ zbits,
                              const int* __restrict__ ids, double trunc, double cap, double gate,
                              double omega_min, uint8_t* __restrict__ is_new,
                              int* __restrict__ block_new) {
  __shared__ int warp_cnt[32];
  const long npx = (long)k.w * k.h;
  const long px = blockIdx.x * (long)blockDim.x + threadIdx.x;
  bool fresh = false;
  if (px < npx) {
    const int p = C.index[px];
    if (p >= 0) {
      const int s = ids[px];
      double xc[3], nc[3];
      cloud_point(C, p, xc, nc);
      bool assoc = false;
      if (s != INT_MAX) {
        const double zs = __longlong_as_double((long long)zbits[px]);
        assoc = fabs(__dsub_rn(xc[2], zs)) <= gate;
      }
      if (assoc) {
        double xw[3], nw[3], d[3];
        const double dd[3] = {__dsub_rn(xc[0], P.m[3]), __dsub_rn(xc[1], P.m[7]),
                              __dsub_rn(xc[2], P.m[11])};
        rot_inv(P, dd, xw);
        rot_inv(P, nc, nw);
        double* X = M.pos + 3L * s;
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = __dsub_rn(xw[i], X[i]);
        const double len = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
        if (len > trunc) {
          const double f = __ddiv_rn(trunc, len);
#pragma unroll
          for (int i = 0; i < 3; ++i) d[i] = __dmul_rn(d[i], f);
        }
        const double wo = M.w[s], inv = __ddiv_rn(1.0, __dadd_rn(wo, 1.0));
#pragma unroll
        for (int i = 0; i < 3; ++i) X[i] = __dadd_rn(X[i], __dmul_rn(d[i], inv));
        double* N = M.nrm + 3L * s;
        double a[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) a[i] = __dadd_rn(__dmul_rn(wo, N[i]), nw[i]);
        const double al = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])), __dmul_rn(a[2], a[2])));
        if (al > 0.0) {
#pragma unroll
          for (int i = 0; i < 3; ++i) N[i] = __ddiv_rn(a[i], al);
        }
        const int u = (int)(px % k.w), v = (int)(px / k.w);
        const double om = omega(u, v, k.w, k.h, omega_min);
        double* Cc = M.col + 3L * s;
        const double cw = M.cw[s], cs = __dadd_rn(cw, om);
#pragma unroll
        for (int i = 0; i < 3; ++i)
          Cc[i] = __ddiv_rn(__dadd_rn(__dmul_rn(cw, Cc[i]), __dmul_rn(om, (double)C.col[3L * p + i])), cs);
        const double w1 = __dadd_rn(wo, 1.0);
        M.w[s] = w1 < cap ? w1 : cap;
        M.cw[s] = cs < cap ? cs : cap;
      } else {
        fresh = true;
      }
    }
    is_new[px] = fresh ? 1 : 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, fresh);
  if ((threadIdx.x & 31) == 0) warp_cnt[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += warp_cnt[i];
    block_new[blockIdx.x] = t;
  }
}

// Exclusive scan of the per-block counts (one block), total to *total.
__global__ void k_fuse_scan(int* __restrict__ block_new, int nblocks, int* __restrict__ total) {
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblocks; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const int x = i < nblocks ? block_new[i] : 0;
    // block-wide inclusive scan via warps
    int y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if ((threadIdx.x & 31) >= o) y += t;
    }
    __shared__ int ws[32];
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = y;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) off += ws[w];
    if (i < nblocks) block_new[i] = carry + off + y - x;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += off + y;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Pass 2: append the new points in raster order at n0 + offset.
__global__ void k_fuse_append(FusionModel M, CloudIn C, Pose P, Cam k,
                              const uint8_t* __restrict__ is_new,
                              const int* __restrict__ block_off, int n0, double omega_min) {
  __shared__ int warp_pre[32];
  const long npx = (long)k.w * k.h;
  const long px = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const bool fresh = px < npx && is_new[px];
  const unsigned bal = __ballot_sync(0xffffffffu, fresh);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_pre[wid] = __popc(bal);
  __syncthreads();
  int off = 0;
  for (int w = 0; w < wid; ++w) off += warp_pre[w];
  if (!fresh) return;
  const int m = n0 + block_off[blockIdx.x] + off + __popc(bal & ((1u << lane) - 1));
  const int p = C.index[px];
  double xc[3], nc[3], xw[3], nw[3];
  cloud_point(C, p, xc, nc);
  const double dd[3] = {__dsub_rn(xc[0], P.m[3]), __dsub_rn(xc[1], P.m[7]),
                        __dsub_rn(xc[2], P.m[11])};
  rot_inv(P, dd, xw);
  rot_inv(P, nc, nw);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    M.pos[3L * m + i] = xw[i];
    M.nrm[3L * m + i] = nw[i];
    M.col[3L * m + i] = (double)C.col[3L * p + i];
  }
  M.w[m] = 1.0;
  M.cw[m] = omega((int)(px % k.w), (int)(px / k.w), k.w, k.h, omega_min);
}

__global__ void k_raster_out(const unsigned long long* __restrict__ zbits,
                             const int* __restrict__ ids, int* __restrict__ out_ids,
                             double* __restrict__ out_depth, long npx) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < npx;
       i += (long)gridDim.x * blockDim.x) {
    const bool hit = ids[i] != INT_MAX;
    out_ids[i] = hit ? ids[i] : -1;
    out_depth[i] = hit ? __longlong_as_double((long long)zbits[i]) : 0.0;
  }
}

// ---- launchers ----
void launch_rasterize(const double* pos, int n, const double* pose12, double fx, double fy,
                      double cx, double cy, int w, int h, unsigned long long* zbits, int* ids,
                      cudaStream_t s) {
  Pose P;
  for (int i = 0; i < 12; ++i) P.m[i] = pose12[i];
  const Cam k{fx, fy, cx, cy, w, h};
  const long npx = (long)w * h;
  k_raster_reset<<<(int)std::min<long>((npx + 255) / 256, 4096), 256, 0, s>>>(zbits, ids, npx);
  if (n > 0) {
    k_raster_depth<<<(n + 255) / 256, 256, 0, s>>>(pos, n, P, k, zbits);
    k_raster_id<<<(n + 255) / 256, 256, 0, s>>>(pos, n, P, k, zbits, ids);
  }
}

void launch_raster_out(const unsigned long long* zbits, const int* ids, int* out_ids,
                       double* out_depth, long npx, cudaStream_t s) {
  k_raster_out<<<(int)std::min<long>((npx + 255) / 256, 4096), 256, 0, s>>>(zbits, ids, out_ids,
                                                                              out_depth, npx);
}

void launch_fuse(double* pos, double* nrm, double* col, double* w, double* cw, const int* index,
                 const double* pd, const double* nd, const float* pf, const float* nf,
                 const uint8_t* colors, const double* pose12, double fx, double fy, double cx,
                 double cy, int W, int H, const unsigned long long* zbits, const int* ids,
                 double trunc, double cap, double gate, double omega_min, uint8_t* is_new,
                 int* block_new, int* total, int n0, cudaStream_t s) {
  Pose P;
  for (int i = 0; i < 12; ++i) P.m[i] = pose12[i];
  const Cam k{fx, fy, cx, cy, W, H};
  const FusionModel M{pos, nrm, col, w, cw};
  const CloudIn C{index, pd, nd, pf, nf, colors};
  const long npx = (long)W * H;
  const int nb = (int)((npx + 255) / 256);
  k_fuse_pixels<<<nb, 256, 0, s>>>(M, C, P, k, zbits, ids, trunc, cap, gate, omega_min, is_new,
                                   block_new);
  k_fuse_scan<<<1, 1024, 0, s>>>(block_new, nb, total);
  // appends land in the capacity the caller reserved for the worst case (all
  // pixels new); the count is read back after this launch
  k_fuse_append<<<nb, 256, 0, s>>>(M, C, P, k, is_new, block_new, n0, omega_min);
}

}  // namespace ssb
