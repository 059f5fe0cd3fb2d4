// Serial masked row prefix sums (smoothing.cpp:25-41), in the reference's
// exact left-to-right order, at memory speed.
//
// The prefix of a row is a chain of W dependent double adds; the rounding of
// every partial sum is part of the contract (the disc means difference these
// partial sums), so the chain cannot be re-associated. Parallelism therefore
// comes from rows: one warp owns 8 rows (lanes 0-7 run the chains). Columns stream through
// shared memory in 32-wide chunks — loaded coalesced (lane = column), read
// transposed for the serial adds (lane = row, padded stride: 2-way banks at
// most), written back coalesced — and the next chunk's loads are issued before
// the current chunk's add chain so HBM/L2 latency overlaps the chain.
//
//   SrcDouble  psum[H][W+1] of a masked double field (o in iteration 0)
//   SrcB       the correction b = (S_o/cnt - a o) - (1-a) d computed on the fly
//              (smoothing.cpp:91-99 fused into the prefix of b)
//   SrcCount   pcnt[H][W+1] of a mask (disc counts, disc-fill support)
//   SrcIntOf   exact int prefix of the integer-valued o (S_o initialisation)
#include <type_traits>

#include "ss_internal.cuh"

namespace ssb {

namespace {
constexpr int kScanWarps = 4;
constexpr int kRowsPerWarp = 8;  // 8 serial chains per warp: more warps in flight per SM
}

// Value sources for the masked prefix (evaluated only under the mask).
struct SrcDouble {  // psum of a double field
  const double* val;
  __device__ double operator()(long i) const { return __ldg(val + i); }
};
struct SrcCount {  // prefix counts of the mask
  __device__ int operator()(long) const { return 1; }
};
struct SrcIntOf {  // exact int prefix of an integer-valued double field
  const double* val;
  __device__ int operator()(long i) const { return (int)__ldg(val + i); }
};
struct SrcB {  // correction b (smoothing.cpp:96-97) from the exact integer disc sum of o
  const int* so;
  const int* cnt;
  const double* o;
  const double* d;
  double alpha, one_minus_alpha;
  __device__ double operator()(long i) const {
    const double avg = __ddiv_rn((double)__ldg(so + i), (double)__ldg(cnt + i));
    return __dsub_rn(__dsub_rn(avg, __dmul_rn(alpha, __ldg(o + i))),
                     __dmul_rn(one_minus_alpha, __ldg(d + i)));
  }
};

template <typename T, class Src>
__global__ void __launch_bounds__(32 * kScanWarps)
    k_row_scan_t(Src src, const uint8_t* __restrict__ mask, T* __restrict__ psum, int W, int H,
                 long stride, long pstride) {
  __shared__ T tile[kScanWarps][kRowsPerWarp][33];
  __shared__ uint8_t mtile[kScanWarps][kRowsPerWarp][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long f = blockIdx.y;
  const int r0 = (blockIdx.x * kScanWarps + warp) * kRowsPerWarp;
  if (r0 >= H) return;  // warp-uniform
  const int nrows = min(kRowsPerWarp, H - r0);
  const long base = f * stride + (long)r0 * W;
  mask += base;
  psum += f * pstride + (long)r0 * (W + 1);
  T(*tl)[33] = tile[warp];  // [kRowsPerWarp][33]
  uint8_t(*mt)[33] = mtile[warp];

  T nx[kRowsPerWarp];
  uint8_t nm[kRowsPerWarp];
  auto load = [&](int c0) {
    const int c = c0 + lane;
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      nm[rr] = 0;
      nx[rr] = T(0);
      if (rr < nrows && c < W) {
        nm[rr] = __ldg(mask + (long)rr * W + c);
        if (nm[rr]) nx[rr] = src(base + (long)rr * W + c);
      }
    }
  };
  if (lane < nrows) psum[(long)lane * (W + 1)] = T(0);
  T s = T(0);
  load(0);
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int cols = min(32, W - c0);
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
      tl[rr][lane] = nx[rr];
      mt[rr][lane] = nm[rr];
    }
    __syncwarp();
    if (c0 + 32 < W) load(c0 + 32);  // in flight during the add chain below
    if (lane < nrows) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c >= cols) break;
        if (mt[lane][c]) {
          if constexpr (std::is_same<T, double>::value) {
            s = __dadd_rn(s, tl[lane][c]);
          } else {
            s += tl[lane][c];
          }
        }
        tl[lane][c] = s;
      }
    }
    __syncwarp();
    if (lane < cols) {
      for (int rr = 0; rr < nrows; ++rr) psum[(long)rr * (W + 1) + c0 + lane + 1] = tl[rr][lane];
    }
    __syncwarp();
  }
}

template <typename T, class Src>
static void launch_scan(Src src, const uint8_t* valid, T* psum, int W, int H, int frames,
                        long stride, long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int rows_per_block = kRowsPerWarp * kScanWarps;
  k_row_scan_t<T, Src><<<dim3((H + rows_per_block - 1) / rows_per_block, frames),
                         32 * kScanWarps, 0, s>>>(src, valid, psum, W, H, stride, pstride);
}

void launch_row_scan(const double* val, const uint8_t* valid, double* psum, int W, int H,
                     int frames, long stride, long pstride, cudaStream_t s) {
  launch_scan<double>(SrcDouble{val}, valid, psum, W, H, frames, stride, pstride, s);
}

void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s) {
  launch_scan<int>(SrcCount{}, valid, pcnt, W, H, frames, stride, pstride, s);
}

void launch_int_scan(const double* val, const uint8_t* valid, int* ipsum, int W, int H,
                     int frames, long stride, long pstride, cudaStream_t s) {
  launch_scan<int>(SrcIntOf{val}, valid, ipsum, W, H, frames, stride, pstride, s);
}

void launch_b_scan(const int* so, const int* cnt, const double* o, const double* d,
                   double alpha, double one_minus_alpha, const uint8_t* valid, double* psum,
                   int W, int H, int frames, long stride, long pstride, cudaStream_t s) {
  launch_scan<double>(SrcB{so, cnt, o, d, alpha, one_minus_alpha}, valid, psum, W, H, frames,
                      stride, pstride, s);
}

}  // namespace ssb
