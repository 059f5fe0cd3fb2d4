// Serial masked row prefix sums (smoothing.cpp:25-41), in the reference's
// exact left-to-right order, at memory speed.
//
// The prefix of a row is a chain of W dependent double adds; the rounding of
// every partial sum is part of the contract (the disc means difference these
// partial sums), so the chain cannot be re-associated. Parallelism therefore
// comes from rows: one warp owns 32 rows (lane = row). Columns stream through
// shared memory in 32-wide chunks — loaded coalesced (lane = column), read
// transposed for the serial adds (lane = row, padded stride: 2-way banks at
// most), written back coalesced — and the next chunk's loads are issued before
// the current chunk's add chain so HBM/L2 latency overlaps the chain.
//
//   k_row_scan_t<double, true>   psum[H][W+1] of a masked double field
//   k_row_scan_t<int, false>     pcnt[H][W+1] of a mask (counts)
#include "ss_internal.cuh"

namespace ssb {

namespace {
constexpr int kScanWarps = 4;
}

template <typename T, bool HAS_VAL>
__global__ void __launch_bounds__(32 * kScanWarps)
    k_row_scan_t(const T* __restrict__ val, const uint8_t* __restrict__ mask,
                 T* __restrict__ psum, int W, int H, long stride, long pstride) {
  __shared__ T tile[kScanWarps][32][33];
  __shared__ uint8_t mtile[kScanWarps][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long f = blockIdx.y;
  const int r0 = (blockIdx.x * kScanWarps + warp) * 32;
  if (r0 >= H) return;  // warp-uniform
  const int nrows = min(32, H - r0);
  val += f * stride + (long)r0 * W;
  mask += f * stride + (long)r0 * W;
  psum += f * pstride + (long)r0 * (W + 1);
  T(*tl)[33] = tile[warp];
  uint8_t(*mt)[33] = mtile[warp];

  T nx[32];
  uint8_t nm[32];
  auto load = [&](int c0) {
    const int c = c0 + lane;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      nm[rr] = 0;
      nx[rr] = T(0);
      if (rr < nrows && c < W) {
        nm[rr] = __ldg(mask + (long)rr * W + c);
        if (HAS_VAL) nx[rr] = __ldg(val + (long)rr * W + c);
      }
    }
  };
  if (lane < nrows) psum[(long)lane * (W + 1)] = T(0);
  T s = T(0);
  load(0);
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int cols = min(32, W - c0);
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
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
          if constexpr (HAS_VAL) {
            s = __dadd_rn(s, tl[lane][c]);
          } else {
            s += 1;
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

void launch_row_scan(const double* val, const uint8_t* valid, double* psum, int W, int H,
                     int frames, long stride, long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int rows_per_block = 32 * kScanWarps;
  k_row_scan_t<double, true><<<dim3((H + rows_per_block - 1) / rows_per_block, frames),
                               32 * kScanWarps, 0, s>>>(val, valid, psum, W, H, stride, pstride);
}

void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int rows_per_block = 32 * kScanWarps;
  k_row_scan_t<int, false><<<dim3((H + rows_per_block - 1) / rows_per_block, frames),
                             32 * kScanWarps, 0, s>>>(nullptr, valid, pcnt, W, H, stride,
                                                      pstride);
}

}  // namespace ssb
