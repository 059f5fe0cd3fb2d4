// Serial masked row prefix sums (smoothing.cpp:25-41), in the reference's
// exact left-to-right order, at memory speed.
//
// The prefix of a row is a chain of W dependent adds whose every rounding is
// part of the contract (the disc means difference the partial sums), so the
// chain cannot be re-associated: parallelism comes only from rows. Two
// implementations:
//
//  * k_scan_bt — refinement scans. Fields live in a row-blocked transposed
//    layout ("BT": element (v, c) at ((v/32)*CW + c)*32 + v%32), so a warp
//    owning 32 rows reads one 256-byte line per column. The warp streams its
//    row block through shared memory with TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx, double-buffered 64-column chunks):
//    the copy engine keeps HBM busy while the lanes run their add chains.
//    psum is written back in BT layout (coalesced), where the tiled disc
//    gathers read it.
//  * k_row_scan_t — normal-layout scan with a shared-memory transpose, used for
//    the cleanup's per-row valid counts.
#include <type_traits>

#include "ss_internal.cuh"

namespace ssb {

namespace {
constexpr int kScanWarps = 4;
constexpr int kRowsPerWarp = 8;
constexpr int kChunk = 64;  // columns per TMA chunk

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

// ---------------- BT-layout scan (refinement) ----------------

template <typename T>
__global__ void __launch_bounds__(32)
    k_scan_bt(const T* __restrict__ xT, const uint8_t* __restrict__ mT, T* __restrict__ pT, int W,
              int RB) {
  __shared__ alignas(128) T xb[2][kChunk][32];
  __shared__ alignas(128) uint8_t mb[2][kChunk][32];
  __shared__ alignas(8) uint64_t bar[2];
  const int lane = threadIdx.x;
  const long f = blockIdx.y;
  const int rb = blockIdx.x;
  const T* xs = xT + (f * RB + rb) * (long)W * 32;
  const uint8_t* ms = mT + (f * RB + rb) * (long)W * 32;
  T* dst = pT + (f * RB + rb) * (long)(W + 1) * 32;
  const int nchunks = (W + kChunk - 1) / kChunk;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int k) {
    const int c0 = k * kChunk, cols = min(kChunk, W - c0);
    const unsigned xbytes = cols * 32 * sizeof(T), mbytes = cols * 32;
    uint64_t* b = &bar[k & 1];
    mbar_expect_tx(b, xbytes + mbytes);
    bulk_g2s(&xb[k & 1][0][0], xs + (long)c0 * 32, xbytes, b);
    bulk_g2s(&mb[k & 1][0][0], ms + (long)c0 * 32, mbytes, b);
  };
  if (lane == 0 && nchunks > 0) issue(0);
  T s = T(0);
  dst[lane] = T(0);
  for (int k = 0; k < nchunks; ++k) {
    if (lane == 0 && k + 1 < nchunks) {
      // buffer (k+1)&1 was last read in iteration k-1 (ordered by __syncwarp)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + 1);
    }
    mbar_wait(&bar[k & 1], (k >> 1) & 1);
    const int c0 = k * kChunk, cols = min(kChunk, W - c0);
    T* out = dst + (long)(c0 + 1) * 32 + lane;
    const T(*xk)[32] = xb[k & 1];
    const uint8_t(*mk)[32] = mb[k & 1];
    if (cols == kChunk) {
#pragma unroll 16
      for (int c = 0; c < kChunk; ++c) {
        const T x = xk[c][lane];
        if (mk[c][lane]) {
          if constexpr (std::is_same<T, double>::value) s = __dadd_rn(s, x);
          else s += x;
        }
        out[(long)c * 32] = s;
      }
    } else {
      for (int c = 0; c < cols; ++c) {
        const T x = xk[c][lane];
        if (mk[c][lane]) {
          if constexpr (std::is_same<T, double>::value) s = __dadd_rn(s, x);
          else s += x;
        }
        out[(long)c * 32] = s;
      }
    }
    __syncwarp();
  }
}

void launch_scan_bt_d(const double* xT, const uint8_t* mT, double* pT, int W, int H, int frames,
                      cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  k_scan_bt<double><<<dim3(RB, frames), 32, 0, s>>>(xT, mT, pT, W, RB);
}

void launch_scan_bt_i(const int* xT, const uint8_t* mT, int* pT, int W, int H, int frames,
                      cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  k_scan_bt<int><<<dim3(RB, frames), 32, 0, s>>>(xT, mT, pT, W, RB);
}

// ---------------- normal layout -> BT layout (value sources) ----------------

struct SrcMask {  // the mask itself
  __device__ uint8_t operator()(long) const { return 1; }
};
struct SrcOne {  // 1 under the mask (disc counts)
  __device__ int operator()(long) const { return 1; }
};
struct SrcDouble {  // a masked double field
  const double* val;
  __device__ double operator()(long i) const { return __ldg(val + i); }
};
struct SrcInt {  // an int field (the integer disparities o)
  const int* val;
  __device__ int operator()(long i) const { return __ldg(val + i); }
};
struct SrcB {  // correction b (smoothing.cpp:96-97) from the exact integer disc sum of o
  const int* so;
  const int* cnt;
  const int* o;
  const double* d;
  double alpha, one_minus_alpha;
  __device__ double operator()(long i) const {
    const double avg = __ddiv_rn((double)__ldg(so + i), (double)__ldg(cnt + i));
    return __dsub_rn(__dsub_rn(avg, __dmul_rn(alpha, (double)__ldg(o + i))),
                     __dmul_rn(one_minus_alpha, __ldg(d + i)));
  }
};

// 32 x 32 tile transpose through shared memory; unmasked entries are 0 and
// rows past H (BT padding) are written as 0 so scans over them are inert.
template <typename T, class Src>
__global__ void __launch_bounds__(32 * 8)
    k_to_bt(Src src, const uint8_t* __restrict__ mask, T* __restrict__ outT, int W, int H, int RB,
            long stride) {
  __shared__ T tile[32][33];
  const long f = blockIdx.z;
  const int c0 = blockIdx.x * 32, v0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int v = v0 + r, c = c0 + threadIdx.x;
    T x = T(0);
    if (v < H && c < W) {
      const long i = f * stride + (long)v * W + c;
      if (mask[i]) x = src(i);
    }
    tile[r][threadIdx.x] = x;
  }
  __syncthreads();
  T* o = outT + (f * RB + blockIdx.y) * (long)W * 32;
  for (int cc = threadIdx.y; cc < 32; cc += 8) {
    const int c = c0 + cc;
    if (c < W) o[(long)c * 32 + threadIdx.x] = tile[threadIdx.x][cc];
  }
}

template <typename T, class Src>
static void launch_to_bt(Src src, const uint8_t* mask, T* outT, int W, int H, int frames,
                         long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  k_to_bt<T, Src><<<dim3((W + 31) / 32, RB, frames), dim3(32, 8), 0, s>>>(src, mask, outT, W, H,
                                                                          RB, stride);
}

void launch_mask_bt(const uint8_t* mask, uint8_t* mT, int W, int H, int frames, long stride,
                    cudaStream_t s) {
  launch_to_bt<uint8_t>(SrcMask{}, mask, mT, W, H, frames, stride, s);
}
void launch_ones_bt(const uint8_t* mask, int* outT, int W, int H, int frames, long stride,
                    cudaStream_t s) {
  launch_to_bt<int>(SrcOne{}, mask, outT, W, H, frames, stride, s);
}
void launch_double_bt(const double* val, const uint8_t* mask, double* outT, int W, int H,
                      int frames, long stride, cudaStream_t s) {
  launch_to_bt<double>(SrcDouble{val}, mask, outT, W, H, frames, stride, s);
}
void launch_int_bt(const int* val, const uint8_t* mask, int* outT, int W, int H, int frames,
                   long stride, cudaStream_t s) {
  launch_to_bt<int>(SrcInt{val}, mask, outT, W, H, frames, stride, s);
}
void launch_b_bt(const int* so, const int* cnt, const int* o, const double* d, double alpha,
                 double one_minus_alpha, const uint8_t* mask, double* bT, int W, int H,
                 int frames, long stride, cudaStream_t s) {
  launch_to_bt<double>(SrcB{so, cnt, o, d, alpha, one_minus_alpha}, mask, bT, W, H, frames,
                       stride, s);
}

// ---------------- normal-layout count scan (cleanup disc support) ----------------

__global__ void __launch_bounds__(32 * kScanWarps)
    k_row_count(const uint8_t* __restrict__ mask, int* __restrict__ psum, int W, int H,
                long stride, long pstride) {
  __shared__ uint8_t mtile[kScanWarps][kRowsPerWarp][33];
  __shared__ int tile[kScanWarps][kRowsPerWarp][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long f = blockIdx.y;
  const int r0 = (blockIdx.x * kScanWarps + warp) * kRowsPerWarp;
  if (r0 >= H) return;  // warp-uniform
  const int nrows = min(kRowsPerWarp, H - r0);
  mask += f * stride + (long)r0 * W;
  psum += f * pstride + (long)r0 * (W + 1);
  uint8_t(*mt)[33] = mtile[warp];
  int(*tl)[33] = tile[warp];
  uint8_t nm[kRowsPerWarp];
  auto load = [&](int c0) {
    const int c = c0 + lane;
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr)
      nm[rr] = (rr < nrows && c < W) ? __ldg(mask + (long)rr * W + c) : 0;
  };
  if (lane < nrows) psum[(long)lane * (W + 1)] = 0;
  int s = 0;
  load(0);
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int cols = min(32, W - c0);
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) mt[rr][lane] = nm[rr];
    __syncwarp();
    if (c0 + 32 < W) load(c0 + 32);
    if (lane < nrows) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c >= cols) break;
        s += mt[lane][c] ? 1 : 0;
        tl[lane][c] = s;
      }
    }
    __syncwarp();
    if (lane < cols)
      for (int rr = 0; rr < nrows; ++rr) psum[(long)rr * (W + 1) + c0 + lane + 1] = tl[rr][lane];
    __syncwarp();
  }
}

void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int rows_per_block = kRowsPerWarp * kScanWarps;
  k_row_count<<<dim3((H + rows_per_block - 1) / rows_per_block, frames), 32 * kScanWarps, 0,
                s>>>(valid, pcnt, W, H, stride, pstride);
}

}  // namespace ssb
