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
#include "tma.cuh"

namespace ssb {

namespace {
constexpr int kChunk = 64;  // columns per TMA chunk

}  // namespace

// ---------------- BT-layout scan (refinement) ----------------

template <typename T>
__device__ __forceinline__ T add_rn(T s, T x) {
  if constexpr (std::is_same<T, double>::value) return __dadd_rn(s, x);
  else return s + x;
}

// xT == nullptr (int only): x = 1 under the mask, i.e. per-row valid counts.
template <typename T>
__global__ void __launch_bounds__(32)
    k_scan_bt(const T* __restrict__ xT, const uint8_t* __restrict__ mT, T* __restrict__ pT, int W,
              int RB, int ext) {
  __shared__ alignas(128) T xb[2][kChunk][32];
  __shared__ alignas(128) uint8_t mb[2][kChunk][32];
  __shared__ alignas(8) uint64_t bar[2];
  const int lane = threadIdx.x;
  const long f = blockIdx.y;
  const int rb = blockIdx.x;
  const bool ones = xT == nullptr;
  const T* xs = ones ? nullptr : xT + (f * RB + rb) * (long)W * 32;
  const uint8_t* ms = mT + (f * RB + rb) * (long)W * 32;
  T* dst = pT + (f * RB + rb) * (long)psum_cw(W, ext) * 32;
  const int nchunks = (W + kChunk - 1) / kChunk;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int k) {
    const int c0 = k * kChunk, cols = min(kChunk, W - c0);
    const unsigned xbytes = ones ? 0u : cols * 32 * sizeof(T), mbytes = cols * 32;
    uint64_t* b = &bar[k & 1];
    mbar_expect_tx(b, xbytes + mbytes);
    if (!ones) bulk_g2s(&xb[k & 1][0][0], xs + (long)c0 * 32, xbytes, b);
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
        const T x = ones ? T(1) : xk[c][lane];
        if (mk[c][lane]) s = add_rn(s, x);
        out[(long)c * 32] = s;
      }
    } else {
      for (int c = 0; c < cols; ++c) {
        const T x = ones ? T(1) : xk[c][lane];
        if (mk[c][lane]) s = add_rn(s, x);
        out[(long)c * 32] = s;
      }
    }
    __syncwarp();
  }
  for (int c = W + 1; c < W + 1 + ext; ++c) dst[(long)c * 32 + lane] = s;  // row total
}

void launch_scan_bt_d(const double* xT, const uint8_t* mT, double* pT, int W, int H, int ext,
                      int frames, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  k_scan_bt<double><<<dim3(RB, frames), 32, 0, s>>>(xT, mT, pT, W, RB, ext);
}

void launch_scan_bt_i(const int* xT, const uint8_t* mT, int* pT, int W, int H, int ext, int frames,
                      cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  k_scan_bt<int><<<dim3(RB, frames), 32, 0, s>>>(xT, mT, pT, W, RB, ext);
}

// Iterations >= 1: the correction b (smoothing.cpp:91-99) formed from the
// exact integer disc sum S_o, o and d, b = (S_o / cnt - a o) - (1 - a) d left
// to right in IEEE double, then the serial prefix. One block per row block:
// thread 0 streams the five fields through shared memory with bulk copies
// (double-buffered 32-column chunks), warps 1..7 form b for chunk k while
// warp 0 runs the add chains over chunk k-1. Invalid pixels contribute +0.0,
// which leaves a prefix bit-identical (it is never -0.0: it starts at +0.0 and
// an exactly-zero round-to-nearest sum is +0.0).
constexpr int kChunkB = 32;
constexpr int kScanBWarps = 16;
struct ScanBRaw {  // [column][row]; the mask is cnt > 0 (disc counts are 0 off the mask)
  int so[kChunkB][32], cnt[kChunkB][32], o[kChunkB][32];
  double d[kChunkB][32];
};
struct ScanBSmem {
  ScanBRaw raw[2];
  double b[2][kChunkB][32];
  uint64_t bar[2];
};

__global__ void __launch_bounds__(32 * kScanBWarps)
    k_scan_b(const int* __restrict__ soT, const int* __restrict__ cntT, const int* __restrict__ oT,
             const double* __restrict__ dT, const uint8_t* __restrict__ mT, double alpha,
             double one_minus_alpha, double* __restrict__ pT, int W, int RB, int ext) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ScanBSmem& S = *reinterpret_cast<ScanBSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long f = blockIdx.y;
  const int rb = blockIdx.x;
  const long base = (f * RB + rb) * (long)W * 32;
  double* dst = pT + (f * RB + rb) * (long)psum_cw(W, ext) * 32;
  const int nchunks = (W + kChunkB - 1) / kChunkB;
  auto issue = [&](int k) {
    const int c0 = k * kChunkB, cols = min(kChunkB, W - c0);
    const long e0 = base + (long)c0 * 32;
    const unsigned n = cols * 32;
    ScanBRaw& B = S.raw[k & 1];
    uint64_t* bar = &S.bar[k & 1];
    mbar_expect_tx(bar, n * (3 * sizeof(int) + sizeof(double)));
    bulk_g2s(&B.so[0][0], soT + e0, n * sizeof(int), bar);
    bulk_g2s(&B.cnt[0][0], cntT + e0, n * sizeof(int), bar);
    bulk_g2s(&B.o[0][0], oT + e0, n * sizeof(int), bar);
    bulk_g2s(&B.d[0][0], dT + e0, n * sizeof(double), bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_fence_init();
    if (nchunks > 0) issue(0);
    if (nchunks > 1) issue(1);
  }
  __syncthreads();
  double s = 0.0;
  if (warp == 0) dst[lane] = 0.0;
  for (int k = 0; k <= nchunks; ++k) {
    if (warp == 0) {
      if (k >= 1) {  // add chains over chunk k-1
        const int c0 = (k - 1) * kChunkB, cols = min(kChunkB, W - c0);
        const double(*bk)[32] = S.b[(k - 1) & 1];
        double* out = dst + (long)(c0 + 1) * 32 + lane;
        if (cols == kChunkB) {
#pragma unroll 8
          for (int c = 0; c < kChunkB; ++c) {
            s = __dadd_rn(s, bk[c][lane]);
            out[(long)c * 32] = s;
          }
        } else {
          for (int c = 0; c < cols; ++c) {
            s = __dadd_rn(s, bk[c][lane]);
            out[(long)c * 32] = s;
          }
        }
      }
    } else if (k < nchunks) {  // form b for chunk k
      mbar_wait(&S.bar[k & 1], (k >> 1) & 1);
      const int cols = min(kChunkB, W - k * kChunkB);
      const ScanBRaw& B = S.raw[k & 1];
      double(*bk)[32] = S.b[k & 1];
      for (int c = warp - 1; c < cols; c += kScanBWarps - 1) {
        double b = 0.0;
        if (B.cnt[c][lane] > 0) {
          const double avg = __ddiv_rn((double)B.so[c][lane], (double)B.cnt[c][lane]);
          b = __dsub_rn(__dsub_rn(avg, __dmul_rn(alpha, (double)B.o[c][lane])),
                        __dmul_rn(one_minus_alpha, B.d[c][lane]));
        }
        bk[c][lane] = b;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && k + 2 < nchunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + 2);  // raw[k & 1] was last read in step k
    }
  }
  if (warp == 0)
    for (int c = W + 1; c < W + 1 + ext; ++c) dst[(long)c * 32 + lane] = s;  // row total
}

void launch_scan_b(const int* soT, const int* cntT, const int* oT, const double* dT,
                   const uint8_t* mT, double alpha, double one_minus_alpha, double* pT, int W,
                   int H, int ext, int frames, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  const int RB = (H + 31) / 32;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_scan_b, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(ScanBSmem));
    configured = true;
  }
  k_scan_b<<<dim3(RB, frames), 32 * kScanBWarps, sizeof(ScanBSmem), s>>>(
      soT, cntT, oT, dT, mT, alpha, one_minus_alpha, pT, W, RB, ext);
}

// ---------------- normal-layout count scan (cleanup disc support) ----------------

// Per-row prefix counts of a u8 mask, psum[r][c + 1] = #nonzero in [0, c]
// (integers, so any order): one warp per row, 32 columns per step by ballot.
constexpr int kCountWarps = 8;

__global__ void __launch_bounds__(32 * kCountWarps)
    k_row_count(const uint8_t* __restrict__ mask, int* __restrict__ psum, int W, int H,
                long stride, long pstride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long f = blockIdx.y;
  const int r = blockIdx.x * kCountWarps + warp;
  if (r >= H) return;  // warp-uniform
  const uint8_t* m = mask + f * stride + (long)r * W;
  int* ps = psum + f * pstride + (long)r * (W + 1);
  if (lane == 0) ps[0] = 0;
  const unsigned below = (1u << lane) - 1u;
  int s = 0;
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int c = c0 + lane;
    const bool on = c < W && __ldg(m + c) != 0;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, on);
    if (c < W) ps[c + 1] = s + __popc(b & below) + (on ? 1 : 0);
    s += __popc(b);
  }
}

void launch_row_count(const uint8_t* valid, int* pcnt, int W, int H, int frames, long stride,
                      long pstride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_row_count<<<dim3((H + kCountWarps - 1) / kCountWarps, frames), 32 * kCountWarps, 0, s>>>(
      valid, pcnt, W, H, stride, pstride);
}

}  // namespace ssb
