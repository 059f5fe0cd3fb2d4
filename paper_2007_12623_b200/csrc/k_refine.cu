// Anti-shrink Laplacian refinement (refine_disparities, smoothing.cpp:68-159).
//
// Every refinement field lives in the BT layout (ss_internal.cuh): a warp owns
// 32 consecutive rows of one column, so per-pixel loads/stores are single
// lines and a block's 32 x 32 pixel tile is one contiguous 1024-entry range.
//
// Iteration 0 (o = the cleanup output, fractional where filled) follows the
// reference literally: FP64 row prefix of o (k_scan.cu), k_avg_b, FP64 row
// prefix of b, k_d_repick. After it, o is integer-valued, so its disc sum is an
// exact integer S_o (and the reference's double sum of it is exact too):
// S_o is built once (int prefix + k_disc_isum) and then maintained by
// k_so_update from the pixels whose o changed; b is formed inside the b
// prefix scan (k_scan_b). Iterations >= 1 are one serial FP64 scan + one
// tiled gather/re-pick + a small scatter.
//   k_avg_b       disc mean of o (31 row-span differences, dy ascending,
//                 smoothing.cpp:43-63) fused with the correction
//                 b = (avg - a o) - (1-a) d_prev (smoothing.cpp:91-99).
//   k_d_repick    disc mean of b, d = clamp(avg - avg(b), lo, hi)
//                 (smoothing.cpp:104-111) fused with the re-pick
//                 (smoothing.cpp:114-146): argmin over integer candidates of
//                 1/max(zncc, 1e-3) + (eta diff) diff, strict < (first min).
//                 Candidate costs come from the sweep's fp16 score windows in
//                 FP32 with rigorous error bars; ambiguous pixels are settled
//                 in FP64 or deferred to k_repick_exact (exact ZNCC), so the
//                 pick equals the reference's.
// Disc gathers: a block's psum tile (its 32 columns + the radius halo, its row
// block + 16-row halo segments) is staged in shared memory column-major by
// one 64/128-byte bulk copy (TMA) per column segment; a warp then reads 32
// consecutive rows per access (conflict-free), and interior pixels use
// compile-time offsets for the 31 disc rows.
#include <limits.h>
#include <math.h>

#include <stdexcept>
#include <type_traits>
#include <utility>

#include "exact.cuh"
#include "ss_internal.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>
#include <stdio.h>

namespace ssb {

namespace {

constexpr int kTC = 32;                 // tile columns; tile rows = one BT row block
constexpr int kTWarps = 16;             // warp w owns tile columns w and w + 16
constexpr int kPX = kTC / kTWarps;      // pixels per thread
constexpr int kThreads = 32 * kTWarps;  // 512
constexpr size_t kSmemCap = 200 * 1024; // larger tiles: read psum from global

// Tile: the block's row block plus ceil(R/32) whole row blocks above and
// below (one TMA box), psum columns [u0 - R, u0 + kTC + R].
__host__ __device__ constexpr int tile_halo_blocks(int R) { return (R + 31) / 32; }
__host__ __device__ constexpr int tile_nb(int R) { return 1 + 2 * tile_halo_blocks(R); }
__host__ __device__ constexpr int tile_rows(int R) { return 32 * tile_nb(R); }
__host__ __device__ constexpr int tile_cols(int R) { return kTC + 2 * R + 1; }
template <typename T>
__host__ __device__ constexpr size_t tile_bytes(int R) {
  return (sizeof(T) * (size_t)tile_rows(R) * tile_cols(R) + 127) / 128 * 128;
}
// score windows stashed as 8 u32 planes (2 fp16 scores each) x kThreads*kPX slots
constexpr size_t kWinSmem = (size_t)(kWin / 2) * kThreads * kPX * sizeof(uint32_t);
constexpr int kWinPlane = kThreads * kPX;
// per-pixel fields of a tile staged by bulk copies: avg (double) or S_o, cnt,
// o, wbase (int), mask (u8)
constexpr int kTilePx = kTC * 32;
constexpr size_t kPxSmem = (size_t)kTilePx * (8 + 4 + 4 + 4 + 1);

template <typename T>
bool use_tile(int R, size_t extra) {
  return tile_cols(R) <= 256 && tile_bytes<T>(R) + extra <= kSmemCap;  // TMA box <= 256
}

template <typename T>
__device__ __forceinline__ T tsub(T a, T b) {
  if constexpr (std::is_same<T, double>::value) return __dsub_rn(a, b);
  else return a - b;
}
template <typename T>
__device__ __forceinline__ T tadd(T a, T b) {
  if constexpr (std::is_same<T, double>::value) return __dadd_rn(a, b);
  else return a + b;
}

// Row-prefix view: the shared-memory tile (element (row r, psum column c) at
// (c - c0) * pitch + (r - r0)) or, when pitch == 0, the global BT prefix.
template <typename T>
struct Tile {
  const T* t;   // shared-memory tile (kept apart from `g` so loads stay LDS)
  const T* g;   // global BT prefix of the frame
  int pitch, c0, r0, CW;
  __device__ __forceinline__ T at(int r, int c) const {
    return pitch ? t[(c - c0) * pitch + (r - r0)]
                 : __ldg(g + ((long)(r >> 5) * CW + c) * 32 + (r & 31));
  }
};

// Thread 0 arms `bar` for the tile (one TMA tensor copy; out-of-range rows and
// columns arrive as zeros) plus `extra_bytes` of copies the caller issues.
// Callers wait with tile_wait().
template <int RF, typename T>
__device__ __forceinline__ Tile<T> tile_issue(T* sm, const T* psf, const CUtensorMap* map,
                                              int W, int Rr, bool glob, uint64_t* bar,
                                              unsigned extra_bytes = 0) {
  const int R = RF > 0 ? RF : Rr;
  const int u0 = blockIdx.x * kTC;
  const int hb = tile_halo_blocks(R), rows = tile_rows(R), cols = tile_cols(R);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
    mbar_expect_tx(bar, extra_bytes + (glob ? 0u : (unsigned)(rows * cols * sizeof(T))));
    if (!glob) tma_load_4d(sm, map, 0, (int)blockIdx.y - hb, u0 - R, (int)blockIdx.z, bar);
  }
  __syncthreads();
  Tile<T> tl;
  tl.CW = psum_cw(W, R);
  tl.t = sm;
  tl.g = psf;
  tl.pitch = glob ? 0 : rows;
  tl.c0 = u0 - R;
  tl.r0 = ((int)blockIdx.y - hb) * 32;
  return tl;
}

__device__ __forceinline__ void tile_wait(uint64_t* bar) {
  mbar_wait(bar, 0);
  __syncthreads();
}

// ---- disc sums of a masked field from its row prefixes (smoothing.cpp:43-63) ----
// For dy ascending, the span difference psum[row][u1+1] - psum[row][u0]:
// the reference's operands and order, so bit-exact.

template <typename T>
__device__ __forceinline__ T disc_sum_generic(const Tile<T>& P, const int* __restrict__ span,
                                              int W, int H, int u, int v, int R) {
  const int lo = max(-R, -v), hi = min(R, H - 1 - v);
  T s = T(0);
  for (int dy = lo; dy <= hi; ++dy) {
    const int sx = __ldg(span + (dy < 0 ? -dy : dy));
    const int c0 = max(0, u - sx), c1 = min(W - 1, u + sx) + 1;
    s = tadd(s, tsub(P.at(v + dy, c1), P.at(v + dy, c0)));
  }
  return s;
}

__host__ __device__ constexpr int isqrt_floor(int x) {
  int r = 0;
  while ((r + 1) * (r + 1) <= x) ++r;
  return r;
}

template <typename T, int R, int DY>
__device__ __forceinline__ T span_diff(const T* q) {
  constexpr int P = tile_rows(R);
  constexpr int SX = isqrt_floor(R * R - DY * DY);
  return tsub(q[(SX + 1) * P + DY], q[-SX * P + DY]);
}

template <typename T, int R, int... I>
__device__ __forceinline__ T disc_sum_fixed(const T* q, std::integer_sequence<int, I...>) {
  T s = T(0);
  ((s = tadd(s, span_diff<T, R, I - R>(q))), ...);  // dy ascending, left to right
  return s;
}

// With a compile-time radius (always a shared-memory tile) every pixel reads
// the tile at immediate offsets from one base pointer: the extended prefix
// layout (psum_cw) makes the clipped spans of border pixels read the values
// the clipped indices would, and out-of-image rows contribute +0.0 terms.
template <int RF, typename T>
__device__ __forceinline__ T disc_sum_any(const Tile<T>& P, const int* span, int W, int H,
                                          int u, int v, int Rr) {
  if constexpr (RF > 0) {
    const T* q = P.t + (u - P.c0) * tile_rows(RF) + (v - P.r0);
    return disc_sum_fixed<T, RF>(q, std::make_integer_sequence<int, 2 * RF + 1>{});
  } else {
    return disc_sum_generic(P, span, W, H, u, v, Rr);
  }
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Tensor map for a launch's prefix tiles; false (global reads) when the tile
// does not fit or the driver rejects the map (reported once on stderr).
template <typename T>
bool psum_map(CUtensorMap* m, const T* psumT, const RefineArgs& a, int frames, bool tile) {
  *m = CUtensorMap{};
  if (!tile) return false;
  if (make_psum_tmap(m, psumT, std::is_same<T, double>::value, a.g.W, a.g.H, a.radius, frames,
                     tile_nb(a.radius), tile_cols(a.radius)))
    return true;
  static bool warned = false;
  if (!warned) {
    fprintf(stderr, "stereoscan-b200: TMA tensor map rejected; disc gathers read global memory\n");
    warned = true;
  }
  return false;
}

}  // namespace

bool make_psum_tmap(CUtensorMap* map, const void* base, bool is_double, int W, int H, int ext,
                    int frames, int nb, int cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t es = is_double ? 8 : 4;
  const cuuint64_t RB = (H + 31) / 32, CW = psum_cw(W, ext);
  const cuuint64_t dims[4] = {32, RB, CW, (cuuint64_t)frames};
  const cuuint64_t strides[3] = {CW * 32 * es, 32 * es, RB * CW * 32 * es};
  const cuuint32_t box[4] = {32, (cuuint32_t)nb, (cuuint32_t)cols, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(map, is_double ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT32,
                4, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------- normal <-> BT ----------------

__global__ void __launch_bounds__(256)
    k_refine_init(const float* __restrict__ disp, const uint8_t* __restrict__ valid,
                  uint8_t* __restrict__ mT, double* __restrict__ oT, double* __restrict__ dT,
                  int W, int H, long stride, long bs, const int2* __restrict__ lstat,
                  int* __restrict__ wbase, int* __restrict__ list, unsigned* __restrict__ count,
                  Geom g) {
  __shared__ float td[32][33];
  __shared__ uint8_t tv[32][33];  // bit 0: valid, bit 1: var_l == 0 (no defined score)
  const long f = blockIdx.z;
  const int u0 = blockIdx.x * 32, rb = blockIdx.y, v0 = rb * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int v = v0 + r, c = u0 + threadIdx.x;
    float x = 0.f;
    uint8_t m = 0;
    if (v < H && c < W) {
      const long i = f * stride + (long)v * W + c;
      m = valid[i] ? 1 : 0;
      x = disp[i];
      if (wbase && m && isnan(__int_as_float(__ldg(&lstat[i].y)))) m |= 2;
    }
    td[r][threadIdx.x] = x;
    tv[r][threadIdx.x] = m;
  }
  __syncthreads();
  for (int cc = threadIdx.y; cc < 32; cc += 8) {
    const int c = u0 + cc;
    if (c >= W) continue;
    const long bi = f * bs + ((long)rb * W + c) * 32 + threadIdx.x;
    const uint8_t m = tv[threadIdx.x][cc];
    const float xf = td[threadIdx.x][cc];
    const double x = (m & 1) ? (double)xf : 0.0;  // rows past H: m = 0
    mT[bi] = m & 1;
    oT[bi] = x;
    dT[bi] = x;
    if (wbase && (m & 1)) {
      // window check (the sweep's window vs one centred on the cleanup output)
      const int v = v0 + threadIdx.x, h = g.half;
      const bool fits = c >= h && c < W - h && v >= h && v < H - h;
      if (!fits || (m & 2)) {
        wbase[bi] = kNoWin;
      } else {
        const int want = window_base((int)floor((double)xf), g.cmin, g.NC);
        if (wbase[bi] != want) list[f * stride + atomicAdd(count + f, 1u)] = v * W + c;
      }
    }
  }
}

void launch_refine_init(const float* disp, const uint8_t* valid, uint8_t* mT, double* oT,
                        double* dT, int W, int H, int frames, long stride, long bs,
                        const int2* lstat, int* wbase, int* list, unsigned* count, const Geom& g,
                        cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_refine_init<<<dim3((W + 31) / 32, (H + 31) / 32, frames), dim3(32, 8), 0, s>>>(
      disp, valid, mT, oT, dT, W, H, stride, bs, lstat, wbase, list, count, g);
}

__global__ void __launch_bounds__(256)
    k_refine_out(const double* __restrict__ dT, const uint8_t* __restrict__ valid,
                 const float* __restrict__ din, float* __restrict__ dout, int W, int H,
                 long stride, long bs) {
  __shared__ float td[32][33];
  const long f = blockIdx.z;
  const int u0 = blockIdx.x * 32, rb = blockIdx.y, v0 = rb * 32;
  for (int cc = threadIdx.y; cc < 32; cc += 8) {
    const int c = u0 + cc;
    td[cc][threadIdx.x] = c < W ? (float)dT[f * bs + ((long)rb * W + c) * 32 + threadIdx.x] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int v = v0 + r, c = u0 + threadIdx.x;
    if (v < H && c < W) {
      const long i = f * stride + (long)v * W + c;
      dout[i] = valid[i] ? td[threadIdx.x][r] : din[i];
    }
  }
}

void launch_refine_out(const double* dT, const uint8_t* valid, const float* din, float* dout,
                       int W, int H, int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_refine_out<<<dim3((W + 31) / 32, (H + 31) / 32, frames), dim3(32, 8), 0, s>>>(
      dT, valid, din, dout, W, H, stride, bt_frame(W, H, 0));
}

// RefineTrace rows (one frame): discrete = valid ? o : 0, smooth = d.
__global__ void __launch_bounds__(256)
    k_trace_rows(const int* __restrict__ oT, const double* __restrict__ dT,
                 const uint8_t* __restrict__ valid, double* __restrict__ to,
                 double* __restrict__ td_out, int W, int H) {
  __shared__ double to_s[32][33], td_s[32][33];
  const int u0 = blockIdx.x * 32, rb = blockIdx.y, v0 = rb * 32;
  for (int cc = threadIdx.y; cc < 32; cc += 8) {
    const int c = u0 + cc;
    if (c < W) {
      const long bi = ((long)rb * W + c) * 32 + threadIdx.x;
      to_s[cc][threadIdx.x] = (double)oT[bi];
      td_s[cc][threadIdx.x] = dT[bi];
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int v = v0 + r, c = u0 + threadIdx.x;
    if (v < H && c < W) {
      const long i = (long)v * W + c;
      if (to) to[i] = valid[i] ? to_s[threadIdx.x][r] : 0.0;
      if (td_out) td_out[i] = td_s[threadIdx.x][r];
    }
  }
}

void launch_trace_rows(const int* oT, const double* dT, const uint8_t* valid, double* trace_o,
                       double* trace_d, int W, int H, cudaStream_t s) {
  if (W <= 0 || H <= 0) return;
  k_trace_rows<<<dim3((W + 31) / 32, (H + 31) / 32), dim3(32, 8), 0, s>>>(oT, dT, valid, trace_o,
                                                                         trace_d, W, H);
}

// ---------------- tiled disc gathers ----------------

// Exact integer disc sums (disc counts, S_o) from an int BT prefix.
template <int RF>
__global__ void __launch_bounds__(kThreads)
    k_disc_isum(const uint8_t* __restrict__ mT, const int* __restrict__ ipsumT,
                int* __restrict__ outT, RefineArgs a, const __grid_constant__ CUtensorMap map,
                int glob) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  const long bs = bt_frame(W, H, 0);
  const Tile<int> P = tile_issue<RF>(reinterpret_cast<int*>(smem), ipsumT + f * bt_frame(W, H, 1 + R),
                                     &map, W, R, glob, &bar);
  tile_wait(&bar);
  const int v = blockIdx.y * 32 + threadIdx.x;
#pragma unroll
  for (int k = 0; k < kPX; ++k) {
    const int u = blockIdx.x * kTC + threadIdx.y + kTWarps * k;
    if (u >= W) continue;
    const long bi = f * bs + bt_index(W, v, u);
    // 0 off the mask and on the padding rows past H: the b scan takes its mask
    // from the disc counts (cnt > 0)
    outT[bi] = (v < H && mT[bi]) ? disc_sum_any<RF>(P, a.span, W, H, u, v, R) : 0;
  }
}

void launch_disc_isum(const uint8_t* mT, const int* ipsumT, int* outT, const RefineArgs& a,
                      int frames, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  CUtensorMap map;
  const bool tile = psum_map(&map, ipsumT, a, frames, use_tile<int>(a.radius, 0));
  const size_t smem = tile ? tile_bytes<int>(a.radius) : 0;
  dim3 grid((a.g.W + kTC - 1) / kTC, (a.g.H + 31) / 32, frames);
  dim3 bl(32, kTWarps);
  if (a.radius == 15 && tile) {
    k_disc_isum<15><<<grid, bl, smem, s>>>(mT, ipsumT, outT, a, map, 0);
  } else {
    set_smem(k_disc_isum<0>, smem);
    k_disc_isum<0><<<grid, bl, smem, s>>>(mT, ipsumT, outT, a, map, tile ? 0 : 1);
  }
}

template <int RF>
__global__ void __launch_bounds__(kThreads)
    k_avg_b(const double* __restrict__ psumT, const uint8_t* __restrict__ mT,
            const int* __restrict__ cntT, const double* __restrict__ oT,
            const double* __restrict__ dT, double* __restrict__ avgT, double* __restrict__ bT,
            RefineArgs a, const __grid_constant__ CUtensorMap map, int glob) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  const long bs = bt_frame(W, H, 0);
  const Tile<double> P = tile_issue<RF>(reinterpret_cast<double*>(smem),
                                        psumT + f * bt_frame(W, H, 1 + R), &map, W, R, glob, &bar);
  tile_wait(&bar);
  const int v = blockIdx.y * 32 + threadIdx.x;
#pragma unroll
  for (int k = 0; k < kPX; ++k) {
    const int u = blockIdx.x * kTC + threadIdx.y + kTWarps * k;
    if (u >= W || v >= H) continue;
    const long bi = f * bs + bt_index(W, v, u);
    if (!mT[bi]) continue;
    const double s = disc_sum_any<RF>(P, a.span, W, H, u, v, R);
    const double av = __ddiv_rn(s, (double)cntT[bi]);
    avgT[bi] = av;
    // averaged - alpha * discrete - (1 - alpha) * smooth, left to right.
    bT[bi] = __dsub_rn(__dsub_rn(av, __dmul_rn(a.alpha, oT[bi])),
                       __dmul_rn(a.one_minus_alpha, dT[bi]));
  }
}

void launch_avg_b(const double* psumT, const uint8_t* mT, const int* cntT, const double* oT,
                  const double* dT, double* avgT, double* bT, const RefineArgs& a, int frames,
                  cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  CUtensorMap map;
  const bool tile = psum_map(&map, psumT, a, frames, use_tile<double>(a.radius, 0));
  const size_t smem = tile ? tile_bytes<double>(a.radius) : 0;
  dim3 grid((a.g.W + kTC - 1) / kTC, (a.g.H + 31) / 32, frames);
  dim3 bl(32, kTWarps);
  if (a.radius == 15 && tile) {
    set_smem(k_avg_b<15>, smem);
    k_avg_b<15><<<grid, bl, smem, s>>>(psumT, mT, cntT, oT, dT, avgT, bT, a, map, 0);
  } else {
    set_smem(k_avg_b<0>, smem);
    k_avg_b<0><<<grid, bl, smem, s>>>(psumT, mT, cntT, oT, dT, avgT, bT, a, map, tile ? 0 : 1);
  }
}

// ---------------- re-pick ----------------

namespace {

// A thread's window: 16 fp16 match costs (m_code: M - 1) in 8 u32 planes.
struct WinView {
  const uint32_t* p;  // plane 0 word of this pixel; plane j at p[j * stride]
  long stride;        // kWinPlane (shared-memory planes) or W * 32 (global BT planes)
  __device__ __forceinline__ float mcost(int k) const {  // M16 of entry k in [0, kWin)
    const uint32_t w = p[(k >> 1) * stride];
    return 1.f +
           __half2float(__ushort_as_half((unsigned short)((k & 1) ? (w >> 16) : (w & 0xFFFFu))));
  }
};

__device__ __forceinline__ double exact_cost(const uint8_t* L, const uint8_t* R, int W, int u,
                                             int v, int c, bool fits, int half, double dval,
                                             double eta) {
  double match = __ddiv_rn(1.0, kZnccEps);
  const int ru = u - c;
  if (fits && ru >= half && ru < W - half) {
    const ExactScore es = zncc_exact(L, R, W, u, v, ru, half, false);
    if (es.defined) match = __ddiv_rn(1.0, es.score < kZnccEps ? kZnccEps : es.score);
  }
  const double diff = __dsub_rn((double)c, dval);
  return __dadd_rn(match, __dmul_rn(__dmul_rn(eta, diff), diff));
}

constexpr int kMaxCand = 2 * kRefineR + 1;

// FP64 version for the rare paths: exact E (reference expression) and exact M
// when the score is undefined/clamped (code 1000); err bounds the window M16's
// error (kMA |M16 - 1| + kMB M16, ss_internal.cuh).
__device__ __forceinline__ void repick_cost_d(const RefineArgs& a, int u, int c, double dv,
                                              const WinView& wv, int wb, int W, int half,
                                              double& cost, double& err) {
  double m = 1000.0;
  err = 0.0;
  const int ru = u - c;
  if (ru >= half && ru < W - half) {
    const float mf = wv.mcost(c - wb);
    if (mf != 1000.f) {
      m = (double)mf;
      err = (double)kMA * fabs((double)mf - 1.0) + (double)kMB * (double)mf;
    }
  }
  const double diff = __dsub_rn((double)c, dv);
  cost = __dadd_rn(m, __dmul_rn(__dmul_rn(a.eta, diff), diff));
}

__device__ __forceinline__ int defer_pixel(Deferred* defer, unsigned* defer_count, long pix,
                                           int c_lo, int mask, double dv) {
  Deferred* e = defer + atomicAdd(defer_count, 1u);
  int2* ei = reinterpret_cast<int2*>(e);  // Deferred is 8-byte aligned
  ei[0] = make_int2((int)pix, c_lo);
  ei[1] = make_int2(mask, 0);
  e->d = dv;
  return INT_MIN;
}

// ---- re-pick certificates ----
// A re-pick that proves its pick b the strict first minimum also proves it for
// every later smoothed d' in an interval around its d: the candidate set is
// fixed while ceil(d' - 5) and floor(d' + 5) (with the [lo, hi] clamps) are,
// and a candidate c's cost gap to b is linear in d',
//   gap_c(d') = gap_c(d) - 2 eta (c - b) (d' - d)     (real arithmetic),
// because the match costs M_c do not depend on d. With a rigorous lower bound
// on every gap_c(d) (the filter's error bars, a safety term that covers the
// FP32 evaluation and the reference's own double roundings) the interval on
// which every gap stays positive is stored per pixel (float, rounded inward);
// a later iteration whose d' falls inside it keeps o = b without re-scoring.
// An empty interval (lo > hi) means "always re-pick".
__device__ __forceinline__ float2 iv_empty() { return make_float2(INFINITY, -INFINITY); }

// [dv + dn, dv + up] intersected with the candidate-set cells, rounded inward.
__device__ __forceinline__ float2 iv_finish(const RefineArgs& a, double dv, double dn, double up,
                                            int c_lo, int c_hi) {
  constexpr double m = 1e-9;  // >> ulp(|d| <= 2^10) / 2: RN(d' -+ 5) stays in the cell
  double lo = dv + dn, hi = dv + up;
  const double cl = ceil(a.lo), fh = floor(a.hi);
  if ((double)c_lo > cl) {  // c_lo = ceil(RN(d - 5)): c_lo - 1 < d' - 5 <= c_lo
    lo = fmax(lo, (double)c_lo + 4.0 + m);
    hi = fmin(hi, (double)c_lo + 5.0);
  } else {  // clamped at ceil(lo): d' - 5 <= ceil(lo)
    hi = fmin(hi, cl + 5.0);
  }
  if ((double)c_hi < fh) {  // c_hi = floor(RN(d + 5)): c_hi <= d' + 5 < c_hi + 1
    lo = fmax(lo, (double)c_hi - 5.0);
    hi = fmin(hi, (double)c_hi - 4.0 - m);
  } else {  // clamped at floor(hi): d' + 5 >= floor(hi)
    lo = fmax(lo, fh - 5.0);
  }
  if (!(lo <= hi)) return iv_empty();
  return make_float2(__double2float_ru(lo), __double2float_rd(hi));
}

// Re-pick of one pixel (smoothing.cpp:119-144) given its smoothed d.
// Returns the new o, or INT_MIN: not found (dmask = 0, unreachable for a
// clamped d) or to be settled exactly (dmask = the candidates c_lo + k to
// score, dclo = c_lo). iv (optional) receives the pick's certificate interval.
//
// Filter error budget: window entries are fp16 match
// costs M16 from the FP32 sweep score s_f (|s_f - s| <= 5 ulp_f32) with
// |M16 - M| <= 5.01e-4 M (m_code), and the float cost M16 + (eta diff) diff
// adds FP32 rounding. Candidates within the error bars of the float minimum
// are re-scored in FP64 / exactly; a single survivor is provably the
// reference's argmin.
__device__ __forceinline__ int repick(const RefineArgs& a, int u, int v, double dv,
                                      const uint8_t* L, const uint8_t* R, bool has_win,
                                      const WinView& wv, int wb, int& dclo, int& dmask,
                                      float2& iv, bool want_iv) {
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const int c_lo = max((int)ceil(__dsub_rn(dv, (double)kRefineR)), (int)ceil(a.lo));
  const int c_hi = min((int)floor(__dadd_rn(dv, (double)kRefineR)), (int)floor(a.hi));
  dclo = c_lo;
  dmask = 0;
  iv = iv_empty();
  if (c_lo > c_hi) return INT_MIN;  // unreachable for a clamped d; mirrors `found`
  const bool fits = u >= half && u < W - half && v >= half && v < H - half;

  if (!has_win) {
    // Generic window size: every candidate in exact FP64 (no score windows).
    double best_cost = 0.0;
    int best = c_lo;
    for (int c = c_lo; c <= c_hi; ++c) {
      const double cost = exact_cost(L, R, W, u, v, c, fits, half, dv, a.eta);
      if (c == c_lo || cost < best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    return best;
  }
  if (!fits || wb == kNoWin) {
    // Window does not fit or var_l == 0: every match cost is exactly
    // 1/kZnccCostEpsilon, so the reference's double costs are computed as is.
    const double m = __ddiv_rn(1.0, kZnccEps);
    double best_cost = 0.0;
    int best = c_lo;
    for (int c = c_lo; c <= c_hi; ++c) {
      const double diff = __dsub_rn((double)c, dv);
      const double cost = __dadd_rn(m, __dmul_rn(__dmul_rn(a.eta, diff), diff));
      if (c == c_lo || cost < best_cost) {
        best_cost = cost;
        best = c;
      }
    }
    if (want_iv) {
      // exact reference costs: the gaps are known up to the reference's
      // roundings (~1e-13 at cost 1000)
      double dn = -INFINITY, up = INFINITY;
      bool ok = true;
      for (int c = c_lo; c <= c_hi; ++c) {
        if (c == best) continue;
        const double diff = __dsub_rn((double)c, dv);
        const double cost = __dadd_rn(m, __dmul_rn(__dmul_rn(a.eta, diff), diff));
        const double gap = cost - best_cost - 1e-9 * (1.0 + fabs(best_cost));
        ok = ok && gap > 0.0;
        const double sl = 2.0 * a.eta * (double)(c - best);
        if (sl > 0.0) up = fmin(up, gap / sl * (1.0 - 1e-9));
        else if (sl < 0.0) dn = fmax(dn, gap / sl * (1.0 - 1e-9));
      }
      if (ok) iv = iv_finish(a, dv, dn, up, c_lo, c_hi);
    }
    return best;
  }
  int best = c_lo;
  if (c_lo >= wb && c_hi <= wb + kWin - 1) {
    // Common path, FP32. cost_f(c) = M16 + E_f with |cost_f - cost| <=
    // err_c = kMA |M16 - 1| + kMB M16 (the window's M, ss_internal.cuh) +
    // 2.4e-7 |cost_f| (the FMA's rounding and that of the bounds) + errE (the
    // FP32 copy of d and E's roundings). The first minimum b is certified
    // when every other candidate's lower bound stays above b's upper bound.
    const float dv_f = (float)dv;
    const float delta = fabsf(dv_f) * 1.2e-7f;  // |dv_f - d|, and FP32 rounding of c - dv_f
    const float errE = fabsf(a.eta_f) * (11.f * delta + 25.f * 4e-7f);
    // The <= 11 candidates are entries off .. off+10 of the window: 6 words
    // from the planes, then one byte-permute per candidate.
    const int off = c_lo - wb, par = off & 1, w0 = off >> 1;
    uint32_t wd[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) wd[i] = wv.p[min(w0 + i, kWin / 2 - 1) * wv.stride];
    const unsigned sel_e = par ? 0x3232u : 0x1010u, sel_o = par ? 0x5454u : 0x3232u;
    // Branch-free over the 11 slots: slots past c_hi cost +inf. The FMA
    // rounds once where M16 + (eta df) df rounded twice, inside the same bar.
    const int nk = c_hi - c_lo;
    // Candidate costs two at a time on the packed FP32 pipe (FADD2 / FMUL2 /
    // FFMA2: per-lane IEEE ops, the same values as the scalar expressions
    // 1 + h, (c - dv_f) and fma(eta df, df, M16)).
    float cost[kMaxCand + 1], errk[kMaxCand + 1];
    const float cf = (float)c_lo;
#pragma unroll
    for (int k = 0; k < kMaxCand; k += 2) {
      float hk[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = k + h;
        if (kk >= kMaxCand) {
          hk[h] = 0.f;
          continue;
        }
        const uint32_t hw = (kk & 1) ? __byte_perm(wd[kk >> 1], wd[min(kk + 1, 11) >> 1], sel_o)
                                     : __byte_perm(wd[kk >> 1], 0u, sel_e);
        hk[h] = __half2float(__ushort_as_half((unsigned short)(hw & 0xFFFFu)));
      }
      const float2 m16 = __fadd2_rn(make_float2(hk[0], hk[1]), make_float2(1.f, 1.f));  // exact
      const float2 c2 = __fadd2_rn(make_float2(cf, cf), make_float2((float)k, (float)(k + 1)));
      const float2 df = __fadd2_rn(c2, make_float2(-dv_f, -dv_f));
      const float2 e = __fmul2_rn(make_float2(a.eta_f, a.eta_f), df);
      const float2 c = __ffma2_rn(e, df, m16);
      cost[k] = c.x;
      cost[k + 1] = c.y;
      errk[k] = kMA * fabsf(hk[0]) + kMB * m16.x + 2.4e-7f * fabsf(c.x) + errE;
      errk[k + 1] = kMA * fabsf(hk[1]) + kMB * m16.y + 2.4e-7f * fabsf(c.y) + errE;
    }
    float best_cost = INFINITY, best_err = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxCand; ++k) {
      const float ck = k <= nk ? cost[k] : INFINITY;
      const bool take = ck < best_cost;
      best = take ? c_lo + k : best;
      best_err = take ? errk[k] : best_err;
      best_cost = fminf(best_cost, ck);
    }
    const int kb = best - c_lo;
    const float ub = best_cost + best_err;
    float lo_min = INFINITY;
#pragma unroll
    for (int k = 0; k < kMaxCand; ++k)
      if (k <= nk && k != kb) lo_min = fminf(lo_min, cost[k] - errk[k]);
    if (lo_min > ub) {
      if (want_iv) {
        // gap_c(d) >= (cost_c - err_c) - ub, less 4e-6 (|cost_c| + |cost_b|)
        // for the FP32 evaluation of that bound and the reference's double
        // roundings. gap_c reaches 0 at d' - d = gap_c / (2 eta (c - b)),
        // formed with approximate reciprocals (rel. error < 1e-6) and shrunk
        // by 1e-4 relative.
        float dn = -INFINITY, up = INFINITY;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < kMaxCand; ++k) {
          if (k > nk || k == kb) continue;
          const float gap =
              (cost[k] - errk[k]) - ub - 4e-6f * (fabsf(cost[k]) + fabsf(best_cost));
          ok = ok && gap > 0.f;
          float r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)(k - kb)));
          const float t = gap * a.inv2eta_f * r * 0.9999f;
          if (t > 0.f) up = fminf(up, t);
          else if (t < 0.f) dn = fmaxf(dn, t);
        }
        if (ok) iv = iv_finish(a, dv, (double)dn, (double)up, c_lo, c_hi);
      }
      return best;
    }
    // Ambiguous: FP64 costs (exact E, exact clamped/undefined M) with error
    // bars on the fp16-derived M only.
    double bc = INFINITY, up = INFINITY;
    for (int c = c_lo; c <= c_hi; ++c) {
      double cost, err;
      repick_cost_d(a, u, c, dv, wv, wb, W, half, cost, err);
      if (cost < bc) {
        bc = cost;
        best = c;
      }
      up = fmin(up, cost + err);
    }
    int mask = 0, approx = 0;
    for (int c = c_lo; c <= c_hi; ++c) {
      double cost, err;
      repick_cost_d(a, u, c, dv, wv, wb, W, half, cost, err);
      if (cost - err <= up) {
        mask |= 1 << (c - c_lo);
        if (err != 0.0) approx |= 1 << (c - c_lo);
      }
    }
    // A single survivor, or survivors whose costs are all reference-exact
    // doubles (first minimum already taken), is the reference's pick.
    if (__popc(mask) == 1 || approx == 0) {
      if (want_iv) {
        // certificate from the same bounds: gap_c >= (cost_c - err_c) -
        // (cost_b + err_b), less a safety for the double roundings
        double cb, eb;
        repick_cost_d(a, u, best, dv, wv, wb, W, half, cb, eb);
        const double ub = cb + eb;
        double dn = -INFINITY, upv = INFINITY;
        bool ok = true;
        for (int c = c_lo; c <= c_hi; ++c) {
          if (c == best) continue;
          double cost, err;
          repick_cost_d(a, u, c, dv, wv, wb, W, half, cost, err);
          const double gap = (cost - err) - ub - 1e-9 * (1.0 + fabs(ub));
          ok = ok && gap > 0.0;
          const double sl = 2.0 * a.eta * (double)(c - best);
          if (sl > 0.0) upv = fmin(upv, gap / sl * (1.0 - 1e-9));
          else if (sl < 0.0) dn = fmax(dn, gap / sl * (1.0 - 1e-9));
        }
        if (ok) iv = iv_finish(a, dv, dn, upv, c_lo, c_hi);
      }
      return best;
    }
    dmask = mask;
    return INT_MIN;
  }
  // Window miss: score every candidate exactly.
  dmask = (1 << (c_hi - c_lo + 1)) - 1;
  return INT_MIN;
}

}  // namespace

// Block = 32 rows (lanes) x 32 columns (16 warps x 2). Everything a block
// needs is issued up front — the psum tile (bulk copies) and, per pixel, the
// scalars and the 32-byte score window (coalesced: a warp's 32 pixels are one
// 1 KB line run) — and consumed after one barrier.
template <int RF, bool USE_SO>
__global__ void __launch_bounds__(kThreads, 2)
    k_d_repick(const double* __restrict__ psumT, const uint8_t* __restrict__ mT,
               const int* __restrict__ cntT, const double* __restrict__ avgT,
               const int* __restrict__ soT, double* __restrict__ dT, int* __restrict__ oT,
               const uint8_t* __restrict__ lgray, const uint8_t* __restrict__ rgray,
               const wscore_t* __restrict__ win, const int* __restrict__ wbase,
               int2* __restrict__ chg, unsigned* __restrict__ chg_count,
               Deferred* __restrict__ defer, unsigned* __restrict__ defer_count,
               float2* __restrict__ ivT, RefineArgs a,
               long gray_stride, const __grid_constant__ CUtensorMap map, int glob) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar, bar_win;
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H, R = RF > 0 ? RF : a.radius;
  const long bs = bt_frame(W, H, 0);
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int v = blockIdx.y * 32 + lane;
  // The score windows (a third of the bytes) land on their own barrier,
  // waited for only before the re-picks: the disc gathers start as soon as
  // the psum box and the scalars are in.
  if (tid == 0 && win) {
    mbar_init(&bar_win, 1);
    mbar_fence_init();
  }
  const int u0 = blockIdx.x * kTC, rb = blockIdx.y;
  const int ncols = min(kTC, W - u0);
  const unsigned npx = ncols * 32;
  const long e0 = f * bs + ((long)rb * W + u0) * 32;  // first BT entry of the tile
  const size_t tb = glob ? 0 : tile_bytes<double>(R);
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + tb);
  double* s_av = reinterpret_cast<double*>(smem + tb + kWinSmem);
  int* s_so = reinterpret_cast<int*>(s_av);
  int* s_cnt = reinterpret_cast<int*>(s_av + kTilePx);
  int* s_o = s_cnt + kTilePx;
  int* s_wb = s_o + kTilePx;
  uint8_t* s_m = reinterpret_cast<uint8_t*>(s_wb + kTilePx);
  // wbase, S_o + o (or avg), cnt, mask (the windows: bar_win)
  const unsigned extra = (win ? npx * 4 : 0) + npx * 8 + npx * 4 + npx;
  const Tile<double> P = tile_issue<RF>(reinterpret_cast<double*>(smem),
                                        psumT + f * bt_frame(W, H, 1 + R), &map, W, R, glob, &bar,
                                        extra);
  if (tid == 0) {
    // the tile's per-pixel fields: contiguous BT ranges of npx entries
    if (win) bulk_g2s(s_wb, wbase + e0, npx * 4, &bar);
    if (USE_SO) {
      bulk_g2s(s_so, soT + e0, npx * 4, &bar);
      bulk_g2s(s_o, oT + e0, npx * 4, &bar);
    } else {
      bulk_g2s(s_av, avgT + e0, npx * 8, &bar);
    }
    bulk_g2s(s_cnt, cntT + e0, npx * 4, &bar);
    bulk_g2s(s_m, mT + e0, npx, &bar);
    if (win) {
      mbar_expect_tx(&bar_win, (kWin / 2) * npx * 4);
      const uint32_t* wsrc = reinterpret_cast<const uint32_t*>(win) + f * bs * (kWin / 2);
#pragma unroll 1
      for (int j = 0; j < kWin / 2; ++j)
        bulk_g2s(planes + j * kWinPlane, wsrc + (((long)rb * (kWin / 2) + j) * W + u0) * 32,
                 npx * 4, &bar_win);
    }
  }
  tile_wait(&bar);
  bool win_ready = win == nullptr;
  const uint8_t* L = lgray + f * gray_stride;
  const uint8_t* Rg = rgray + f * gray_stride;
#pragma unroll 1
  for (int k = 0; k < kPX; ++k) {
    const int t = warp + kTWarps * k;  // tile column
    const int slot = t * 32 + lane;
    if (t >= ncols || v >= H || !s_m[slot]) continue;
    const int u = u0 + t;
    const long px = ((long)rb * W + u) * 32 + lane;  // frame-local BT index
    const long bi = f * bs + px;
    const int cnk = s_cnt[slot];
    const int olk = USE_SO ? s_o[slot] : 0;
    const int wbk = win ? s_wb[slot] : kNoWin;
    const WinView wv{planes + slot, kWinPlane};
    const double s = disc_sum_any<RF>(P, a.span, W, H, u, v, R);
    const double c = (double)cnk;
    const double bav = __ddiv_rn(s, c);
    // avg = s_o / c: with integer o the reference's double disc sum is exact,
    // so the integer sum reproduces it bit for bit.
    const double a_o = USE_SO ? __ddiv_rn((double)s_so[slot], c) : s_av[slot];
    const double x = __dsub_rn(a_o, bav);
    const double dv = x < a.lo ? a.lo : (a.hi < x ? a.hi : x);  // std::clamp
    dT[bi] = dv;
    if (!win_ready) {
      mbar_wait(&bar_win, 0);
      win_ready = true;
    }
    int dclo, dmask;
    float2 iv;
    int best = repick(a, u, v, dv, L, Rg, win != nullptr, wv, wbk, dclo, dmask, iv,
                      ivT != nullptr);
    if (ivT) ivT[bi] = iv;  // empty when the pick is deferred
    if (best == INT_MIN && dmask)
      best = defer_pixel(defer + f * bs, defer_count + f, px, dclo, dmask, dv);
    if (best != INT_MIN) {
      if (!USE_SO) {
        oT[bi] = best;
      } else if (best != olk) {  // o only changes for a few hundred pixels per frame
        chg[f * bs + atomicAdd(chg_count + f, 1u)] = make_int2((int)px, best - olk);
        oT[bi] = best;
      }
    }
  }
  // the window copies must land before the block's shared memory is released
  if (!win_ready) mbar_wait(&bar_win, 0);
}

void launch_d_repick(const double* psumT, const uint8_t* mT, const int* cntT,
                     const double* avgT, const int* soT, double* dT, int* oT,
                     const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                     const int* wbase, int2* chg, unsigned* chg_count, Deferred* defer,
                     unsigned* defer_count, float2* ivT, const RefineArgs& a, int frames,
                     long gray_stride, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  CUtensorMap map;
  const bool tile = psum_map(&map, psumT, a, frames, use_tile<double>(a.radius, kWinSmem + kPxSmem));
  const size_t smem = (tile ? tile_bytes<double>(a.radius) : 0) + kWinSmem + kPxSmem;
  dim3 grid((a.g.W + kTC - 1) / kTC, (a.g.H + 31) / 32, frames);
  dim3 bl(32, kTWarps);
#define SS_REPICK_ARGS                                                                        \
  psumT, mT, cntT, avgT, soT, dT, oT, lgray, rgray, win, wbase, chg, chg_count, defer,        \
      defer_count, ivT, a, gray_stride
  if (a.radius == 15 && tile) {
    static bool configured = false;
    if (!configured) {
      set_smem(k_d_repick<15, false>, smem);
      set_smem(k_d_repick<15, true>, smem);
      configured = true;
    }
    if (avgT) k_d_repick<15, false><<<grid, bl, smem, s>>>(SS_REPICK_ARGS, map, 0);
    else k_d_repick<15, true><<<grid, bl, smem, s>>>(SS_REPICK_ARGS, map, 0);
  } else {
    set_smem(k_d_repick<0, false>, smem);
    set_smem(k_d_repick<0, true>, smem);
    if (avgT) k_d_repick<0, false><<<grid, bl, smem, s>>>(SS_REPICK_ARGS, map, tile ? 0 : 1);
    else k_d_repick<0, true><<<grid, bl, smem, s>>>(SS_REPICK_ARGS, map, tile ? 0 : 1);
  }
#undef SS_REPICK_ARGS
}

// ---- certified path (window 11, radius 15 tile): gather + listed re-picks ----
//
// Iterations >= 1 (iteration 0 is k_d_repick, which stores the first
// certificates). k_d_gather: the b-disc gather, d = clamp(S_o / cnt -
// avg(b)) stored for every masked pixel, and the pixel listed for a re-pick
// unless d falls inside its certificate interval. k_repick_list: one thread
// per listed pixel (score window read from the global BT planes), the
// interval of the new pick stored, the block's exact settles spread over its
// warps (no deferred list, no extra launch).
__global__ void __launch_bounds__(kThreads, 3)
    k_d_gather(const double* __restrict__ psumT, const uint8_t* __restrict__ mT,
               const int* __restrict__ cntT, const int* __restrict__ soT,
               const float2* __restrict__ ivT,
               double* __restrict__ dT, int* __restrict__ list, unsigned* __restrict__ list_count,
               RefineArgs a, const __grid_constant__ CUtensorMap map) {
  constexpr int RF = 15;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const long f = blockIdx.z;
  const int W = a.g.W, H = a.g.H;
  const long bs = bt_frame(W, H, 0);
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int v = blockIdx.y * 32 + lane;
  const int u0 = blockIdx.x * kTC, rb = blockIdx.y;
  const int ncols = min(kTC, W - u0);
  const unsigned npx = ncols * 32;
  const long e0 = f * bs + ((long)rb * W + u0) * 32;
  const size_t tb = tile_bytes<double>(RF);
  float2* s_iv = reinterpret_cast<float2*>(smem + tb);
  int* s_so = reinterpret_cast<int*>(s_iv + kTilePx);
  int* s_cnt = s_so + kTilePx;
  uint8_t* s_m = reinterpret_cast<uint8_t*>(s_cnt + kTilePx);
  const unsigned extra = npx * (4 + 8 + 4 + 1);
  const Tile<double> P = tile_issue<RF>(reinterpret_cast<double*>(smem),
                                        psumT + f * bt_frame(W, H, 1 + RF), &map, W, RF, false,
                                        &bar, extra);
  if (lane == 0 && warp == 0) {
    bulk_g2s(s_iv, ivT + e0, npx * 8, &bar);
    bulk_g2s(s_so, soT + e0, npx * 4, &bar);
    bulk_g2s(s_cnt, cntT + e0, npx * 4, &bar);
    bulk_g2s(s_m, mT + e0, npx, &bar);
  }
  tile_wait(&bar);
#pragma unroll 1
  for (int k = 0; k < kPX; ++k) {
    const int t = warp + kTWarps * k;  // tile column (warp-uniform)
    if (t >= ncols) break;
    const int slot = t * 32 + lane;
    const int u = u0 + t;
    const long px = ((long)rb * W + u) * 32 + lane;
    bool need = false;
    if (v < H && s_m[slot]) {
      const double s = disc_sum_any<RF>(P, a.span, W, H, u, v, RF);
      const double c = (double)s_cnt[slot];
      const double bav = __ddiv_rn(s, c);
      // avg = S_o / c: with integer o the reference's double disc sum is
      // exact, so the integer sum reproduces it bit for bit
      const double a_o = __ddiv_rn((double)s_so[slot], c);
      const double x = __dsub_rn(a_o, bav);
      const double dv = x < a.lo ? a.lo : (a.hi < x ? a.hi : x);  // std::clamp
      dT[f * bs + px] = dv;
      const float2 iv = s_iv[slot];
      need = !((double)iv.x <= dv && dv <= (double)iv.y);
    }
    warp_append(list + f * bs, list_count + f, need, (int)px);
  }
}

template <bool USE_SO>
__global__ void __launch_bounds__(256)
    k_repick_list(const int* __restrict__ list, const unsigned* __restrict__ list_count,
                  const double* __restrict__ dT,
                  int* __restrict__ oT,
                  const uint8_t* __restrict__ lgray, const uint8_t* __restrict__ rgray,
                  const wscore_t* __restrict__ win, const int* __restrict__ wbase,
                  float2* __restrict__ ivT, int2* __restrict__ chg, unsigned* __restrict__ chg_count,
                  RefineArgs a, long gray_stride, unsigned long long* __restrict__ counters) {
  const long f = blockIdx.y;
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const long bs = bt_frame(W, H, 0);
  const unsigned n = list_count[f];
  const int lane = threadIdx.x & 31;
  const uint8_t* L = lgray + f * gray_stride;
  const uint8_t* R = rgray + f * gray_stride;
  const uint32_t* wplanes = reinterpret_cast<const uint32_t*>(win) + f * bs * (kWin / 2);
  constexpr int kQ = 256;  // block size: one queue entry per thread at most
  __shared__ int q_px[kQ], q_clo[kQ], q_old[kQ];
  __shared__ double q_d[kQ];
  __shared__ unsigned q_n;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned n_scored = 0;
  auto finalize = [&](long bi, int px, int best, int old, float2 iv) {
    ivT[bi] = iv;
    if (best != INT_MIN) {
      if (!USE_SO) {
        oT[bi] = best;
      } else if (best != old) {
        chg[f * bs + atomicAdd(chg_count + f, 1u)] = make_int2(px, best - old);
        oT[bi] = best;
      }
    }
  };
  // block-uniform rounds of blockDim.x entries: the filter per thread, then
  // the round's exact settles spread over the block's warps
  for (unsigned b0 = blockIdx.x * blockDim.x; b0 < n; b0 += gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) q_n = 0;
    __syncthreads();
    const unsigned i = b0 + threadIdx.x;
    const bool act = i < n;
    const int px = act ? list[f * bs + i] : 0;
    n_scored += __popc(__ballot_sync(0xffffffffu, act));
    int v, u;
    bt_decode(W, px, v, u);
    const long bi = f * bs + px;
    if (act) {
      const double dv = dT[bi];
      const int old = USE_SO ? oT[bi] : 0;
      const WinView wv{wplanes + win_word(W, v, u, 0), (long)W * 32};
      int dclo = 0, dmask = 0;
      float2 iv;
      const int best = repick(a, u, v, dv, L, R, true, wv, wbase[bi], dclo, dmask, iv, true);
      if (best == INT_MIN && dmask != 0) {
        const unsigned k = atomicAdd(&q_n, 1u);
        q_px[k] = px;
        q_clo[k] = dclo;
        q_old[k] = old;
        q_d[k] = dv;
      } else {
        finalize(bi, px, best, old, iv);
      }
    }
    __syncthreads();
    // exact settles: a warp scores one queued pixel's candidates (lane k:
    // c_lo + k) and takes the first minimum, as smoothing.cpp:138 does;
    // every candidate is scored (the lanes run in parallel anyway), so the
    // pick's certificate comes out of the same costs
    const unsigned nq = q_n;
    if (counters && threadIdx.x == 0 && nq) atomicAdd(counters, (unsigned long long)nq);
    for (unsigned q = warp; q < nq; q += nw) {
      const int qpx = q_px[q], pc = q_clo[q];
      const double pd = q_d[q];
      int pv, pu;
      bt_decode(W, qpx, pv, pu);
      const int pch = min((int)floor(__dadd_rn(pd, (double)kRefineR)), (int)floor(a.hi));
      const int pm = (1 << (pch - pc + 1)) - 1;
      const bool fits = pu >= half && pu < W - half && pv >= half && pv < H - half;
      const bool mine = lane < kMaxCand && ((pm >> lane) & 1);
      double mycost = INFINITY;
      if (mine) mycost = exact_cost(L, R, W, pu, pv, pc + lane, fits, half, pd, a.eta);
      double cost = mycost;
      int k = mine ? lane : 64;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_down_sync(0xffffffffu, cost, o);
        const int ok = __shfl_down_sync(0xffffffffu, k, o);
        if (oc < cost || (oc == cost && ok < k)) {
          cost = oc;
          k = ok;
        }
      }
      k = __shfl_sync(0xffffffffu, k, 0);
      // The reference's own costs of every candidate: the pick's certificate
      // interval follows as on the exact no-window path (gaps known to the
      // reference's roundings).
      float2 piv = iv_empty();
      if (k < 64) {
        const double cb = __shfl_sync(0xffffffffu, mycost, k);
        double up = INFINITY, dn = -INFINITY;
        bool ok = true;
        if (mine && lane != k) {
          const double gap = mycost - cb - 1e-9 * (1.0 + fabs(cb));
          ok = gap > 0.0;
          const double sl = 2.0 * a.eta * (double)(lane - k);
          if (sl > 0.0) up = gap / sl * (1.0 - 1e-9);
          else if (sl < 0.0) dn = gap / sl * (1.0 - 1e-9);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          up = fmin(up, __shfl_xor_sync(0xffffffffu, up, o));
          dn = fmax(dn, __shfl_xor_sync(0xffffffffu, dn, o));
        }
        if (__all_sync(0xffffffffu, ok)) piv = iv_finish(a, pd, dn, up, pc, pch);
      }
      if (lane == 0) finalize(f * bs + qpx, qpx, k < 64 ? pc + k : INT_MIN, q_old[q], piv);
    }
    __syncthreads();  // the queue is reset by the next round
  }
  // counters[1] (ctx counter 2): (pixel, iteration) re-picks scored (the rest were certified)
  if (counters && lane == 0 && n_scored) atomicAdd(counters + 1, (unsigned long long)n_scored);
}

bool certified_repick_ok(const RefineArgs& a, bool has_win) {
  return has_win && a.radius == 15 &&
         use_tile<double>(15, (size_t)kTilePx * (8 + 8 + 4 + 1));
}

void launch_d_gather(const double* psumT, const uint8_t* mT, const int* cntT, const int* soT,
                     const float2* ivT, double* dT, int* list, unsigned* list_count,
                     const RefineArgs& a, int frames, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  CUtensorMap map;
  if (!psum_map(&map, psumT, a, frames, true))
    throw std::runtime_error("k_d_gather: TMA tensor map rejected");
  const size_t smem = tile_bytes<double>(15) + (size_t)kTilePx * (8 + 4 + 4 + 1);
  static bool configured = false;
  if (!configured) {
    set_smem(k_d_gather, smem);
    configured = true;
  }
  dim3 grid((a.g.W + kTC - 1) / kTC, (a.g.H + 31) / 32, frames);
  k_d_gather<<<grid, dim3(32, kTWarps), smem, s>>>(psumT, mT, cntT, soT, ivT, dT, list,
                                                   list_count, a, map);
}

void launch_repick_list(const int* list, const unsigned* list_count, const double* dT, int* oT,
                        const uint8_t* lgray, const uint8_t* rgray, const wscore_t* win,
                        const int* wbase, float2* ivT, int2* chg, unsigned* chg_count,
                        const RefineArgs& a, int frames, long gray_stride,
                        unsigned long long* counters, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  // the lists hold a few percent of the pixels
  k_repick_list<true><<<dim3(48, frames), 256, 0, s>>>(list, list_count, dT, oT, lgray, rgray,
                                                        win, wbase, ivT, chg, chg_count, a,
                                                        gray_stride, counters);
}

// Deferred re-picks: one warp per pixel, lane k scores candidate c_lo + k in
// exact FP64 (zncc_exact, reference cost formula); the warp takes the first
// minimum (smallest candidate among equal costs), as smoothing.cpp:138 does.
__global__ void k_repick_exact(const Deferred* __restrict__ defer,
                               const unsigned* __restrict__ defer_count, int* __restrict__ oT,
                               const uint8_t* __restrict__ lgray,
                               const uint8_t* __restrict__ rgray, int2* __restrict__ chg,
                               unsigned* __restrict__ chg_count, RefineArgs a, long gray_stride,
                               unsigned long long* __restrict__ counters) {
  const long f = blockIdx.y;
  const unsigned n = defer_count[f];
  if (blockIdx.x == 0 && threadIdx.x == 0 && counters) atomicAdd(counters, (unsigned long long)n);
  const int lane = threadIdx.x & 31;
  const int W = a.g.W, H = a.g.H, half = a.g.half;
  const long bs = bt_frame(W, H, 0);
  const uint8_t* L = lgray + f * gray_stride;
  const uint8_t* R = rgray + f * gray_stride;
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  for (unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nwarps) {
    const Deferred e = defer[f * bs + t];
    int u, v;
    bt_decode(W, e.pix, v, u);
    const bool fits = u >= half && u < W - half && v >= half && v < H - half;
    const bool mine = lane < kMaxCand && ((e.mask >> lane) & 1);
    double cost = INFINITY;
    if (mine) cost = exact_cost(L, R, W, u, v, e.c_lo + lane, fits, half, e.d, a.eta);
    int k = mine ? lane : 64;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oc = __shfl_down_sync(0xffffffffu, cost, off);
      const int ok = __shfl_down_sync(0xffffffffu, k, off);
      if (oc < cost || (oc == cost && ok < k)) {
        cost = oc;
        k = ok;
      }
    }
    if (lane == 0 && k < 64) {
      const int best = e.c_lo + k;
      const long i = f * bs + e.pix;
      if (chg) {
        const int old = oT[i];
        if (best != old)
          chg[f * bs + atomicAdd(chg_count + f, 1u)] = make_int2(e.pix, best - old);
      }
      oT[i] = best;
    }
  }
}

void launch_repick_exact(const Deferred* defer, const unsigned* defer_count, int* oT,
                         const uint8_t* lgray, const uint8_t* rgray, int2* chg,
                         unsigned* chg_count, const RefineArgs& a, int frames, long gray_stride,
                         unsigned long long* counters, cudaStream_t s) {
  if (frames <= 0) return;
  k_repick_exact<<<dim3(64, frames), 256, 0, s>>>(defer, defer_count, oT, lgray, rgray, chg,
                                                  chg_count, a, gray_stride, counters);
}

// One warp per changed pixel j: S_o(i) += delta_j for every valid i whose disc
// contains j. The relation is symmetric (|dx| <= span(|dy|) <=> dx^2 + dy^2 <=
// R^2) and clipped to the image exactly as the reference's row spans are.
// Lanes walk rows (contiguous in BT), the loop walks columns.
__global__ void k_so_update(const int2* __restrict__ chg, const unsigned* __restrict__ chg_count,
                            const uint8_t* __restrict__ mT, int* __restrict__ soT,
                            RefineArgs a) {
  const long f = blockIdx.y;
  const int W = a.g.W, H = a.g.H, R = a.radius;
  const long bs = bt_frame(W, H, 0);
  const unsigned n = chg_count[f];
  const int lane = threadIdx.x & 31;
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  for (unsigned t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += nwarps) {
    const int2 e = chg[f * bs + t];
    int v, u;
    bt_decode(W, e.x, v, u);
    const int xlo = max(0, u - R), xhi = min(W - 1, u + R);
    for (int dy0 = -R; dy0 <= R; dy0 += 32) {
      const int dy = dy0 + lane, y = v + dy;
      const bool rok = dy <= R && y >= 0 && y < H;
      const int sy = rok ? __ldg(a.span + (dy < 0 ? -dy : dy)) : -1;
      const long rowbase = rok ? f * bs + ((long)(y >> 5) * W) * 32 + (y & 31) : 0;
      for (int x = xlo; x <= xhi; ++x) {
        const int dx = x - u;
        // unmasked targets are updated too: their S_o is never read (k_scan_b
        // and k_d_repick use it under the mask), which saves the mask loads
        if ((dx < 0 ? -dx : dx) <= sy) atomicAdd(soT + rowbase + (long)x * 32, e.y);
      }
    }
  }
}

void launch_so_update(const int2* chg, const unsigned* chg_count, const uint8_t* mT, int* soT,
                      const RefineArgs& a, int frames, cudaStream_t s) {
  if (a.g.W <= 0 || a.g.H <= 0 || frames <= 0) return;
  k_so_update<<<dim3(148, frames), 256, 0, s>>>(chg, chg_count, mT, soT, a);
}

}  // namespace ssb
