// Per-SM issue rates of the instruction classes the stereo kernels are built
// from ("confirm the SM count and the INT32 and FP64 lane rates
// on the box by micro-benchmark"). Each kernel runs 8 independent dependency
// chains per thread over a long unrolled loop on every SM (one 1024-thread
// block per SM) and reports lane-ops per clock per SM, with the clock taken
// from clock64() deltas on the SMs themselves (so the rate does not depend on
// the boost clock the run happened to get).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/pipe_rates scripts/pipe_rates.cu
//   scripts/pipe_rates > profiles/r2/pipe_rates.json
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));             \
      return 1;                                                            \
    }                                                                      \
  } while (0)

constexpr int kIters = 32768;
constexpr int kChains = 8;

struct Clk {
  unsigned long long t0, t1;
};

__device__ __forceinline__ void clk_begin(Clk* c) {
  __syncthreads();
  if (threadIdx.x == 0) c[blockIdx.x].t0 = clock64();
}
__device__ __forceinline__ void clk_end(Clk* c) {
  __syncthreads();
  if (threadIdx.x == 0) c[blockIdx.x].t1 = clock64();
}

__global__ void k_iadd(int* out, int seed, Clk* c) {
  int a[kChains];
  for (int k = 0; k < kChains; ++k) a[k] = seed + threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k)  // add, xor alternate: ptxas cannot fold them into IADD3
      asm volatile("add.s32 %0, %0, %1;\n\txor.b32 %0, %0, %2;" : "+r"(a[k]) : "r"(seed), "r"(k));
  clk_end(c);
  int s = 0;
  for (int k = 0; k < kChains; ++k) s ^= a[k];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_imad(int* out, int seed, Clk* c) {
  int a[kChains];
  for (int k = 0; k < kChains; ++k) a[k] = seed + threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(seed), "r"(k));
  clk_end(c);
  int s = 0;
  for (int k = 0; k < kChains; ++k) s ^= a[k];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_dp4a(int* out, int seed, Clk* c) {
  unsigned a[kChains];
  for (int k = 0; k < kChains; ++k) a[k] = seed + threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("dp4a.u32.u32 %0, %1, %2, %0;" : "+r"(a[k]) : "r"(seed), "r"(0x01010101u));
  clk_end(c);
  unsigned s = 0;
  for (int k = 0; k < kChains; ++k) s ^= a[k];
  if (s == 0x7fffffffu) out[0] = (int)s;
}

__global__ void k_ffma(int* out, int seed, Clk* c) {
  float a[kChains];
  const float m = 1.0f + 1e-7f * seed, b = 1e-9f;
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(m), "f"(b));
  clk_end(c);
  float s = 0;
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == -1.f) out[0] = 1;
}

__global__ void k_dadd(int* out, int seed, Clk* c) {
  double a[kChains];
  const double b = 1e-12 * seed;
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(b));
  clk_end(c);
  double s = 0;
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == -1.0) out[0] = 1;
}

__global__ void k_dfma(int* out, int seed, Clk* c) {
  double a[kChains];
  const double m = 1.0 + 1e-15 * seed, b = 1e-12;
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x + k;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(m), "d"(b));
  clk_end(c);
  double s = 0;
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == -1.0) out[0] = 1;
}

// Shared-memory loads: lane-consecutive (conflict-free) addresses, W bytes per
// lane per instruction, results folded with one XOR per 32-bit word.
template <int W>
__global__ void k_lds(int* out, int seed, Clk* c) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u + seed;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  (void)warp;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + lane * W;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) {
    const uint32_t a = base + (i & 15) * 32 * W;  // immediate offsets once unrolled
    if constexpr (W == 4) {
      uint32_t x;
      asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
      acc ^= x;
    } else if constexpr (W == 8) {
      uint32_t x, y;
      asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
      acc ^= x ^ y;
    } else {
      uint32_t x, y, z, w;
      asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                   : "r"(a));
      acc ^= x ^ y ^ z ^ w;
    }
  }
  clk_end(c);
  if (acc == 0x12345678u) out[0] = (int)acc;
}

// Warp shuffles (32-bit, index from a register): lane-ops per clock.
__global__ void k_shfl(int* out, int seed, Clk* c) {
  uint32_t a[kChains];
  for (int k = 0; k < kChains; ++k) a[k] = seed + threadIdx.x + k;
  const int src = (threadIdx.x + 1) & 31;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("shfl.sync.idx.b32 %0, %0, %1, 31, -1;" : "+r"(a[k]) : "r"(src));
  clk_end(c);
  uint32_t s = 0;
  for (int k = 0; k < kChains; ++k) s ^= a[k];
  if (s == 0x7fffffffu) out[0] = (int)s;
}

// LDS.64 and 64-bit shuffles interleaved one to one: if the two share the
// shared-memory data path, the byte rate of the pair stays at the LDS rate.
__global__ void k_lds_shfl(int* out, int seed, Clk* c) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u + seed;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0, b0 = seed, b1 = seed + 1;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + lane * 8;
  const int src = (lane + 1) & 31;
  clk_begin(c);
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) {
    const uint32_t a = base + (i & 15) * 256;
    uint32_t x, y;
    asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
    asm volatile("shfl.sync.idx.b32 %0, %0, %2, 31, -1;\n\tshfl.sync.idx.b32 %1, %1, %2, 31, -1;"
                 : "+r"(b0), "+r"(b1) : "r"(src));
    acc ^= x ^ y;
  }
  clk_end(c);
  if ((acc ^ b0 ^ b1) == 0x12345678u) out[0] = (int)acc;
}

typedef void (*Kern)(int*, int, Clk*);

// lane-ops (or bytes) per clock per SM: a block's work over its cycle count
static int run(const char* name, Kern k, double work_per_thread, const char* unit, int nsm,
               int* d_out, Clk* d_clk, Clk* h_clk, bool last) {
  const int blocks_per_sm = 1, threads = 1024, nb = nsm * blocks_per_sm;
  k<<<nb, threads>>>(d_out, 3, d_clk);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nb, threads>>>(d_out, 3, d_clk);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  CK(cudaMemcpy(h_clk, d_clk, sizeof(Clk) * nb, cudaMemcpyDeviceToHost));
  double cyc = 0;
  for (int b = 0; b < nb; ++b) cyc += (double)(h_clk[b].t1 - h_clk[b].t0);
  cyc /= nb;  // one block per SM: a block's span is its SM's span
  const double per_sm = work_per_thread * threads * blocks_per_sm;
  printf("    \"%s\": {\"per_clk_per_sm\": %.2f, \"unit\": \"%s\", \"kernel_ms\": %.4f, "
         "\"implied_sm_mhz\": %.0f}%s\n",
         name, per_sm / cyc, unit, ms, cyc / (ms * 1e3), last ? "" : ",");
  return 0;
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  const int nsm = p.multiProcessorCount;
  int* d_out;
  Clk *d_clk, *h_clk;
  CK(cudaMalloc(&d_out, 16));
  CK(cudaMalloc(&d_clk, sizeof(Clk) * nsm));
  h_clk = new Clk[nsm];
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\n  \"device\": \"%s\", \"sm_count\": %d, \"sm_clock_max_mhz\": %d,\n", p.name, nsm,
         clk_khz / 1000);
  printf("  \"method\": \"8 independent chains per thread, one 1024-thread block per SM, "
         "clock64() cycles per block\",\n  \"rates\": {\n");
  const double ops = (double)kIters * kChains;
  int rc = 0;
  rc |= run("iadd_xor_s32", k_iadd, 2 * ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("imad_s32", k_imad, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("dp4a_u8", k_dp4a, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("ffma_f32", k_ffma, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("dadd_f64", k_dadd, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("dfma_f64", k_dfma, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  rc |= run("lds_32", k_lds<4>, (double)kIters * 4, "bytes", nsm, d_out, d_clk, h_clk, false);
  rc |= run("lds_64", k_lds<8>, (double)kIters * 8, "bytes", nsm, d_out, d_clk, h_clk, false);
  rc |= run("lds_128", k_lds<16>, (double)kIters * 16, "bytes", nsm, d_out, d_clk, h_clk, false);
  rc |= run("shfl_32", k_shfl, ops, "lane-ops", nsm, d_out, d_clk, h_clk, false);
  // pair rate: LDS.64 bytes per clock with two 32-bit shuffles beside each load
  rc |= run("lds_64_with_2_shfl", k_lds_shfl, (double)kIters * 8, "LDS bytes", nsm, d_out, d_clk,
            h_clk, true);
  printf("  }\n}\n");
  return rc;
}
