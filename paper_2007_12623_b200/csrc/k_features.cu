// Feature front end on the GPU: features.cpp:86-208.
//
//   k_fast_score     segment-test corner score per pixel (features.cpp:22-48):
//                    16-pixel Bresenham circle, the largest margin over
//                    contiguous arcs of >= 9 pixels all brighter / darker by
//                    `threshold`. The best arc of a start is its 9-long one
//                    (the running minimum only falls as the arc grows), so
//                    score = max over 16 starts of the min of 9 consecutive
//                    circular diffs, when that min >= threshold. A compass
//                    test (any 9-arc covers >= 2 of the 4 compass pixels)
//                    rejects most pixels after 5 loads.
//   k_corner_keys    3x3 non-maximum suppression with the raster tie-break
//                    (features.cpp:99-111); survivors become 64-bit keys
//                    (0xFFFF - score, v, u) so one ascending radix sort (CUB)
//                    gives score descending, ties in raster order
//                    (features.cpp:116-121), then truncation to max_count.
//   k_describe       one warp per corner: 256 comparisons of 5x5 box sums at
//                    the seeded pattern (features.cpp:52-70,126-166; the
//                    pattern is drawn on the host with the same std::mt19937
//                    stream), lane l decides bits l + 32 k, ballots assemble
//                    the 4 x 64-bit words. Box sums are exact integers, as the
//                    reference's integral-image differences.
//   k_match_best     brute-force Hamming nearest neighbour, first minimum
//                    (features.cpp:172-194), both directions; k_match_mutual
//                    keeps mutual pairs within max_hamming in index_a order.
// All integer work: results are bit-identical to the reference.
#include <cub/device/device_radix_sort.cuh>

#include "ss_internal.cuh"

namespace ssb {

namespace {
__constant__ int c_cu[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
__constant__ int c_cv[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};
__constant__ int4 c_pat[256];  // ax, ay, bx, by
}  // namespace

void upload_feature_pattern(const int* pat4x256, cudaStream_t s) {
  cudaMemcpyToSymbolAsync(c_pat, pat4x256, sizeof(int4) * 256, 0, cudaMemcpyHostToDevice, s);
}

__device__ __forceinline__ int arc_best(const int (&d)[16], int thr) {
  int best = 0;
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    int m = d[s];
#pragma unroll
    for (int k = 1; k < 9; ++k) m = min(m, d[(s + k) & 15]);
    best = m >= thr ? max(best, m) : best;
  }
  return best;
}

__global__ void k_fast_score(const uint8_t* __restrict__ g, int* __restrict__ score, int W, int H,
                             int thr) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= W || v >= H) return;
  int s = 0;
  if (u >= 3 && u < W - 3 && v >= 3 && v < H - 3) {
    const uint8_t* row = g + (long)v * W + u;
    const int c = row[0];
    // compass pixels 0, 4, 8, 12 (N, E, S, W)
    const int n0 = row[-3 * W], n4 = row[3], n8 = row[3 * W], n12 = row[-3];
    const int bc = (n0 - c >= thr) + (n4 - c >= thr) + (n8 - c >= thr) + (n12 - c >= thr);
    const int dc = (c - n0 >= thr) + (c - n4 >= thr) + (c - n8 >= thr) + (c - n12 >= thr);
    if (bc >= 2 || dc >= 2) {
      int b[16], d[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int p = row[c_cv[i] * W + c_cu[i]];
        b[i] = p - c;
        d[i] = c - p;
      }
      s = max(bc >= 2 ? arc_best(b, thr) : 0, dc >= 2 ? arc_best(d, thr) : 0);
    }
  }
  score[(long)v * W + u] = s;
}

__global__ void k_corner_keys(const int* __restrict__ score, int W, int H,
                              unsigned long long* __restrict__ keys,
                              unsigned* __restrict__ count) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u < 3 || u >= W - 3 || v < 3 || v >= H - 3) return;
  const int s = score[(long)v * W + u];
  if (s <= 0) return;
#pragma unroll
  for (int dv = -1; dv <= 1; ++dv)
#pragma unroll
    for (int du = -1; du <= 1; ++du) {
      if (du == 0 && dv == 0) continue;
      const int ns = score[(long)(v + dv) * W + u + du];
      if (ns > s || (ns == s && (dv < 0 || (dv == 0 && du < 0)))) return;
    }
  keys[atomicAdd(count, 1u)] = ((unsigned long long)(0xFFFF - s) << 32) |
                               ((unsigned long long)v << 16) | (unsigned long long)u;
}

// Sort n keys (ascending) into keys_out; tmp/tmp_bytes: CUB scratch
// (tmp == nullptr: *tmp_bytes receives the size needed).
cudaError_t sort_corner_keys(void* tmp, size_t* tmp_bytes, const unsigned long long* keys,
                             unsigned long long* keys_out, int n, cudaStream_t s) {
  return cub::DeviceRadixSort::SortKeys(tmp, *tmp_bytes, keys, keys_out, n, 0, 48, s);
}

__global__ void k_keys_to_corners(const unsigned long long* __restrict__ keys, int n,
                                  int* __restrict__ cu, int* __restrict__ cv,
                                  int* __restrict__ cs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  cu[i] = (int)(k & 0xFFFF);
  cv[i] = (int)((k >> 16) & 0xFFFF);
  cs[i] = 0xFFFF - (int)(k >> 32);
}

__device__ __forceinline__ int box5(const uint8_t* g, int W, int u, int v) {
  int s = 0;
#pragma unroll
  for (int dy = -2; dy <= 2; ++dy) {
    const uint8_t* r = g + (long)(v + dy) * W + u;
#pragma unroll
    for (int dx = -2; dx <= 2; ++dx) s += __ldg(r + dx);
  }
  return s;
}

// One warp per corner; keep[i] = 1 and desc[i] filled when the 31x31 patch
// (plus the box radius) is inside the image (features.cpp:152-156).
__global__ void k_describe(const uint8_t* __restrict__ g, int W, int H,
                           const int* __restrict__ cu, const int* __restrict__ cv, int n,
                           unsigned long long* __restrict__ desc, int* __restrict__ keep) {
  constexpr int kBorder = 16;  // kPatchBorder, features.cpp:72
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int u = cu[i], v = cv[i];
  const bool in = u >= kBorder && u < W - kBorder && v >= kBorder && v < H - kBorder;
  if (lane == 0) keep[i] = in ? 1 : 0;
  if (!in) return;
  unsigned word[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int4 p = c_pat[32 * k + lane];
    const int a = box5(g, W, u + p.x, v + p.y);
    const int b = box5(g, W, u + p.z, v + p.w);
    word[k] = __ballot_sync(0xffffffffu, a < b);
  }
  if (lane < 4)
    desc[4L * i + lane] = (unsigned long long)word[2 * lane] |
                          ((unsigned long long)word[2 * lane + 1] << 32);
}

// Order-preserving compaction of the kept features (one block, running offset).
__global__ void k_compact_features(const int* __restrict__ keep, int n,
                                   const int* __restrict__ cu, const int* __restrict__ cv,
                                   const unsigned long long* __restrict__ desc_in,
                                   double* __restrict__ pos, unsigned long long* __restrict__ desc,
                                   int* __restrict__ n_out) {
  __shared__ int warp_sums[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const int k = i < n ? keep[i] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 31) warp_sums[wid] = pre + k;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      off += w < wid ? warp_sums[w] : 0;
      tot += warp_sums[w];
    }
    if (k) {
      const int o = base + off + pre;
      pos[2L * o] = (double)cu[i];
      pos[2L * o + 1] = (double)cv[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) desc[4L * o + q] = desc_in[4L * i + q];
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = base;
}

// best[i] = first j minimising Hamming(a_i, b_j) (features.cpp:176-184).
__global__ void k_match_best(const unsigned long long* __restrict__ da, int na,
                             const unsigned long long* __restrict__ db, int nb,
                             int* __restrict__ best, int* __restrict__ best_d) {
  __shared__ ulonglong4 sb[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  ulonglong4 a = make_ulonglong4(0, 0, 0, 0);
  if (i < na) a = reinterpret_cast<const ulonglong4*>(da)[i];
  int bj = -1, bd = 257;
  for (int j0 = 0; j0 < nb; j0 += 256) {
    __syncthreads();
    if (j0 + (int)threadIdx.x < nb) sb[threadIdx.x] = reinterpret_cast<const ulonglong4*>(db)[j0 + threadIdx.x];
    __syncthreads();
    const int m = min(256, nb - j0);
    for (int t = 0; t < m; ++t) {
      const ulonglong4 b = sb[t];
      const int d = __popcll(a.x ^ b.x) + __popcll(a.y ^ b.y) + __popcll(a.z ^ b.z) +
                    __popcll(a.w ^ b.w);
      if (d < bd) {
        bd = d;
        bj = j0 + t;
      }
    }
  }
  if (i < na) {
    best[i] = bj;
    best_d[i] = bd;
  }
}

__global__ void k_match_mutual(const int* __restrict__ best_b, const int* __restrict__ best_b_d,
                               const int* __restrict__ best_a, int na, int max_hamming,
                               int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const int j = best_b[i];
  keep[i] = (j >= 0 && best_a[j] == i && best_b_d[i] <= max_hamming) ? 1 : 0;
}

// Order-preserving compaction of the mutual matches (one block).
__global__ void k_compact_matches(const int* __restrict__ keep, int na,
                                  const int* __restrict__ best_b, const int* __restrict__ best_b_d,
                                  const double* __restrict__ pos_a,
                                  const double* __restrict__ pos_b, int* __restrict__ ia,
                                  int* __restrict__ ib, int* __restrict__ ham,
                                  double* __restrict__ disp, int* __restrict__ n_out) {
  __shared__ int warp_sums[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < na; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const int k = i < na ? keep[i] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 31) warp_sums[wid] = pre + k;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      off += w < wid ? warp_sums[w] : 0;
      tot += warp_sums[w];
    }
    if (k) {
      const int o = base + off + pre;
      const int j = best_b[i];
      ia[o] = i;
      ib[o] = j;
      ham[o] = best_b_d[i];
      // b.position - a.position (features.cpp:202), exact for pixel positions
      disp[2L * o] = __dsub_rn(pos_b[2L * j], pos_a[2L * i]);
      disp[2L * o + 1] = __dsub_rn(pos_b[2L * j + 1], pos_a[2L * i + 1]);
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = base;
}

// ---- launchers ----
void launch_fast_score(const uint8_t* g, int* score, int W, int H, int thr, cudaStream_t s) {
  dim3 b(32, 8), gr((W + 31) / 32, (H + 7) / 8);
  k_fast_score<<<gr, b, 0, s>>>(g, score, W, H, thr);
}
void launch_corner_keys(const int* score, int W, int H, unsigned long long* keys,
                        unsigned* count, cudaStream_t s) {
  dim3 b(32, 8), gr((W + 31) / 32, (H + 7) / 8);
  k_corner_keys<<<gr, b, 0, s>>>(score, W, H, keys, count);
}
void launch_keys_to_corners(const unsigned long long* keys, int n, int* cu, int* cv, int* cs,
                            cudaStream_t s) {
  if (n > 0) k_keys_to_corners<<<(n + 255) / 256, 256, 0, s>>>(keys, n, cu, cv, cs);
}
void launch_describe(const uint8_t* g, int W, int H, const int* cu, const int* cv, int n,
                     unsigned long long* desc_tmp, int* keep, double* pos,
                     unsigned long long* desc, int* n_out, cudaStream_t s) {
  if (n > 0) k_describe<<<(n * 32 + 255) / 256, 256, 0, s>>>(g, W, H, cu, cv, n, desc_tmp, keep);
  k_compact_features<<<1, 1024, 0, s>>>(keep, n, cu, cv, desc_tmp, pos, desc, n_out);
}
void launch_match(const unsigned long long* da, const double* pa, int na,
                  const unsigned long long* db, const double* pb, int nb, int max_hamming,
                  int* best_b, int* best_b_d, int* best_a, int* best_a_d, int* keep, int* ia,
                  int* ib, int* ham, double* disp, int* n_out, cudaStream_t s) {
  if (na > 0 && nb > 0) {
    k_match_best<<<(na + 255) / 256, 256, 0, s>>>(da, na, db, nb, best_b, best_b_d);
    k_match_best<<<(nb + 255) / 256, 256, 0, s>>>(db, nb, da, na, best_a, best_a_d);
    k_match_mutual<<<(na + 255) / 256, 256, 0, s>>>(best_b, best_b_d, best_a, na, max_hamming,
                                                    keep);
  }
  k_compact_matches<<<1, 1024, 0, s>>>(keep, (na > 0 && nb > 0) ? na : 0, best_b, best_b_d, pa,
                                       pb, ia, ib, ham, disp, n_out);
}

}  // namespace ssb
