// Left-right consistency (opt-in, north_star: "winner-
// take-all disparity selection with left-right consistency"). The reference
// has no LR check (it only notes unmatched pixels), so this is
// an extension with its own CPU restatement in the test oracle (orc_compute_disparity_
// right, orc_lr_check) and is off unless asked for.
//
// Right-view WTA: d_R(x) = first argmax over d in [d_min, d_max] of
// zncc(L at x + d, R at x). The chessboard window is symmetric under
// du -> -du and the ZNCC statistics are symmetric in L and R, so the right
// view is the left-view sweep of the mirrored, swapped pair
// (L' = flip(R), R' = flip(L)) read back mirrored: k_flip_pair prepares it and
// the unmodified sweep + FP64 resolve run on it (bit-identical scores).
//
// k_lr_check: a valid left pixel u with disparity d stays valid iff
// x = u - d is inside the image, the right view is valid at x and
// |d_R(x) - d| <= max_diff; rejected pixels become (0, invalid), what the
// WTA itself writes for an unmatched pixel (matcher.cpp:172).
#include "ss_internal.cuh"

namespace ssb {

// out_l[f] = flip(gray_r[f]), out_r[f] = flip(gray_l[f]) (rows mirrored).
__global__ void k_flip_pair(const uint8_t* __restrict__ gl, const uint8_t* __restrict__ gr,
                            uint8_t* __restrict__ out_l, uint8_t* __restrict__ out_r, int W,
                            long stride) {
  const long f = blockIdx.z;
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
    const long i = f * stride + (long)y * W + x, m = f * stride + (long)y * W + (W - 1 - x);
    out_l[m] = gr[i];
    out_r[m] = gl[i];
  }
}

void launch_flip_pair(const uint8_t* gl, const uint8_t* gr, uint8_t* out_l, uint8_t* out_r,
                      int W, int H, int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_flip_pair<<<dim3((W + 255) / 256, H, frames), 256, 0, s>>>(gl, gr, out_l, out_r, W, stride);
}

// disp_rm / valid_rm: the right view in mirrored coordinates (x' = W-1-x).
__global__ void k_lr_check(float* __restrict__ disp, uint8_t* __restrict__ valid,
                           const float* __restrict__ disp_rm,
                           const uint8_t* __restrict__ valid_rm, int W, int H, float max_diff,
                           long stride) {
  const long f = blockIdx.z;
  const int y = blockIdx.y;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= W) return;
  const long i = f * stride + (long)y * W + u;
  if (!valid[i]) return;
  const float d = disp[i];  // integer-valued WTA pick
  const int x = u - (int)d;
  bool ok = x >= 0 && x < W;
  if (ok) {
    const long j = f * stride + (long)y * W + (W - 1 - x);
    ok = valid_rm[j] && fabsf(disp_rm[j] - d) <= max_diff;
  }
  if (!ok) {
    disp[i] = 0.f;
    valid[i] = 0;
  }
}

void launch_lr_check(float* disp, uint8_t* valid, const float* disp_rm, const uint8_t* valid_rm,
                     int W, int H, int max_diff, int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_lr_check<<<dim3((W + 255) / 256, H, frames), 256, 0, s>>>(disp, valid, disp_rm, valid_rm, W,
                                                              H, (float)max_diff, stride);
}

// Mirror a map back to image coordinates (per-stage API output of d_R).
__global__ void k_unflip_map(const float* __restrict__ dm, const uint8_t* __restrict__ vm,
                             float* __restrict__ d, uint8_t* __restrict__ v, int W, long stride) {
  const long f = blockIdx.z;
  const int y = blockIdx.y;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  const long i = f * stride + (long)y * W + x, m = f * stride + (long)y * W + (W - 1 - x);
  d[i] = dm[m];
  v[i] = vm[m];
}

void launch_unflip_map(const float* dm, const uint8_t* vm, float* d, uint8_t* v, int W, int H,
                       int frames, long stride, cudaStream_t s) {
  if (W <= 0 || H <= 0 || frames <= 0) return;
  k_unflip_map<<<dim3((W + 255) / 256, H, frames), 256, 0, s>>>(dm, vm, d, v, W, stride);
}

}  // namespace ssb
