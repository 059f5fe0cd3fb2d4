// Exact (reference-identical) chessboard ZNCC on the device.
//
// zncc_chessboard, matcher.cpp:38-64: int64 statistics over the taps with
// (du + dv) even, score = double(num) / sqrt(double(var_l * var_r)), IEEE
// round-to-nearest (CUDA's double sqrt and division are correctly rounded).
// `wta_semantics` reproduces compute_disparity's patch_stats, which stores
// sum and var as int32 (matcher.cpp:132-133): identical for window <= 19.
#pragma once

#include <stdint.h>

namespace ssb {

struct ExactScore {
  double score;
  bool defined;
};

// Window-11 tap sums, fully unrolled (all 122 loads in flight); the sums fit
// int32 (61 * 255^2 < 2^31), so they equal the int64 ones. Out of line: the
// unrolled body would otherwise count against the re-pick's register budget.
static __device__ __noinline__ void zncc_taps11(const uint8_t* __restrict__ L,
                                         const uint8_t* __restrict__ R, int W, int lu, int lv,
                                         int ru, int (&s)[5]) {
  int s_l = 0, s_r = 0, s_ll = 0, s_rr = 0, s_lr = 0;
#pragma unroll
  for (int dv = -5; dv <= 5; ++dv) {
    const uint8_t* lr = L + (long)(lv + dv) * W + lu;
    const uint8_t* rr = R + (long)(lv + dv) * W + ru;
#pragma unroll
    for (int du = -5 + ((dv + 5) & 1); du <= 5; du += 2) {
      const int a = __ldg(lr + du), b = __ldg(rr + du);
      s_l += a;
      s_r += b;
      s_ll += a * a;
      s_rr += b * b;
      s_lr += a * b;
    }
  }
  s[0] = s_l;
  s[1] = s_r;
  s[2] = s_ll;
  s[3] = s_rr;
  s[4] = s_lr;
}

__device__ __forceinline__ ExactScore zncc_exact(const uint8_t* __restrict__ L,
                                                 const uint8_t* __restrict__ R, int W, int lu,
                                                 int lv, int ru, int half,
                                                 bool wta_semantics) {
  int64_t n = 0, sl = 0, sr = 0, sll = 0, srr = 0, slr = 0;
  if (half == 5) {
    int s[5];
    zncc_taps11(L, R, W, lu, lv, ru, s);
    n = 61;
    sl = s[0];
    sr = s[1];
    sll = s[2];
    srr = s[3];
    slr = s[4];
  } else {
    for (int dv = -half; dv <= half; ++dv) {
      const uint8_t* lr = L + (long)(lv + dv) * W + lu;
      const uint8_t* rr = R + (long)(lv + dv) * W + ru;
      for (int du = -half + ((dv + half) & 1); du <= half; du += 2) {
        const int64_t a = __ldg(lr + du), b = __ldg(rr + du);
        n += 1;
        sl += a;
        sr += b;
        sll += a * a;
        srr += b * b;
        slr += a * b;
      }
    }
  }
  int64_t var_l = n * sll - sl * sl;
  int64_t var_r = n * srr - sr * sr;
  int64_t num;
  if (wta_semantics) {
    var_l = (int32_t)var_l;
    var_r = (int32_t)var_r;
    num = n * slr - (int64_t)(int32_t)sl * (int64_t)(int32_t)sr;
  } else {
    num = n * slr - sl * sr;
  }
  ExactScore r;
  r.defined = !(var_l == 0 || var_r == 0);
  r.score = r.defined ? __ddiv_rn((double)num, __dsqrt_rn((double)(var_l * var_r))) : 0.0;
  return r;
}

}  // namespace ssb
