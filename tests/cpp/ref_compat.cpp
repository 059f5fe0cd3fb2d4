// Source-compatibility check of the drop-in headers: the reference's own,
// UNMODIFIED proj/src/stereo/reference.cpp (naive exhaustive matcher and
// 8-ray outlier test) is compiled against include/stereoscan/stereo/*.hpp
// of this repository (only reference.hpp comes from /root/reference) and
// linked with libstereoscan_b200(_cxx).so. The program then holds the GPU
// drop-ins to the reference's naive code on seeded inputs.
#include <cstdint>
#include <cstdio>
#include <random>

#include "stereoscan/stereo/cleanup.hpp"
#include "stereoscan/stereo/matcher.hpp"
#include "stereoscan/stereo/reference.hpp"

using namespace stereoscan;

static bool same(const DisparityMap& a, const DisparityMap& b) {
  if (a.width != b.width || a.height != b.height) return false;
  for (size_t i = 0; i < a.valid.size(); ++i)
    if (a.valid[i] != b.valid[i] || (a.valid[i] && a.disparity[i] != b.disparity[i])) return false;
  return true;
}

int main() {
  std::mt19937 rng(2024);
  StereoParams p;
  p.d_min = 0;
  p.d_max = 15;
  int bad = 0;
  for (int t = 0; t < 20; ++t) {
    GrayImage L(64, 48), R(64, 48);
    const int shift = (int)(rng() % 12);
    for (int v = 0; v < 48; ++v)
      for (int u = 0; u < 64; ++u) L.at(u, v) = (uint8_t)(rng() & 255);
    for (int v = 0; v < 48; ++v)
      for (int u = 0; u < 64; ++u) {
        const int su = u + shift < 64 ? u + shift : 63;
        const int n = (int)(rng() % 5) - 2;
        const int x = L.at(su, v) + n;
        R.at(u, v) = (uint8_t)(x < 0 ? 0 : x > 255 ? 255 : x);
      }
    if (!same(compute_disparity(L, R, p), reference::compute_disparity(L, R, p))) ++bad;
    DisparityMap f(48, 48);
    for (size_t i = 0; i < f.disparity.size(); ++i) {
      f.disparity[i] = 10.0f + (float)(rng() % 100) * 0.03f + ((rng() % 5) == 0 ? 8.0f : 0.0f);
      f.valid[i] = (rng() % 10) != 0;
    }
    const int r = 1 + (int)(rng() % 12);
    if (!same(remove_outliers(f, r, 2.5), reference::remove_outliers(f, r, 2.5))) ++bad;
  }
  if (bad) {
    std::printf("ref_compat FAILED: %d mismatching cases\n", bad);
    return 1;
  }
  std::printf("ref_compat OK\n");
  return 0;
}
