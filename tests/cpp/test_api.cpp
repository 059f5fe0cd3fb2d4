// C++ drop-in test: the reference's own entry points (include/stereoscan/),
// called exactly as reference code calls them, running on the B200.
// Mirrors the SPEC.md examples for the stereo module.
// Built by paper_2007_12623_b200/build.py, run by tests/test_cpp_api.py (gpu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>

#include "stereoscan/features/features.hpp"
#include "stereoscan/stereo/cleanup.hpp"
#include "stereoscan/stereo/cloud.hpp"
#include "stereoscan/stereo/matcher.hpp"
#include "stereoscan/stereo/smoothing.hpp"

using namespace stereoscan;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                    \
    }                                                                \
  } while (0)

int main() {
  std::mt19937 rng(7);
  // shift-by-7 texture -> disparity 7 at every interior pixel
  GrayImage tex(170, 64);
  for (auto& p : tex.pixels) p = static_cast<uint8_t>(rng() & 0xFF);
  GrayImage left(160, 64), right(160, 64);
  for (int v = 0; v < 64; ++v)
    for (int u = 0; u < 160; ++u) {
      left.at(u, v) = tex.at(u, v);
      right.at(u, v) = tex.at(u + 7, v);
    }
  StereoParams p;
  p.d_min = 0;
  p.d_max = 15;
  const DisparityMap m = compute_disparity(left, right, p);
  CHECK(m.valid_count() > 0);
  for (size_t i = 0; i < m.valid.size(); ++i)
    if (m.valid[i]) CHECK(m.disparity[i] == 7.0f);
  // match_pixel agrees with the dense search
  const auto mp = match_pixel(left, right, 80, 30, p);
  CHECK(mp.has_value() && *mp == 7);
  // LR-consistency extension: a pure shift is consistent wherever the right
  // view sees the same match; the right view holds 7 too.
  DisparityMap rm;
  const DisparityMap lr = compute_disparity_lr(left, right, p, 1, &rm);
  CHECK(lr.valid_count() > 0 && lr.valid_count() <= m.valid_count());
  for (size_t i = 0; i < lr.valid.size(); ++i)
    if (lr.valid[i]) CHECK(m.valid[i] && lr.disparity[i] == 7.0f);
  for (size_t i = 0; i < rm.valid.size(); ++i)
    if (rm.valid[i]) CHECK(rm.disparity[i] == 7.0f);
  try {
    compute_disparity_lr(left, right, p, -1);
    CHECK(false);
  } catch (const std::invalid_argument&) {
  }

  // uniform pair -> all invalid
  GrayImage flat(64, 48, 77);
  CHECK(compute_disparity(flat, flat, p).valid_count() == 0);

  // zncc_score KATs
  GrayImage a(11, 11), b(11, 11), c(11, 11);
  for (int i = 0; i < 121; ++i) {
    a.pixels[i] = static_cast<uint8_t>(20 + (rng() % 100));
    b.pixels[i] = static_cast<uint8_t>(2 * a.pixels[i] + 12);
    c.pixels[i] = static_cast<uint8_t>(255 - a.pixels[i]);
  }
  CHECK(std::fabs(*zncc_score(a, a) - 1.0) < 1e-9);
  CHECK(std::fabs(*zncc_score(a, b) - 1.0) < 1e-9);
  CHECK(std::fabs(*zncc_score(a, c) + 1.0) < 1e-9);

  // errors: same types and messages as the reference (matcher.cpp:10,169)
  try {
    compute_disparity(left, GrayImage(10, 10), p);
    CHECK(false);
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "compute_disparity: image sizes differ");
  }
  try {
    StereoParams bad = p;
    bad.window = 8;
    compute_disparity(left, right, bad);
    CHECK(false);
  } catch (const Error& e) {
    CHECK(std::string(e.what()) == "stereo: window must be odd and >= 3");
  }

  // cleanup: constant field is a fixed point; fully invalid stays invalid
  DisparityMap cst(40, 40);
  for (size_t i = 0; i < cst.valid.size(); ++i) {
    cst.valid[i] = 1;
    cst.disparity[i] = 12.0f;
  }
  const DisparityMap cc = cleanup_pass(cst, p);
  CHECK(cc.valid_count() == cst.valid.size() && cc.disparity == cst.disparity);
  CHECK(cleanup_pass(DisparityMap(40, 40), p).valid_count() == 0);
  CHECK(disc_neighbor_count(20) == 1256 && disc_fill_min_support(20) == 314);
  // spike removed then refilled
  DisparityMap spike = cst;
  spike.disparity[spike.idx(20, 20)] = 22.0f;
  CHECK(!remove_outliers(spike, 10, 2.5).is_valid(20, 20));
  const DisparityMap sc = cleanup_pass(spike, p);
  CHECK(sc.is_valid(20, 20) && std::fabs(sc.at(20, 20) - 12.0f) < 1e-5f);

  // refine: constant field with consistent images is a fixed point
  GrayImage L2(40, 40), R2(40, 40);
  GrayImage t2(60, 40);
  for (auto& q : t2.pixels) q = static_cast<uint8_t>(rng() & 0xFF);
  for (int v = 0; v < 40; ++v)
    for (int u = 0; u < 40; ++u) {
      L2.at(u, v) = t2.at(u, v);
      R2.at(u, v) = t2.at(u + 12, v);
    }
  DisparityMap m2(40, 40);
  for (int v = 5; v < 35; ++v)
    for (int u = 22; u < 35; ++u) {
      m2.valid[m2.idx(u, v)] = 1;
      m2.disparity[m2.idx(u, v)] = 12.0f;
    }
  RefineTrace tr;
  const DisparityMap r2 = refine_disparities(m2, L2, R2, p, &tr);
  CHECK(tr.discrete.size() == static_cast<size_t>(p.refine_iterations));
  for (size_t i = 0; i < r2.valid.size(); ++i)
    if (r2.valid[i]) CHECK(std::fabs(r2.disparity[i] - 12.0f) < 1e-6f);

  // cloud: on-axis point and fronto-parallel normals
  StereoRig rig;
  rig.intrinsics.fx = rig.intrinsics.fy = 1000.0;
  rig.intrinsics.cx = 10.0;
  rig.intrinsics.cy = 8.0;
  rig.intrinsics.width = 21;
  rig.intrinsics.height = 17;
  rig.baseline_mm = 5.0;
  DisparityMap fp(21, 17);
  for (size_t i = 0; i < fp.valid.size(); ++i) {
    fp.valid[i] = 1;
    fp.disparity[i] = 50.0f;
  }
  const StereoCloud cl = disparity_to_cloud(fp, ColorImage(21, 17), rig);
  const Vec3& q = cl.points[cl.point_at(10, 8)];
  CHECK(q.x() == 0.0 && q.y() == 0.0 && q.z() == 100.0);
  for (const Vec3& n : cl.normals) CHECK(std::fabs(n.z() + 1.0) < 1e-3);
  try {
    StereoRig r0 = rig;
    r0.baseline_mm = 0.0;
    disparity_to_cloud(fp, ColorImage(21, 17), r0);
    CHECK(false);
  } catch (const Error& e) {
    CHECK(std::string(e.what()) == "rig: baseline_mm must be > 0");
  }

  // ---- feature front end (features.hpp) ----
  {
    namespace fe = stereoscan::features;
    GrayImage sq(64, 64, 0);
    for (int v = 20; v < 44; ++v)
      for (int u = 20; u < 44; ++u) sq.at(u, v) = 255;
    const auto cs = fe::detect_corners(sq, 100, 30);
    CHECK(cs.size() == 4 && cs[0].score == 255 && cs[0].u == 20 && cs[0].v == 20);
    try {
      fe::detect_corners(sq, 10, 0);
      CHECK(false);
    } catch (const std::invalid_argument& e) {
      CHECK(std::string(e.what()) == "detect_corners: threshold must be >= 1");
    }
    // self-matching a textured frame: every feature matches itself at distance 0
    const auto corners = fe::detect_corners(left, 200, 10);
    const auto feats = fe::describe(left, corners);
    CHECK(!feats.empty() && feats.size() <= corners.size());
    const auto ms = fe::match_features(feats, feats, 0);
    CHECK(ms.size() >= feats.size() / 2);
    for (const auto& m : ms) CHECK(m.hamming == 0 && m.displacement.x() == 0.0);
    const auto ranked = fe::histogram_vote(ms, 4.0);
    CHECK(ranked.size() == ms.size());
    for (size_t r = 0; r < ranked.size(); ++r) CHECK(ranked[r].rank == static_cast<int>(r));
    try {
      fe::read_match_file("/nonexistent/matches.txt");
      CHECK(false);
    } catch (const stereoscan::Error&) {
    }
  }

  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("test_api OK\n");
  return 0;
}
