// C++ drop-in for the reference's stereo entry points (include/stereoscan/),
// layered on the C-ABI (include/ss_stereo.h). Same declarations, same value
// types, same exception types and messages as
// /root/reference/proj/include/stereoscan/stereo/*.hpp; the per-frame work
// runs on the GPU. The scalar helpers zncc_chessboard / zncc_score /
// match_pixel (matcher.cpp:38-100) are per-pixel API utilities, not part of
// the frame path, and stay on the host with the reference's exact arithmetic.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "ss_stereo.h"
#include "stereoscan/stereo/cleanup.hpp"
#include "stereoscan/stereo/cloud.hpp"
#include "stereoscan/stereo/matcher.hpp"
#include "stereoscan/stereo/smoothing.hpp"

namespace stereoscan {

static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");

namespace {

void throw_on(ss_status st) {
  if (st == SS_OK) return;
  const std::string msg = ss_last_error();
  if (st == SS_EINVAL) throw std::invalid_argument(msg);
  throw Error(msg);
}

ss_stereo_params to_c(const StereoParams& p) {
  ss_stereo_params c;
  c.window = p.window;
  c.d_min = p.d_min;
  c.d_max = p.d_max;
  c.neighbor_jump_threshold = p.neighbor_jump_threshold;
  c.outlier_radius_start = p.outlier_radius_start;
  c.outlier_radius_step = p.outlier_radius_step;
  c.cleanup_iterations = p.cleanup_iterations;
  c.fill_radius_radial = p.fill_radius_radial;
  c.fill_radius_disc = p.fill_radius_disc;
  c.smoothing_radius = p.smoothing_radius;
  c.alpha = p.alpha;
  c.eta_smooth = p.eta_smooth;
  c.refine_iterations = p.refine_iterations;
  c.min_zncc = p.min_zncc;
  return c;
}

ss_stereo_rig to_c(const StereoRig& r) {
  ss_stereo_rig c;
  c.fx = r.intrinsics.fx;
  c.fy = r.intrinsics.fy;
  c.cx = r.intrinsics.cx;
  c.cy = r.intrinsics.cy;
  c.width = r.intrinsics.width;
  c.height = r.intrinsics.height;
  c.baseline_mm = r.baseline_mm;
  return c;
}

}  // namespace

void StereoParams::validate() const {
  const ss_stereo_params c = to_c(*this);
  throw_on(ss_params_validate(&c));
}

void CameraIntrinsics::validate() const {
  StereoRig r;
  r.intrinsics = *this;
  r.baseline_mm = 1.0;
  const ss_stereo_rig c = to_c(r);
  throw_on(ss_rig_validate(&c));
}

void StereoRig::validate() const {
  const ss_stereo_rig c = to_c(*this);
  throw_on(ss_rig_validate(&c));
}

size_t DisparityMap::valid_count() const {
  size_t n = 0;
  for (uint8_t v : valid) n += v;
  return n;
}

GrayImage to_gray(const ColorImage& color) {
  GrayImage gray(color.width, color.height);
  throw_on(ss_to_gray(color.pixels.data(), color.width, color.height, gray.pixels.data()));
  return gray;
}

std::optional<double> zncc_chessboard(const GrayImage& left, int lu, int lv,
                                      const GrayImage& right, int ru, int rv, int window) {
  const int h = window / 2;
  int64_t n = 0, sl = 0, sr = 0, sll = 0, srr = 0, slr = 0;
  for (int dv = -h; dv <= h; ++dv) {
    for (int du = -h + ((dv + h) & 1); du <= h; du += 2) {
      const int64_t a = left.at(lu + du, lv + dv);
      const int64_t b = right.at(ru + du, rv + dv);
      n += 1;
      sl += a;
      sr += b;
      sll += a * a;
      srr += b * b;
      slr += a * b;
    }
  }
  const int64_t var_l = n * sll - sl * sl;
  const int64_t var_r = n * srr - sr * sr;
  if (var_l == 0 || var_r == 0) return std::nullopt;
  const int64_t num = n * slr - sl * sr;
  return static_cast<double>(num) / std::sqrt(static_cast<double>(var_l * var_r));
}

std::optional<double> zncc_score(const GrayImage& left_patch, const GrayImage& right_patch) {
  if (left_patch.width != left_patch.height || left_patch.width != right_patch.width ||
      left_patch.height != right_patch.height) {
    throw std::invalid_argument("zncc_score: patches must be square and equal-sized");
  }
  const int w = left_patch.width;
  return zncc_chessboard(left_patch, w / 2, w / 2, right_patch, w / 2, w / 2, w);
}

std::optional<int> match_pixel(const GrayImage& left, const GrayImage& right, int u, int v,
                               const StereoParams& params) {
  const int h = params.window / 2;
  if (u < h || u >= left.width - h || v < h || v >= left.height - h) return std::nullopt;
  bool found = false;
  double best = 0.0;
  int best_d = 0;
  for (int d = params.d_min; d <= params.d_max; ++d) {
    const int ru = u - d;
    if (ru < h || ru >= right.width - h) continue;
    const auto s = zncc_chessboard(left, u, v, right, ru, v, params.window);
    if (!s) continue;
    if (!found || *s > best) {
      found = true;
      best = *s;
      best_d = d;
    }
  }
  if (!found || best < params.min_zncc) return std::nullopt;
  return best_d;
}

DisparityMap compute_disparity(const GrayImage& left, const GrayImage& right,
                               const StereoParams& params) {
  if (left.width != right.width || left.height != right.height) {
    throw std::invalid_argument("compute_disparity: image sizes differ");
  }
  const ss_stereo_params c = to_c(params);
  throw_on(ss_params_validate(&c));
  DisparityMap map(left.width, left.height);
  throw_on(ss_compute_disparity(&c, left.pixels.data(), left.width, left.height,
                                right.pixels.data(), right.width, right.height,
                                map.disparity.data(), map.valid.data()));
  return map;
}

DisparityMap compute_disparity_lr(const GrayImage& left, const GrayImage& right,
                                  const StereoParams& params, int max_diff,
                                  DisparityMap* right_map) {
  if (left.width != right.width || left.height != right.height) {
    throw std::invalid_argument("compute_disparity: image sizes differ");
  }
  const ss_stereo_params c = to_c(params);
  throw_on(ss_params_validate(&c));
  DisparityMap map(left.width, left.height);
  DisparityMap rmap(left.width, left.height);
  throw_on(ss_compute_disparity_lr(&c, left.pixels.data(), left.width, left.height,
                                   right.pixels.data(), right.width, right.height, max_diff,
                                   map.disparity.data(), map.valid.data(),
                                   rmap.disparity.data(), rmap.valid.data()));
  if (right_map) *right_map = std::move(rmap);
  return map;
}

DisparityMap remove_outliers(const DisparityMap& map, int radius, double threshold) {
  DisparityMap out(map.width, map.height);
  throw_on(ss_remove_outliers(map.disparity.data(), map.valid.data(), map.width, map.height,
                              radius, threshold, out.disparity.data(), out.valid.data()));
  return out;
}

DisparityMap fill_holes(const DisparityMap& map, FillMode mode, int radius, int min_support) {
  DisparityMap out(map.width, map.height);
  throw_on(ss_fill_holes(map.disparity.data(), map.valid.data(), map.width, map.height,
                         mode == FillMode::Radial ? SS_FILL_RADIAL : SS_FILL_DISC, radius,
                         min_support, out.disparity.data(), out.valid.data()));
  return out;
}

int disc_neighbor_count(int radius) { return ss_disc_neighbor_count(radius); }
int disc_fill_min_support(int radius) { return ss_disc_fill_min_support(radius); }

DisparityMap cleanup_pass(const DisparityMap& map, const StereoParams& params) {
  const ss_stereo_params c = to_c(params);
  DisparityMap out(map.width, map.height);
  throw_on(ss_cleanup_pass(&c, map.disparity.data(), map.valid.data(), map.width, map.height,
                           out.disparity.data(), out.valid.data()));
  return out;
}

DisparityMap refine_disparities(const DisparityMap& map, const GrayImage& left,
                                const GrayImage& right, const StereoParams& params,
                                RefineTrace* trace) {
  const ss_stereo_params c = to_c(params);
  DisparityMap out(map.width, map.height);
  const size_t n = static_cast<size_t>(map.width) * map.height;
  const int iters = params.refine_iterations > 0 ? params.refine_iterations : 0;
  std::vector<double> td, ts;
  if (trace) {
    td.resize(n * iters);
    ts.resize(n * iters);
  }
  throw_on(ss_refine_disparities(&c, map.disparity.data(), map.valid.data(), map.width,
                                 map.height, left.pixels.data(), left.width, left.height,
                                 right.pixels.data(), right.width, right.height,
                                 out.disparity.data(), out.valid.data(),
                                 trace ? td.data() : nullptr, trace ? ts.data() : nullptr));
  if (trace) {
    for (int it = 0; it < iters; ++it) {
      trace->discrete.emplace_back(td.begin() + it * n, td.begin() + (it + 1) * n);
      trace->smooth.emplace_back(ts.begin() + it * n, ts.begin() + (it + 1) * n);
    }
  }
  return out;
}

StereoCloud disparity_to_cloud(const DisparityMap& map, const ColorImage& color,
                               const StereoRig& rig) {
  const ss_stereo_rig c = to_c(rig);
  StereoCloud cloud;
  cloud.width = map.width;
  cloud.height = map.height;
  const size_t n = static_cast<size_t>(map.width) * map.height;
  cloud.index.assign(n, -1);
  std::vector<Vec3> pts(n), nrm(n);
  std::vector<uint8_t> col(3 * n);
  std::vector<int32_t> pix(2 * n);
  int32_t np = 0;
  throw_on(ss_disparity_to_cloud(map.disparity.data(), map.valid.data(), map.width, map.height,
                                 color.pixels.empty() ? nullptr : color.pixels.data(),
                                 color.width, color.height, &c, cloud.index.data(),
                                 reinterpret_cast<double*>(pts.data()),
                                 reinterpret_cast<double*>(nrm.data()), col.data(), pix.data(),
                                 &np));
  cloud.points.assign(pts.begin(), pts.begin() + np);
  cloud.normals.assign(nrm.begin(), nrm.begin() + np);
  cloud.colors.resize(np);
  cloud.pixels.resize(np);
  for (int i = 0; i < np; ++i) {
    cloud.colors[i] = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
    cloud.pixels[i] = {pix[2 * i], pix[2 * i + 1]};
  }
  return cloud;
}

}  // namespace stereoscan
