// C++ drop-in for the reference's stereo entry points (include/stereoscan/),
// layered on the C-ABI (include/ss_stereo.h). Same declarations, same value
// types, same exception types and messages as
// /root/reference/proj/include/stereoscan/stereo/*.hpp; the per-frame work
// runs on the GPU. The scalar helpers zncc_chessboard / zncc_score /
// match_pixel (matcher.cpp:38-100) are per-pixel API utilities, not part of
// the frame path, and stay on the host with the reference's exact arithmetic.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>

#include "ss_stereo.h"
#include "stereoscan/features/features.hpp"
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

#ifndef SSB_USE_REFERENCE_GEOMETRY
// Compiled into the reference's build, geometry.cpp keeps these definitions
// (INTEGRATION.md): -DSSB_USE_REFERENCE_GEOMETRY drops ours.
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
#endif

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
                                 &np, nullptr));
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

// ---------------- feature front end (features.hpp) ----------------

#ifndef SSB_USE_REFERENCE_FEATURES
// -DSSB_USE_REFERENCE_FEATURES: the reference keeps its own features.cpp.
namespace stereoscan::features {

int Descriptor256::hamming(const Descriptor256& other) const {
  int d = 0;
  for (size_t k = 0; k < bits.size(); ++k) d += __builtin_popcountll(bits[k] ^ other.bits[k]);
  return d;
}

std::vector<Corner> detect_corners(const GrayImage& img, int max_count, int threshold) {
  const int cap = std::max(max_count, 0);
  std::vector<int32_t> u(std::max(cap, 1)), v(std::max(cap, 1)), s(std::max(cap, 1));
  int32_t n = 0;
  throw_on(ss_detect_corners(img.pixels.data(), img.width, img.height, max_count, threshold,
                             u.data(), v.data(), s.data(), &n));
  std::vector<Corner> out(n);
  for (int i = 0; i < n; ++i) out[i] = {u[i], v[i], s[i]};
  return out;
}

std::vector<Feature> describe(const GrayImage& img, const std::vector<Corner>& corners) {
  const int nc = static_cast<int>(corners.size());
  std::vector<int32_t> u(nc), v(nc), s(nc);
  for (int i = 0; i < nc; ++i) {
    u[i] = corners[i].u;
    v[i] = corners[i].v;
    s[i] = corners[i].score;
  }
  std::vector<double> pos(2 * std::max(nc, 1));
  std::vector<uint64_t> desc(4 * std::max(nc, 1));
  int32_t n = 0;
  throw_on(ss_describe(img.pixels.data(), img.width, img.height, u.data(), v.data(), s.data(),
                       nc, pos.data(), desc.data(), &n));
  std::vector<Feature> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].position = Vec2(pos[2 * i], pos[2 * i + 1]);
    for (int k = 0; k < 4; ++k) out[i].descriptor.bits[k] = desc[4 * i + k];
  }
  return out;
}

MatchSet match_features(const std::vector<Feature>& a, const std::vector<Feature>& b,
                        int max_hamming) {
  const int na = static_cast<int>(a.size()), nb = static_cast<int>(b.size());
  auto pack = [](const std::vector<Feature>& f, std::vector<double>& p,
                 std::vector<uint64_t>& d) {
    p.resize(2 * std::max<size_t>(f.size(), 1));
    d.resize(4 * std::max<size_t>(f.size(), 1));
    for (size_t i = 0; i < f.size(); ++i) {
      p[2 * i] = f[i].position.x();
      p[2 * i + 1] = f[i].position.y();
      for (int k = 0; k < 4; ++k) d[4 * i + k] = f[i].descriptor.bits[k];
    }
  };
  std::vector<double> pa, pb;
  std::vector<uint64_t> da, db;
  pack(a, pa, da);
  pack(b, pb, db);
  const int cap = std::max(std::min(na, nb), 1);
  std::vector<int32_t> ia(cap), ib(cap), hm(cap);
  std::vector<double> dp(2 * cap);
  int32_t n = 0;
  throw_on(ss_match_features(pa.data(), da.data(), na, pb.data(), db.data(), nb, max_hamming,
                             ia.data(), ib.data(), hm.data(), dp.data(), &n));
  MatchSet out(n);
  for (int i = 0; i < n; ++i) {
    out[i].index_a = ia[i];
    out[i].index_b = ib[i];
    out[i].hamming = hm[i];
    out[i].weight = 1.0;
    out[i].displacement = Vec2(dp[2 * i], dp[2 * i + 1]);
  }
  return out;
}

MatchSet histogram_vote(const MatchSet& matches, double bin_size) {
  if (!(bin_size > 0.0)) throw std::invalid_argument("histogram_vote: bin_size must be > 0");
  const size_t n = matches.size();
  // bin of each displacement (floor(x / bin)), counts per occupied bin
  std::vector<std::pair<int64_t, int64_t>> bin(n);
  std::map<std::pair<int64_t, int64_t>, int> count;
  for (size_t i = 0; i < n; ++i) {
    bin[i] = {static_cast<int64_t>(std::floor(matches[i].displacement.x() / bin_size)),
              static_cast<int64_t>(std::floor(matches[i].displacement.y() / bin_size))};
    ++count[bin[i]];
  }
  std::vector<int> prio(n, 0);
  for (size_t i = 0; i < n; ++i)
    for (int64_t dy = -1; dy <= 1; ++dy)
      for (int64_t dx = -1; dx <= 1; ++dx) {
        const auto it = count.find({bin[i].first + dx, bin[i].second + dy});
        if (it != count.end()) prio[i] += it->second;
      }
  std::vector<int> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&](int l, int r) {
    return prio[l] != prio[r] ? prio[l] > prio[r] : matches[l].hamming < matches[r].hamming;
  });
  MatchSet out;
  out.reserve(n);
  for (size_t r = 0; r < n; ++r) {
    out.push_back(matches[order[r]]);
    out.back().rank = static_cast<int>(r);
  }
  return out;
}

std::vector<std::pair<Vec2, Vec2>> read_match_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error("cannot open match file: " + path);
  std::vector<std::pair<Vec2, Vec2>> out;
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream fields(line);
    double a, b, c, d;
    if (!(fields >> a >> b >> c >> d))
      throw Error(path + ":" + std::to_string(no) + ": expected 'u1 v1 u2 v2'");
    out.push_back({Vec2(a, b), Vec2(c, d)});
  }
  return out;
}

}  // namespace stereoscan::features
#endif
