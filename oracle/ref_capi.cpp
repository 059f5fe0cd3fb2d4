// ORACLE — test infrastructure only.
//
// extern "C" wrapper that lets the tests call the UNMODIFIED reference
// implementation of the hot path. This file contains no algorithm; every
// function copies the caller's buffers into the reference's value types,
// calls the reference entry point and copies the result back.
//
//   compute_disparity   matcher.cpp:166-211
//   reference::*        reference.cpp:7-85
//   remove_outliers     cleanup.cpp:12-42
//   fill_holes          cleanup.cpp:44-92
//   cleanup_pass        cleanup.cpp:111-123
//   refine_disparities  smoothing.cpp:68-159
//   to_gray             matcher.cpp:21-30
//   zncc_chessboard     matcher.cpp:38-64
//   features::*         features.cpp:86-258 (detect_corners, describe,
//                       match_features, histogram_vote)
//
// Built by oracle/Makefile against /root/reference/proj/src (never copied).

#include <cstring>
#include <stdexcept>
#include <string>

#include "stereoscan/features/features.hpp"
#include "stereoscan/stereo/cleanup.hpp"
#include "stereoscan/stereo/matcher.hpp"
#include "stereoscan/stereo/reference.hpp"
#include "stereoscan/stereo/smoothing.hpp"
#include "ss_oracle.h"

namespace ss = stereoscan;

namespace {

thread_local std::string g_err;

ss::StereoParams to_params(const orc_params* p) {
  ss::StereoParams s;
  s.window = p->window;
  s.d_min = p->d_min;
  s.d_max = p->d_max;
  s.neighbor_jump_threshold = p->neighbor_jump_threshold;
  s.outlier_radius_start = p->outlier_radius_start;
  s.outlier_radius_step = p->outlier_radius_step;
  s.cleanup_iterations = p->cleanup_iterations;
  s.fill_radius_radial = p->fill_radius_radial;
  s.fill_radius_disc = p->fill_radius_disc;
  s.smoothing_radius = p->smoothing_radius;
  s.alpha = p->alpha;
  s.eta_smooth = p->eta_smooth;
  s.refine_iterations = p->refine_iterations;
  s.min_zncc = p->min_zncc;
  return s;
}

ss::GrayImage gray_of(const uint8_t* px, int w, int h) {
  ss::GrayImage g(w, h);
  if (w > 0 && h > 0) std::memcpy(g.pixels.data(), px, static_cast<size_t>(w) * h);
  return g;
}

ss::DisparityMap map_of(const float* d, const uint8_t* v, int w, int h) {
  ss::DisparityMap m(w, h);
  const size_t n = static_cast<size_t>(w) * h;
  if (n) {
    std::memcpy(m.disparity.data(), d, n * sizeof(float));
    std::memcpy(m.valid.data(), v, n);
  }
  return m;
}

void emit(const ss::DisparityMap& m, float* d, uint8_t* v) {
  const size_t n = m.disparity.size();
  if (n) {
    std::memcpy(d, m.disparity.data(), n * sizeof(float));
    std::memcpy(v, m.valid.data(), n);
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const ss::Error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_params_validate(const orc_params* p) {
  return guarded([&] { to_params(p).validate(); });
}

int ref_to_gray(const uint8_t* rgb, int32_t w, int32_t h, uint8_t* gray) {
  return guarded([&] {
    ss::ColorImage c(w, h);
    if (w > 0 && h > 0) std::memcpy(c.pixels.data(), rgb, static_cast<size_t>(w) * h * 3);
    const ss::GrayImage g = ss::to_gray(c);
    if (w > 0 && h > 0) std::memcpy(gray, g.pixels.data(), static_cast<size_t>(w) * h);
  });
}

double ref_zncc_chessboard(const uint8_t* left, const uint8_t* right, int32_t w,
                           int32_t h, int32_t lu, int32_t lv, int32_t ru, int32_t rv,
                           int32_t window, int32_t* defined) {
  const ss::GrayImage l = gray_of(left, w, h), r = gray_of(right, w, h);
  const auto s = ss::zncc_chessboard(l, lu, lv, r, ru, rv, window);
  *defined = s.has_value() ? 1 : 0;
  return s.value_or(0.0);
}

int ref_compute_disparity(const orc_params* p, const uint8_t* left, const uint8_t* right,
                          int32_t w, int32_t h, float* disp, uint8_t* valid) {
  return guarded([&] {
    emit(ss::compute_disparity(gray_of(left, w, h), gray_of(right, w, h), to_params(p)),
         disp, valid);
  });
}

int ref_naive_compute_disparity(const orc_params* p, const uint8_t* left,
                                const uint8_t* right, int32_t w, int32_t h, float* disp,
                                uint8_t* valid) {
  return guarded([&] {
    emit(ss::reference::compute_disparity(gray_of(left, w, h), gray_of(right, w, h),
                                          to_params(p)),
         disp, valid);
  });
}

int ref_remove_outliers(const float* disp, const uint8_t* valid, int32_t w, int32_t h,
                        int32_t radius, double threshold, float* out_disp,
                        uint8_t* out_valid) {
  return guarded([&] {
    emit(ss::remove_outliers(map_of(disp, valid, w, h), radius, threshold), out_disp,
         out_valid);
  });
}

int ref_naive_remove_outliers(const float* disp, const uint8_t* valid, int32_t w,
                              int32_t h, int32_t radius, double threshold,
                              float* out_disp, uint8_t* out_valid) {
  return guarded([&] {
    emit(ss::reference::remove_outliers(map_of(disp, valid, w, h), radius, threshold),
         out_disp, out_valid);
  });
}

int ref_fill_holes(const float* disp, const uint8_t* valid, int32_t w, int32_t h,
                   int32_t mode, int32_t radius, int32_t min_support, float* out_disp,
                   uint8_t* out_valid) {
  return guarded([&] {
    const ss::FillMode m = mode == 0 ? ss::FillMode::Radial : ss::FillMode::Disc;
    emit(ss::fill_holes(map_of(disp, valid, w, h), m, radius, min_support), out_disp,
         out_valid);
  });
}

int32_t ref_disc_neighbor_count(int32_t radius) { return ss::disc_neighbor_count(radius); }
int32_t ref_disc_fill_min_support(int32_t radius) {
  return ss::disc_fill_min_support(radius);
}

int ref_cleanup_pass(const orc_params* p, const float* disp, const uint8_t* valid,
                     int32_t w, int32_t h, float* out_disp, uint8_t* out_valid) {
  return guarded([&] {
    emit(ss::cleanup_pass(map_of(disp, valid, w, h), to_params(p)), out_disp, out_valid);
  });
}

int ref_refine_disparities(const orc_params* p, const float* disp, const uint8_t* valid,
                           const uint8_t* left, const uint8_t* right, int32_t w,
                           int32_t h, float* out_disp, uint8_t* out_valid,
                           double* trace_discrete, double* trace_smooth) {
  return guarded([&] {
    ss::RefineTrace trace;
    const bool want = trace_discrete != nullptr || trace_smooth != nullptr;
    const ss::DisparityMap out =
        ss::refine_disparities(map_of(disp, valid, w, h), gray_of(left, w, h),
                               gray_of(right, w, h), to_params(p), want ? &trace : nullptr);
    emit(out, out_disp, out_valid);
    const size_t n = static_cast<size_t>(w) * h;
    for (size_t it = 0; want && it < trace.discrete.size(); ++it) {
      if (trace_discrete) std::memcpy(trace_discrete + it * n, trace.discrete[it].data(), n * 8);
      if (trace_smooth) std::memcpy(trace_smooth + it * n, trace.smooth[it].data(), n * 8);
    }
  });
}

// ---- features (features.cpp) ----
// Corners: u/v/score arrays of capacity max_count; *n receives the count.
int ref_detect_corners(const uint8_t* gray, int32_t w, int32_t h, int32_t max_count,
                       int32_t threshold, int32_t* us, int32_t* vs, int32_t* scores,
                       int32_t* n) {
  return guarded([&] {
    const auto cs = ss::features::detect_corners(gray_of(gray, w, h), max_count, threshold);
    for (size_t i = 0; i < cs.size(); ++i) {
      us[i] = cs[i].u;
      vs[i] = cs[i].v;
      scores[i] = cs[i].score;
    }
    *n = static_cast<int32_t>(cs.size());
  });
}

// Features of the given corners: pos (u, v) doubles and 4 x u64 descriptor
// words per feature, capacity nc; *n receives the count.
int ref_describe(const uint8_t* gray, int32_t w, int32_t h, const int32_t* us,
                 const int32_t* vs, const int32_t* scores, int32_t nc, double* pos,
                 uint64_t* desc, int32_t* n) {
  return guarded([&] {
    std::vector<ss::features::Corner> cs(nc);
    for (int i = 0; i < nc; ++i) cs[i] = {us[i], vs[i], scores[i]};
    const auto fs = ss::features::describe(gray_of(gray, w, h), cs);
    for (size_t i = 0; i < fs.size(); ++i) {
      pos[2 * i] = fs[i].position.x();
      pos[2 * i + 1] = fs[i].position.y();
      for (int k = 0; k < 4; ++k) desc[4 * i + k] = fs[i].descriptor.bits[k];
    }
    *n = static_cast<int32_t>(fs.size());
  });
}

static std::vector<ss::features::Feature> feats_of(const double* pos, const uint64_t* desc,
                                                   int32_t n) {
  std::vector<ss::features::Feature> fs(n);
  for (int i = 0; i < n; ++i) {
    fs[i].position = ss::Vec2(pos[2 * i], pos[2 * i + 1]);
    for (int k = 0; k < 4; ++k) fs[i].descriptor.bits[k] = desc[4 * i + k];
  }
  return fs;
}

// Matches: index_a, index_b, hamming per match (capacity min(na, nb)),
// displacement (du, dv) doubles; *n receives the count.
int ref_match_features(const double* pos_a, const uint64_t* desc_a, int32_t na,
                       const double* pos_b, const uint64_t* desc_b, int32_t nb,
                       int32_t max_hamming, int32_t* ia, int32_t* ib, int32_t* ham,
                       double* disp, int32_t* n) {
  return guarded([&] {
    const auto ms = ss::features::match_features(feats_of(pos_a, desc_a, na),
                                                 feats_of(pos_b, desc_b, nb), max_hamming);
    for (size_t i = 0; i < ms.size(); ++i) {
      ia[i] = ms[i].index_a;
      ib[i] = ms[i].index_b;
      ham[i] = ms[i].hamming;
      disp[2 * i] = ms[i].displacement.x();
      disp[2 * i + 1] = ms[i].displacement.y();
    }
    *n = static_cast<int32_t>(ms.size());
  });
}

// histogram_vote over n matches (index_a, index_b, hamming, displacement);
// writes the permutation `order` (input index at each rank).
int ref_histogram_vote(const int32_t* ia, const int32_t* ib, const int32_t* ham,
                       const double* disp, int32_t n, double bin_size, int32_t* order) {
  return guarded([&] {
    ss::features::MatchSet ms(n);
    for (int i = 0; i < n; ++i) {
      ms[i].index_a = ia[i];
      ms[i].index_b = ib[i];
      ms[i].hamming = ham[i];
      ms[i].displacement = ss::Vec2(disp[2 * i], disp[2 * i + 1]);
    }
    const auto out = ss::features::histogram_vote(ms, bin_size);
    for (size_t r = 0; r < out.size(); ++r) {
      int k = 0;  // recover the input index (index_a is unique per input match)
      while (k < n && !(ms[k].index_a == out[r].index_a && ms[k].index_b == out[r].index_b)) ++k;
      order[r] = k;
    }
  });
}

}  // extern "C"
