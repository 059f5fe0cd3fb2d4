/*
 * ORACLE — CPU restatement of the reference's per-frame stereo hot path.
 * TEST INFRASTRUCTURE ONLY: called by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs as the checker. The product
 * (paper_2007_12623_b200) never links or calls this file.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * compiled reference (oracle/_ref, when /root/reference is present) and against
 * the committed golden vectors in tests/golden/ (generated from oracle/_ref by
 * tests/golden/make_golden.py). disparity_to_cloud cannot be pinned that way:
 * the reference needs Eigen, which is absent. Its points follow
 * cloud.cpp:23-39 operation for operation; its normals restate, operation for
 * operation, the eigensolver the reference calls (cloud.cpp:78:
 * Eigen::SelfAdjointEigenSolver<Matrix3d>, Eigen 3.4.0 — the version is not
 * pinned by the reference, whose vendored Eigen is git-ignored): see
 * eigen3_sym below. Pinned to the SPEC examples and, as an
 * eigensolver, to LAPACK (numpy.linalg.eigh) in tests/test_oracle.py.
 *
 * Floating point: build with -ffp-contract=off and no -ffast-math/-march
 * (SURVEY.md fact 7). Every double expression below keeps the reference's
 * association order; the comments cite the line it restates.
 */
#include "ss_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_SQRT2
#define M_SQRT2 1.41421356237309504880
#endif

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* StereoParams::validate, matcher.cpp:9-19 (same messages, same order). */
int orc_params_validate(const orc_params* p) {
  if (p->window < 3 || p->window % 2 == 0) return fail(2, "stereo: window must be odd and >= 3");
  if (p->d_min >= p->d_max) return fail(2, "stereo: d_min must be < d_max");
  if (p->outlier_radius_start <= 0 || p->outlier_radius_step <= 0 ||
      p->fill_radius_radial <= 0 || p->fill_radius_disc <= 0 || p->smoothing_radius <= 0)
    return fail(2, "stereo: radii must be > 0");
  if (!(p->alpha >= 0.0 && p->alpha <= 1.0)) return fail(2, "stereo: alpha must be in [0,1]");
  if (p->cleanup_iterations < 0) return fail(2, "stereo: cleanup_iterations must be >= 0");
  if (p->refine_iterations < 0) return fail(2, "stereo: refine_iterations must be >= 0");
  return 0;
}

/* CameraIntrinsics/StereoRig::validate, geometry.cpp:7-19. */
int orc_rig_validate(const orc_rig* r) {
  if (!(r->fx > 0.0)) return fail(2, "intrinsics: fx must be > 0");
  if (!(r->fy > 0.0)) return fail(2, "intrinsics: fy must be > 0");
  if (r->width <= 0) return fail(2, "intrinsics: width must be > 0");
  if (r->height <= 0) return fail(2, "intrinsics: height must be > 0");
  if (!(r->cx >= 0.0 && r->cx < r->width)) return fail(2, "intrinsics: cx out of image bounds");
  if (!(r->cy >= 0.0 && r->cy < r->height)) return fail(2, "intrinsics: cy out of image bounds");
  if (!(r->baseline_mm > 0.0)) return fail(2, "rig: baseline_mm must be > 0");
  return 0;
}

/* to_gray, matcher.cpp:21-30: luma = (0.299 R + 0.587 G) + 0.114 B in double,
 * lround (half away from zero). */
int orc_to_gray(const uint8_t* rgb, int32_t w, int32_t h, uint8_t* gray) {
  const long n = (long)w * h;
  for (long i = 0; i < n; ++i) {
    const double r = 0.299 * rgb[3 * i + 0];
    const double g = 0.587 * rgb[3 * i + 1];
    const double b = 0.114 * rgb[3 * i + 2];
    gray[i] = (uint8_t)lround(r + g + b);
  }
  return 0;
}

/* Chessboard window statistics, matcher.cpp:38-64: taps with (du+dv) even. */
typedef struct {
  int64_t n, sl, sr, sll, srr, slr;
} orc_stats;

static orc_stats chess_stats(const uint8_t* L, const uint8_t* R, int32_t w, int32_t lu,
                             int32_t lv, int32_t ru, int32_t rv, int32_t half) {
  orc_stats s = {0, 0, 0, 0, 0, 0};
  for (int dv = -half; dv <= half; ++dv) {
    const uint8_t* lr = L + (long)(lv + dv) * w;
    const uint8_t* rr = R + (long)(rv + dv) * w;
    for (int du = -half; du <= half; ++du) {
      if (((du + dv) & 1) != 0) continue;
      const int64_t a = lr[lu + du], b = rr[ru + du];
      s.n += 1;
      s.sl += a;
      s.sr += b;
      s.sll += a * a;
      s.srr += b * b;
      s.slr += a * b;
    }
  }
  return s;
}

/* Score of matcher.cpp:59-63; returns 0 and *defined=0 on zero variance. */
static double chess_score(const orc_stats* s, int* defined) {
  const int64_t var_l = s->n * s->sll - s->sl * s->sl;
  const int64_t var_r = s->n * s->srr - s->sr * s->sr;
  if (var_l == 0 || var_r == 0) {
    *defined = 0;
    return 0.0;
  }
  *defined = 1;
  const int64_t num = s->n * s->slr - s->sl * s->sr;
  return (double)num / sqrt((double)(var_l * var_r));
}

double orc_zncc_chessboard(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                           int32_t lu, int32_t lv, int32_t ru, int32_t rv, int32_t window,
                           int32_t* defined) {
  (void)h;
  const orc_stats s = chess_stats(left, right, w, lu, lv, ru, rv, window / 2);
  int def = 0;
  const double v = chess_score(&s, &def);
  *defined = def;
  return v;
}

/* compute_disparity, matcher.cpp:166-211 (== reference.cpp:7-53): per pixel
 * with the window inside the image, first maximum of the chessboard ZNCC over
 * d in [d_min, d_max] (right window must fit), accepted when >= min_zncc. */
int orc_compute_disparity(const orc_params* p, const uint8_t* L, const uint8_t* R,
                          int32_t w, int32_t h, float* disp, uint8_t* valid) {
  const int rc = orc_params_validate(p);
  if (rc) return rc;
  const long n = (long)w * h;
  memset(disp, 0, (size_t)n * sizeof(float));
  memset(valid, 0, (size_t)n);
  const int half = p->window / 2;
#pragma omp parallel for schedule(dynamic, 4)
  for (int v = half; v < h - half; ++v) {
    for (int u = half; u < w - half; ++u) {
      int found = 0, best_d = 0;
      double best = 0.0;
      for (int d = p->d_min; d <= p->d_max; ++d) {
        const int ru = u - d;
        if (ru < half || ru >= w - half) continue;
        const orc_stats s = chess_stats(L, R, w, u, v, ru, v, half);
        /* patch_stats (matcher.cpp:132-133) stores sum and var as int32; only
         * windows >= 27 can wrap, mirrored here for fidelity. */
        const int64_t var_l = (int32_t)(s.n * s.sll - s.sl * s.sl);
        const int64_t var_r = (int32_t)(s.n * s.srr - s.sr * s.sr);
        if (var_l == 0 || var_r == 0) continue;
        const int64_t num = s.n * s.slr - (int64_t)(int32_t)s.sl * (int32_t)s.sr;
        const double score = (double)num / sqrt((double)(var_l * var_r));
        if (!found || score > best) {
          found = 1;
          best = score;
          best_d = d;
        }
      }
      if (found && best >= p->min_zncc) {
        disp[(long)v * w + u] = (float)best_d;
        valid[(long)v * w + u] = 1;
      }
    }
  }
  return 0;
}

/* ---- Opt-in left-right consistency (extension: the reference has none;
 * SURVEY.md §8f row 1). Restated from its definition, independently of the
 * GPU's mirrored-sweep implementation (paper_2007_12623_b200/csrc/k_lr.cu).
 *
 * Right-view WTA: for a right pixel (x, v) whose window fits, the first
 * maximum over d in [d_min, d_max] of the chessboard ZNCC of (left at x + d,
 * right at x), the left window fitting and both variances non-zero (the same
 * arithmetic as compute_disparity above); valid iff found and >= min_zncc. */
int orc_compute_disparity_right(const orc_params* p, const uint8_t* L, const uint8_t* R,
                                int32_t w, int32_t h, float* disp, uint8_t* valid) {
  const int rc = orc_params_validate(p);
  if (rc) return rc;
  const long n = (long)w * h;
  memset(disp, 0, (size_t)n * sizeof(float));
  memset(valid, 0, (size_t)n);
  const int half = p->window / 2;
#pragma omp parallel for schedule(dynamic, 4)
  for (int v = half; v < h - half; ++v) {
    for (int x = half; x < w - half; ++x) {
      int found = 0, best_d = 0;
      double best = 0.0;
      for (int d = p->d_min; d <= p->d_max; ++d) {
        const int u = x + d;
        if (u < half || u >= w - half) continue;
        const orc_stats s = chess_stats(L, R, w, u, v, x, v, half);
        const int64_t var_l = (int32_t)(s.n * s.sll - s.sl * s.sl);
        const int64_t var_r = (int32_t)(s.n * s.srr - s.sr * s.sr);
        if (var_l == 0 || var_r == 0) continue;
        const int64_t num = s.n * s.slr - (int64_t)(int32_t)s.sl * (int32_t)s.sr;
        const double score = (double)num / sqrt((double)(var_l * var_r));
        if (!found || score > best) {
          found = 1;
          best = score;
          best_d = d;
        }
      }
      if (found && best >= p->min_zncc) {
        disp[(long)v * w + x] = (float)best_d;
        valid[(long)v * w + x] = 1;
      }
    }
  }
  return 0;
}

/* LR check: a valid left pixel u with disparity d is kept iff x = u - d is in
 * the image, the right view is valid at x and |d_R(x) - d| <= max_diff;
 * otherwise it becomes (0, invalid), the WTA's own "no match" output
 * (matcher.cpp:172). */
int orc_lr_check(const float* disp, const uint8_t* valid, const float* disp_r,
                 const uint8_t* valid_r, int32_t w, int32_t h, int32_t max_diff,
                 float* out_disp, uint8_t* out_valid) {
  if (max_diff < 0) return fail(1, "lr_check: max_diff must be >= 0");
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      const long i = (long)v * w + u;
      out_disp[i] = disp[i];
      out_valid[i] = valid[i];
      if (!valid[i]) continue;
      const int x = u - (int)disp[i];
      int ok = x >= 0 && x < w;
      if (ok) {
        const long j = (long)v * w + x;
        ok = valid_r[j] && fabsf(disp_r[j] - disp[i]) <= (float)max_diff;
      }
      if (!ok) {
        out_disp[i] = 0.f;
        out_valid[i] = 0;
      }
    }
  }
  return 0;
}

/* Ray directions of cleanup.cpp:8-9. */
static const int kDU[8] = {1, -1, 0, 0, 1, 1, -1, -1};
static const int kDV[8] = {0, 0, 1, -1, 1, -1, 1, -1};

/* remove_outliers, cleanup.cpp:12-42: keep a valid pixel iff one of the 8 rays
 * is in-bounds, valid and smooth (|cur - prev| <= thr in double) for r steps. */
int orc_remove_outliers(const float* disp, const uint8_t* valid, int32_t w, int32_t h,
                        int32_t radius, double thr, float* out_disp, uint8_t* out_valid) {
  const long n = (long)w * h;
  if (n) {
    memcpy(out_disp, disp, (size_t)n * sizeof(float));
    memcpy(out_valid, valid, (size_t)n);
  }
#pragma omp parallel for schedule(static)
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      if (!valid[(long)v * w + u]) continue;
      int keep = 0;
      for (int dir = 0; dir < 8 && !keep; ++dir) {
        double prev = disp[(long)v * w + u];
        int ok = 1;
        for (int step = 1; step <= radius; ++step) {
          const int nu = u + kDU[dir] * step, nv = v + kDV[dir] * step;
          if (nu < 0 || nu >= w || nv < 0 || nv >= h || !valid[(long)nv * w + nu]) {
            ok = 0;
            break;
          }
          const double cur = disp[(long)nv * w + nu];
          if (fabs(cur - prev) > thr) {
            ok = 0;
            break;
          }
          prev = cur;
        }
        keep = ok;
      }
      if (!keep) out_valid[(long)v * w + u] = 0;
    }
  }
  return 0;
}

/* fill_holes, cleanup.cpp:44-92. Accumulation order is the reference's:
 * direction 0..7 (radial), raster dv then du (disc). */
int orc_fill_holes(const float* disp, const uint8_t* valid, int32_t w, int32_t h,
                   int32_t mode, int32_t radius, int32_t min_support, float* out_disp,
                   uint8_t* out_valid) {
  const long n = (long)w * h;
  if (n) {
    memcpy(out_disp, disp, (size_t)n * sizeof(float));
    memcpy(out_valid, valid, (size_t)n);
  }
#pragma omp parallel for schedule(dynamic, 4)
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      if (valid[(long)v * w + u]) continue;
      double wsum = 0.0, vsum = 0.0;
      int support = 0;
      if (mode == 0) {
        for (int dir = 0; dir < 8; ++dir) {
          const double len = dir < 4 ? 1.0 : M_SQRT2;
          for (int step = 1; step <= radius; ++step) {
            const int nu = u + kDU[dir] * step, nv = v + kDV[dir] * step;
            if (nu < 0 || nu >= w || nv < 0 || nv >= h) break;
            if (!valid[(long)nv * w + nu]) continue;
            const double wt = 1.0 / (step * len);
            wsum += wt;
            vsum += wt * disp[(long)nv * w + nu];
            ++support;
            break;
          }
        }
      } else {
        const int r2 = radius * radius;
        for (int dv = -radius; dv <= radius; ++dv) {
          for (int du = -radius; du <= radius; ++du) {
            const int dd = du * du + dv * dv;
            if (dd == 0 || dd > r2) continue;
            const int nu = u + du, nv = v + dv;
            if (nu < 0 || nu >= w || nv < 0 || nv >= h || !valid[(long)nv * w + nu]) continue;
            const double wt = 1.0 / sqrt((double)dd);
            wsum += wt;
            vsum += wt * disp[(long)nv * w + nu];
            ++support;
          }
        }
      }
      if (support >= min_support && wsum > 0.0) {
        out_disp[(long)v * w + u] = (float)(vsum / wsum);
        out_valid[(long)v * w + u] = 1;
      }
    }
  }
  return 0;
}

/* cleanup.cpp:94-109. */
int32_t orc_disc_neighbor_count(int32_t radius) {
  int32_t c = 0;
  for (int dv = -radius; dv <= radius; ++dv)
    for (int du = -radius; du <= radius; ++du) {
      const int dd = du * du + dv * dv;
      if (dd != 0 && dd <= radius * radius) ++c;
    }
  return c;
}

int32_t orc_disc_fill_min_support(int32_t radius) {
  return (int32_t)ceil(0.25 * orc_disc_neighbor_count(radius));
}

/* cleanup_pass, cleanup.cpp:111-123. */
int orc_cleanup_pass(const orc_params* p, const float* disp, const uint8_t* valid, int32_t w,
                     int32_t h, float* out_disp, uint8_t* out_valid) {
  const long n = (long)w * h;
  float* d0 = malloc((size_t)(n ? n : 1) * sizeof(float));
  float* d1 = malloc((size_t)(n ? n : 1) * sizeof(float));
  uint8_t* v0 = malloc((size_t)(n ? n : 1));
  uint8_t* v1 = malloc((size_t)(n ? n : 1));
  if (n) {
    memcpy(d0, disp, (size_t)n * sizeof(float));
    memcpy(v0, valid, (size_t)n);
  }
  const int disc_support = orc_disc_fill_min_support(p->fill_radius_disc);
  for (int k = 0; k < p->cleanup_iterations; ++k) {
    const int r = p->outlier_radius_start + k * p->outlier_radius_step;
    orc_remove_outliers(d0, v0, w, h, r, p->neighbor_jump_threshold, d1, v1);
    orc_fill_holes(d1, v1, w, h, 0, p->fill_radius_radial, 4, d0, v0);
    orc_fill_holes(d0, v0, w, h, 1, p->fill_radius_disc, disc_support, d1, v1);
    float* td = d0; d0 = d1; d1 = td;
    uint8_t* tv = v0; v0 = v1; v1 = tv;
  }
  if (n) {
    memcpy(out_disp, d0, (size_t)n * sizeof(float));
    memcpy(out_valid, v0, (size_t)n);
  }
  free(d0); free(d1); free(v0); free(v1);
  return 0;
}

/* disc_average, smoothing.cpp:16-64: masked disc mean through serial
 * left-to-right double row prefixes, rows accumulated dy ascending. */
static void disc_average(const double* val, const uint8_t* mask, int w, int h, int radius,
                         double* psum, int* pcnt, double* out) {
  int span[1024];
  for (int dy = 0; dy <= radius; ++dy)
    span[dy] = (int)floor(sqrt((double)radius * radius - (double)dy * dy));
#pragma omp parallel for schedule(static)
  for (int v = 0; v < h; ++v) {
    double s = 0.0;
    int c = 0;
    double* ps = psum + (long)v * (w + 1);
    int* pc = pcnt + (long)v * (w + 1);
    ps[0] = 0.0;
    pc[0] = 0;
    for (int u = 0; u < w; ++u) {
      if (mask[(long)v * w + u]) {
        s += val[(long)v * w + u];
        c += 1;
      }
      ps[u + 1] = s;
      pc[u + 1] = c;
    }
  }
#pragma omp parallel for schedule(static)
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      const long i = (long)v * w + u;
      out[i] = 0.0;
      if (!mask[i]) continue;
      double s = 0.0;
      int c = 0;
      const int lo = -radius > -v ? -radius : -v;
      const int hi = radius < h - 1 - v ? radius : h - 1 - v;
      for (int dy = lo; dy <= hi; ++dy) {
        const int sx = span[dy < 0 ? -dy : dy];
        const int u0 = u - sx > 0 ? u - sx : 0;
        const int u1 = u + sx < w - 1 ? u + sx : w - 1;
        const long row = (long)(v + dy) * (w + 1);
        s += psum[row + u1 + 1] - psum[row + u0];
        c += pcnt[row + u1 + 1] - pcnt[row + u0];
      }
      out[i] = s / c;
    }
  }
}

/* refine_disparities, smoothing.cpp:68-159. */
int orc_refine_disparities(const orc_params* p, const float* disp, const uint8_t* valid,
                           const uint8_t* L, const uint8_t* R, int32_t w, int32_t h,
                           float* out_disp, uint8_t* out_valid, double* trace_discrete,
                           double* trace_smooth) {
  const long n = (long)w * h;
  if (p->smoothing_radius >= 1024) return fail(1, "refine: smoothing_radius too large for oracle");
  const double lo = p->d_min - 5;
  const double hi = p->d_max + 5;
  const long nn = n ? n : 1;
  double* o = calloc((size_t)nn, sizeof(double));
  double* d = calloc((size_t)nn, sizeof(double));
  double* avg = calloc((size_t)nn, sizeof(double));
  double* b = calloc((size_t)nn, sizeof(double));
  double* bavg = calloc((size_t)nn, sizeof(double));
  double* psum = malloc((size_t)(w + 1) * (h ? h : 1) * sizeof(double));
  int* pcnt = malloc((size_t)(w + 1) * (h ? h : 1) * sizeof(int));
  for (long i = 0; i < n; ++i)
    if (valid[i]) o[i] = d[i] = disp[i];
  const int half = p->window / 2;
  const double one_minus_alpha = 1.0 - p->alpha;
  for (int it = 0; it < p->refine_iterations; ++it) {
    disc_average(o, valid, w, h, p->smoothing_radius, psum, pcnt, avg);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i)
      if (valid[i]) b[i] = avg[i] - p->alpha * o[i] - one_minus_alpha * d[i];
    disc_average(b, valid, w, h, p->smoothing_radius, psum, pcnt, bavg);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
      if (!valid[i]) continue;
      const double x = avg[i] - bavg[i];
      d[i] = x < lo ? lo : (hi < x ? hi : x); /* std::clamp */
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int v = 0; v < h; ++v) {
      for (int u = 0; u < w; ++u) {
        const long i = (long)v * w + u;
        if (!valid[i]) continue;
        const double dv = d[i];
        const int c_lo0 = (int)ceil(dv - 5), c_lo1 = (int)ceil(lo);
        const int c_hi0 = (int)floor(dv + 5), c_hi1 = (int)floor(hi);
        const int c_lo = c_lo0 > c_lo1 ? c_lo0 : c_lo1;
        const int c_hi = c_hi0 < c_hi1 ? c_hi0 : c_hi1;
        const int fits = u >= half && u < w - half && v >= half && v < h - half;
        double best_cost = 0.0;
        int best = 0, found = 0;
        for (int c = c_lo; c <= c_hi; ++c) {
          double match = 1.0 / 1e-3;
          const int ru = u - c;
          if (fits && ru >= half && ru < w - half) {
            const orc_stats s = chess_stats(L, R, w, u, v, ru, v, half);
            int def = 0;
            const double score = chess_score(&s, &def);
            if (def) match = 1.0 / (score > 1e-3 ? score : 1e-3);
          }
          const double diff = c - dv;
          const double cost = match + p->eta_smooth * diff * diff;
          if (!found || cost < best_cost) {
            found = 1;
            best_cost = cost;
            best = c;
          }
        }
        if (found) o[i] = best;
      }
    }
    if (trace_discrete) memcpy(trace_discrete + (long)it * n, o, (size_t)n * sizeof(double));
    if (trace_smooth) memcpy(trace_smooth + (long)it * n, d, (size_t)n * sizeof(double));
  }
  for (long i = 0; i < n; ++i) {
    out_disp[i] = valid[i] ? (float)d[i] : disp[i];
    out_valid[i] = valid[i];
  }
  free(o); free(d); free(avg); free(b); free(bavg); free(psum); free(pcnt);
  return 0;
}

/* ---- disparity_to_cloud restatement (cloud.cpp:14-94), Eigen-free ---- */

/* Restatement of Eigen 3.4.0 SelfAdjointEigenSolver<Matrix3d>::compute(A,
 * ComputeEigenvectors) — the call at cloud.cpp:78 — in the same operations
 * and order (Eigen/src/Eigenvalues/SelfAdjointEigenSolver.h,
 * Tridiagonalization.h, Jacobi/Jacobi.h, scalar double, no FMA):
 *  1. mat = lower triangle of A; scale = max |mat_ij| (1 if 0); mat /= scale;
 *  2. tridiagonalization_inplace_selector<Matrix3d, 3, false>::run: one
 *     Householder reflection, Q returned in mat;
 *  3. computeFromTridiagonal_impl: deflate (|e_i| < DBL_MIN, or
 *     (e_i / eps)^2 <= |d_i| + |d_i+1|), implicit symmetric QR steps with a
 *     Wilkinson shift (tridiagonal_qr_step), Givens rotations from
 *     JacobiRotation::makeGivens applied to Q on the right; at most 30 n
 *     iterations;
 *  4. eigenvalues sorted ascending with their columns (first minimum),
 *     then multiplied by scale.
 * evec[r][k] = component r of the eigenvector of evals[k]. Returns 0, or 1
 * when the QR iteration did not converge (Eigen's NoConvergence). */
static double eg_hypot(double x, double y) { /* Eigen positive_real_hypot(|x|, |y|) */
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  const double p = x > y ? x : y; /* numext::maxi(x, y) */
  if (p == 0.0) return 0.0;
  const double qp = (y < x ? y : x) / p; /* numext::mini(y, x) / p */
  return p * sqrt(1.0 + qp * qp);
}

static void eg_givens(double p, double q, double* c, double* s) { /* makeGivens(p, q) */
  if (q == 0.0) {
    *c = p < 0.0 ? -1.0 : 1.0;
    *s = 0.0;
  } else if (p == 0.0) {
    *c = 0.0;
    *s = q < 0.0 ? 1.0 : -1.0;
  } else if (fabs(p) > fabs(q)) {
    const double t = q / p;
    double u = sqrt(1.0 + t * t);
    if (p < 0.0) u = -u;
    *c = 1.0 / u;
    *s = -t * *c;
  } else {
    const double t = p / q;
    double u = sqrt(1.0 + t * t);
    if (q < 0.0) u = -u;
    *s = -1.0 / u;
    *c = -t * *s;
  }
}

/* tridiagonal_qr_step<ColMajor>(diag, subdiag, start, end, Q, 3) */
static void eg_qr_step(double* diag, double* sub, int start, int end, double Q[3][3]) {
  const double td = (diag[end - 1] - diag[end]) * 0.5;
  const double e = sub[end - 1];
  double mu = diag[end];
  if (td == 0.0) {
    mu -= fabs(e);
  } else if (e != 0.0) {
    const double e2 = e * e;
    const double h = eg_hypot(td, e);
    if (e2 == 0.0)
      mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
    else
      mu -= e2 / (td + (td > 0.0 ? h : -h));
  }
  double x = diag[start] - mu;
  double z = sub[start];
  for (int k = start; k < end && z != 0.0; ++k) {
    double c, s;
    eg_givens(x, z, &c, &s);
    const double sdk = s * diag[k] + c * sub[k];
    const double dkp1 = s * sub[k] + c * diag[k + 1];
    diag[k] = c * (c * diag[k] - s * sub[k]) - s * (c * sub[k] - s * diag[k + 1]);
    diag[k + 1] = s * sdk + c * dkp1;
    sub[k] = c * sdk - s * dkp1;
    if (k > start) sub[k - 1] = c * sub[k - 1] - s * z;
    x = sub[k];
    if (k < end - 1) {
      z = -s * sub[k + 1];
      sub[k + 1] = c * sub[k + 1];
    }
    /* Q = Q * G: columns k, k+1 rotated by G' = (c, -s) (applyOnTheRight) */
    for (int i = 0; i < 3; ++i) {
      const double xi = Q[i][k], yi = Q[i][k + 1];
      Q[i][k] = c * xi + (-s) * yi;
      Q[i][k + 1] = -(-s) * xi + c * yi;
    }
  }
}

static int eigen3_sym(const double A[3][3], double evals[3], double evec[3][3]) {
  double m[3][3] = {{0}};
  double scale = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c <= r; ++c) {
      m[r][c] = A[r][c];
      if (fabs(m[r][c]) > scale) scale = fabs(m[r][c]);
    }
  if (scale == 0.0) scale = 1.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c <= r; ++c) m[r][c] /= scale;
  double diag[3], sub[2];
  /* tridiagonalization_inplace_selector<MatrixType, 3, false>::run */
  diag[0] = m[0][0];
  const double v1norm2 = m[2][0] * m[2][0];
  if (v1norm2 <= DBL_MIN) {
    diag[1] = m[1][1];
    diag[2] = m[2][2];
    sub[0] = m[1][0];
    sub[1] = m[2][1];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) evec[r][c] = r == c ? 1.0 : 0.0;
  } else {
    const double beta = sqrt(m[1][0] * m[1][0] + v1norm2);
    const double invBeta = 1.0 / beta;
    const double m01 = m[1][0] * invBeta;
    const double m02 = m[2][0] * invBeta;
    const double q = 2.0 * m01 * m[2][1] + m02 * (m[2][2] - m[1][1]);
    diag[1] = m[1][1] + m02 * q;
    diag[2] = m[2][2] - m02 * q;
    sub[0] = beta;
    sub[1] = m[2][1] - m01 * q;
    const double Q[3][3] = {{1, 0, 0}, {0, m01, m02}, {0, m02, -m01}};
    memcpy(evec, Q, sizeof Q);
  }
  /* computeFromTridiagonal_impl(diag, subdiag, 30, true, evec) */
  const int n = 3, max_iter = 30;
  const double precision_inv = 1.0 / DBL_EPSILON;
  int end = n - 1, start = 0, iter = 0;
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (fabs(sub[i]) < DBL_MIN) {
        sub[i] = 0.0;
      } else {
        const double scaled = precision_inv * sub[i];
        if (scaled * scaled <= (fabs(diag[i]) + fabs(diag[i + 1]))) sub[i] = 0.0;
      }
    }
    while (end > 0 && sub[end - 1] == 0.0) end--;
    if (end <= 0) break;
    iter++;
    if (iter > max_iter * n) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;
    eg_qr_step(diag, sub, start, end, evec);
  }
  const int ok = iter <= max_iter * n;
  if (ok) {
    for (int i = 0; i < n - 1; ++i) {
      int k = 0; /* minCoeff over diag[i..n): first minimum */
      for (int j = 1; j < n - i; ++j)
        if (diag[i + j] < diag[i + k]) k = j;
      if (k > 0) {
        const double t = diag[i];
        diag[i] = diag[k + i];
        diag[k + i] = t;
        for (int r = 0; r < 3; ++r) {
          const double tv = evec[r][i];
          evec[r][i] = evec[r][k + i];
          evec[r][k + i] = tv;
        }
      }
    }
  }
  for (int k = 0; k < 3; ++k) evals[k] = diag[k] * scale;
  return ok ? 0 : 1;
}

int orc_eigen3_sym(const double* a9, double* evals, double* evec9) {
  double A[3][3], V[3][3];
  memcpy(A, a9, sizeof A);
  const int rc = eigen3_sym(A, evals, V);
  memcpy(evec9, V, sizeof V);
  return rc;
}

int orc_disparity_to_cloud(const float* disp, const uint8_t* valid, int32_t w, int32_t h,
                           const uint8_t* rgb, int32_t cw, int32_t ch, const orc_rig* rig,
                           int32_t* index, double* points, double* normals, uint8_t* colors,
                           int32_t* pixels, int32_t* n_points, double* eigen_gap,
                           double* decision) {
  const int rc = orc_rig_validate(rig);
  if (rc) return rc;
  const long n = (long)w * h;
  int32_t np = 0;
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      const long i = (long)v * w + u;
      index[i] = -1;
      if (!valid[i]) continue;
      const double d = disp[i];
      if (!(d > 1e-6)) continue;
      const double z = rig->fx * rig->baseline_mm / d;
      index[i] = np;
      points[3 * np + 0] = z * (u - rig->cx) / rig->fx;
      points[3 * np + 1] = z * (v - rig->cy) / rig->fy;
      points[3 * np + 2] = z;
      if (u >= 0 && u < cw && v >= 0 && v < ch) {
        const uint8_t* c = rgb + ((long)v * cw + u) * 3;
        colors[3 * np + 0] = c[0];
        colors[3 * np + 1] = c[1];
        colors[3 * np + 2] = c[2];
      } else {
        colors[3 * np + 0] = colors[3 * np + 1] = colors[3 * np + 2] = 0;
      }
      pixels[2 * np + 0] = u;
      pixels[2 * np + 1] = v;
      ++np;
    }
  }
  (void)n;
  *n_points = np;
#pragma omp parallel for schedule(dynamic, 4)
  for (int v = 0; v < h; ++v) {
    for (int u = 0; u < w; ++u) {
      const int32_t pi = index[(long)v * w + u];
      if (pi < 0) continue;
      const double* p = points + 3 * pi;
      double mean[3] = {0, 0, 0};
      int count = 0;
      for (int dv = -3; dv <= 3; ++dv)
        for (int du = -3; du <= 3; ++du) {
          const int nu = u + du, nv = v + dv;
          if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
          const int32_t ni = index[(long)nv * w + nu];
          if (ni < 0) continue;
          mean[0] += points[3 * ni + 0];
          mean[1] += points[3 * ni + 1];
          mean[2] += points[3 * ni + 2];
          ++count;
        }
      double nrm[3] = {0.0, 0.0, -1.0};
      int fitted = 0;
      double gap = -1.0, margin = -INFINITY;
      if (count >= 3) {
        mean[0] /= count;
        mean[1] /= count;
        mean[2] /= count;
        double cov[3][3] = {{0}};
        for (int dv = -3; dv <= 3; ++dv)
          for (int du = -3; du <= 3; ++du) {
            const int nu = u + du, nv = v + dv;
            if (nu < 0 || nu >= w || nv < 0 || nv >= h) continue;
            const int32_t ni = index[(long)nv * w + nu];
            if (ni < 0) continue;
            const double q[3] = {points[3 * ni] - mean[0], points[3 * ni + 1] - mean[1],
                                 points[3 * ni + 2] - mean[2]};
            for (int r = 0; r < 3; ++r)
              for (int c = 0; c < 3; ++c) cov[r][c] += q[r] * q[c];
          }
        double ev[3], vec[3][3];
        eigen3_sym(cov, ev, vec);
        const double m = ev[2] > 1.0 ? ev[2] : 1.0; /* std::max(1.0, ev(2)) */
        margin = (ev[1] - 1e-9 * m) / (1e-9 * m);
        if (ev[1] > 1e-9 * m) { /* cloud.cpp:81 */
          nrm[0] = vec[0][0];
          nrm[1] = vec[1][0];
          nrm[2] = vec[2][0];
          fitted = 1;
          gap = ev[2] > 0 ? (ev[1] - ev[0]) / ev[2] : 0.0;
        }
      }
      if (!fitted) {
        const double len = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        nrm[0] = -p[0] / len;
        nrm[1] = -p[1] / len;
        nrm[2] = -p[2] / len;
      }
      if (nrm[0] * p[0] + nrm[1] * p[1] + nrm[2] * p[2] > 0.0) {
        nrm[0] = -nrm[0];
        nrm[1] = -nrm[1];
        nrm[2] = -nrm[2];
      }
      normals[3 * pi + 0] = nrm[0];
      normals[3 * pi + 1] = nrm[1];
      normals[3 * pi + 2] = nrm[2];
      if (eigen_gap) eigen_gap[pi] = gap;
      if (decision) decision[pi] = margin;
    }
  }
  return 0;
}

/* ---- Fusion consumer (SPEC.md:440-476 [MODULE]
 * fusion). No reference source exists (SPEC only): this is the restatement
 * the GPU fusion is held to, with the SPEC's examples and properties as KATs
 * ("parity unpinned" against reference code). Conventions (also
 * include/ss_stereo.h):
 *   pose[12]  row-major [R | t], world -> camera: X_cam = R X_world + t
 *   surfels   SoA, pos/normal/color/weight/color_weight in double
 *   rasterize: X_cam.z > 0; pixel = (floor(fx x/z + cx + 0.5),
 *              floor(fy y/z + cy + 0.5)); smallest depth wins, then the
 *              smaller surfel id
 *   fuse     : per stereo pixel with a point (raster order), associate with
 *              the raster's surfel when |z - z_s| <= gate, else append. */
static void orc_apply(const double* P, const double x[3], double y[3]) {
  for (int r = 0; r < 3; ++r)
    y[r] = ((P[4 * r] * x[0] + P[4 * r + 1] * x[1]) + P[4 * r + 2] * x[2]) + P[4 * r + 3];
}
static void orc_apply_inv(const double* P, const double y[3], double x[3]) {
  const double d0 = y[0] - P[3], d1 = y[1] - P[7], d2 = y[2] - P[11];
  for (int c = 0; c < 3; ++c) x[c] = (P[c] * d0 + P[4 + c] * d1) + P[8 + c] * d2;
}
static void orc_rot_inv(const double* P, const double y[3], double x[3]) {
  for (int c = 0; c < 3; ++c) x[c] = (P[c] * y[0] + P[4 + c] * y[1]) + P[8 + c] * y[2];
}

int orc_rasterize(const double* pos, int32_t n, const double* pose, double fx, double fy,
                  double cx, double cy, int32_t w, int32_t h, int32_t* ids, double* depth) {
  for (long i = 0; i < (long)w * h; ++i) {
    ids[i] = -1;
    depth[i] = 0.0;
  }
  for (int32_t s = 0; s < n; ++s) {
    double q[3];
    orc_apply(pose, pos + 3L * s, q);
    if (!(q[2] > 0.0)) continue;
    const double u = (fx * q[0]) / q[2] + cx, v = (fy * q[1]) / q[2] + cy;
    const double fu = floor(u + 0.5), fv = floor(v + 0.5);
    if (!(fu >= 0.0 && fu < (double)w && fv >= 0.0 && fv < (double)h)) continue;
    const long k = (long)fv * w + (long)fu;
    if (ids[k] < 0 || q[2] < depth[k] || (q[2] == depth[k] && s < ids[k])) {
      ids[k] = s;
      depth[k] = q[2];
    }
  }
  return 0;
}

/* Colour weight of pixel (u, v): clamp(1 - r / R, omega_min, 1), r the
 * distance to the image centre ((w-1)/2, (h-1)/2), R the half-diagonal. */
static double orc_omega(int u, int v, int w, int h, double omega_min) {
  const double cu = 0.5 * (double)(w - 1), cv = 0.5 * (double)(h - 1);
  const double du = (double)u - cu, dv = (double)v - cv;
  const double r = sqrt(du * du + dv * dv), R = sqrt(cu * cu + cv * cv);
  double o = R > 0.0 ? 1.0 - r / R : 1.0;
  if (o < omega_min) o = omega_min;
  if (o > 1.0) o = 1.0;
  return o;
}

/* One frame into the model (arrays of capacity cap; *n in/out). */
int orc_fuse_frame(double* pos, double* nrm, double* col, double* wgt, double* cwgt, int32_t* n,
                   int32_t cap, const int32_t* index, const double* pts, const double* nrms,
                   const uint8_t* colors, int32_t w, int32_t h, const double* pose, double fx,
                   double fy, double cx, double cy, double trunc, double weight_cap,
                   double gate, double omega_min) {
  const long N = (long)w * h;
  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
  double* dep = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
  orc_rasterize(pos, *n, pose, fx, fy, cx, cy, w, h, ids, dep);
  int32_t m = *n;
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const long k = (long)v * w + u;
      const int32_t p = index[k];
      if (p < 0) continue;
      double xw[3], nw[3];
      orc_apply_inv(pose, pts + 3L * p, xw);
      orc_rot_inv(pose, nrms + 3L * p, nw);
      const double om = orc_omega(u, v, w, h, omega_min);
      const double c[3] = {(double)colors[3L * p], (double)colors[3L * p + 1],
                           (double)colors[3L * p + 2]};
      const int32_t s = ids[k];
      if (s >= 0 && fabs(pts[3L * p + 2] - dep[k]) <= gate) {
        double* P = pos + 3L * s;
        double d[3] = {xw[0] - P[0], xw[1] - P[1], xw[2] - P[2]};
        const double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        if (len > trunc) {
          const double f = trunc / len;
          d[0] *= f;
          d[1] *= f;
          d[2] *= f;
        }
        const double wo = wgt[s], inv = 1.0 / (wo + 1.0);
        for (int i = 0; i < 3; ++i) P[i] = P[i] + d[i] * inv;
        double* Nn = nrm + 3L * s;
        double a[3];
        for (int i = 0; i < 3; ++i) a[i] = wo * Nn[i] + nw[i];
        const double al = sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
        if (al > 0.0)
          for (int i = 0; i < 3; ++i) Nn[i] = a[i] / al;
        double* C = col + 3L * s;
        const double cw = cwgt[s], cs = cw + om;
        for (int i = 0; i < 3; ++i) C[i] = (cw * C[i] + om * c[i]) / cs;
        wgt[s] = wo + 1.0 < weight_cap ? wo + 1.0 : weight_cap;
        cwgt[s] = cs < weight_cap ? cs : weight_cap;
      } else {
        if (m >= cap) {
          free(ids);
          free(dep);
          return fail(2, "fuse_frame: surfel capacity exceeded");
        }
        for (int i = 0; i < 3; ++i) {
          pos[3L * m + i] = xw[i];
          nrm[3L * m + i] = nw[i];
          col[3L * m + i] = c[i];
        }
        wgt[m] = 1.0;
        cwgt[m] = om;
        ++m;
      }
    }
  *n = m;
  free(ids);
  free(dep);
  return 0;
}
