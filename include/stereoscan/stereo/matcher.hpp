// ZNCC matching entry points — /root/reference/proj/include/stereoscan/stereo/matcher.hpp:16-36.
// compute_disparity runs on the GPU (ss_compute_disparity); the scalar helpers
// are host utilities with the reference's exact integer/double arithmetic.
#pragma once

#include <optional>

#include "stereoscan/stereo/image.hpp"
#include "stereoscan/stereo/params.hpp"

namespace stereoscan {

std::optional<double> zncc_chessboard(const GrayImage& left, int lu, int lv,
                                      const GrayImage& right, int ru, int rv, int window);

std::optional<double> zncc_score(const GrayImage& left_patch, const GrayImage& right_patch);

std::optional<int> match_pixel(const GrayImage& left, const GrayImage& right, int u, int v,
                               const StereoParams& params);

// Dense integer disparity search on the B200 (bit-exact with the reference).
DisparityMap compute_disparity(const GrayImage& left, const GrayImage& right,
                               const StereoParams& params);

// Extension (no reference analogue): compute_disparity
// followed by a left-right consistency check. A valid pixel u with disparity d
// is kept iff x = u - d is inside the image, the right-view WTA (first argmax
// over d of zncc(left at x + d, right at x)) is valid at x and within max_diff
// of d; rejected pixels become (0, invalid). `right_map`, when given, receives
// the right-view map. max_diff < 0 throws std::invalid_argument.
DisparityMap compute_disparity_lr(const GrayImage& left, const GrayImage& right,
                                  const StereoParams& params, int max_diff = 1,
                                  DisparityMap* right_map = nullptr);

}  // namespace stereoscan
