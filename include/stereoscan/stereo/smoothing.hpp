// Refinement — /root/reference/proj/include/stereoscan/stereo/smoothing.hpp:10-24.
#pragma once

#include <vector>

#include "stereoscan/stereo/image.hpp"
#include "stereoscan/stereo/params.hpp"

namespace stereoscan {

struct RefineTrace {
  std::vector<std::vector<double>> discrete;
  std::vector<std::vector<double>> smooth;
};

DisparityMap refine_disparities(const DisparityMap& map, const GrayImage& left,
                                const GrayImage& right, const StereoParams& params,
                                RefineTrace* trace = nullptr);

}  // namespace stereoscan
