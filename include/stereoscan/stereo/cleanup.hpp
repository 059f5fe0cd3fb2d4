// Outlier removal / hole filling — /root/reference/proj/include/stereoscan/stereo/cleanup.hpp:12-32.
#pragma once

#include "stereoscan/stereo/image.hpp"
#include "stereoscan/stereo/params.hpp"

namespace stereoscan {

DisparityMap remove_outliers(const DisparityMap& map, int radius, double threshold);

enum class FillMode { Radial, Disc };

DisparityMap fill_holes(const DisparityMap& map, FillMode mode, int radius, int min_support);

int disc_neighbor_count(int radius);
int disc_fill_min_support(int radius);

DisparityMap cleanup_pass(const DisparityMap& map, const StereoParams& params);

}  // namespace stereoscan
