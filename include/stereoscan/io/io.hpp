// io formats either side of the stereo path (SPEC.md
// [MODULE] io, :517-534, and run_stereo_only, :581-589). The reference ships
// no io source; these follow the SPEC's formats and error rules. Host code
// (zlib for PNG); run_stereo_only drives the GPU path.
#pragma once

#include <string>
#include <utility>

#include "stereoscan/core/types.hpp"
#include "stereoscan/stereo/cloud.hpp"
#include "stereoscan/stereo/image.hpp"
#include "stereoscan/stereo/params.hpp"

namespace stereoscan::io {

// "key = value" lines ('#' comments) with fx, fy, cx, cy, baseline_mm, width,
// height. Errors (stereoscan::Error) name the file, the line and the key:
// missing key, non-numeric value, unknown key; then StereoRig::validate().
StereoRig load_calibration(const std::string& path);

// 8-bit PNG (grey, grey+alpha, RGB, RGBA; non-interlaced) -> RGB.
ColorImage load_png(const std::string& path);
// RGB -> 8-bit RGB PNG (deterministic bytes for identical inputs).
void save_png(const std::string& path, const ColorImage& img);

// <dir>/left_NNNNNN.png and right_NNNNNN.png (6-digit zero padded); both must
// match the calibration's width/height (Error otherwise).
std::pair<ColorImage, ColorImage> load_frame_pair(const std::string& dir, int index,
                                                  const StereoRig& rig);

// 16-bit binary PGM (P5, maxval 65535, big-endian): clamp(lround(256 d), 0,
// 65535) on valid pixels, 0 on invalid ones.
void write_disparity_pgm16(const std::string& path, const DisparityMap& map);
// Reads it back (values as stored).
std::vector<uint16_t> read_pgm16(const std::string& path, int* width, int* height);

// Binary little-endian PLY: x y z nx ny nz float32 (mm), red green blue uchar,
// points in cloud order; byte-deterministic.
void export_ply(const std::string& path, const StereoCloud& cloud);

// run_stereo_only: load frame `index` from `dir`, run the
// full stereo stage on the GPU (to_gray -> compute_disparity -> cleanup_pass
// -> refine_disparities -> disparity_to_cloud) and write <out_prefix>.ply and
// <out_prefix>_disparity.pgm. Returns the number of points.
int run_stereo_only(const std::string& calibration, const std::string& dir, int index,
                    const StereoParams& params, const std::string& out_prefix);

}  // namespace stereoscan::io
