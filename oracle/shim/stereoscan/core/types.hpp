// ORACLE BUILD SHIM — test infrastructure only, never part of the product.
//
// The reference's real core/types.hpp pulls in Eigen (absent on this machine,
// see SURVEY.md fact 3). The four stereo translation units (matcher.cpp,
// reference.cpp, cleanup.cpp, smoothing.cpp) only need stereoscan::Error from
// it (via stereo/params.hpp:3); features.cpp additionally stores positions in
// Vec2 / Vec3 and subtracts Vec2s, so this shim provides Error plus minimal
// Eigen-free Vec2 / Vec3 with the members features.cpp uses (2-/3-argument
// construction, x(), y(), z(), binary minus) and nothing else. It is placed
// ahead of the reference include directory by oracle/Makefile.
//
// Mirrors /root/reference/proj/include/stereoscan/core/types.hpp:10-21.
#pragma once

#include <stdexcept>
#include <string>

namespace stereoscan {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct Vec2 {
  double c[2] = {0.0, 0.0};
  Vec2() = default;
  Vec2(double x, double y) : c{x, y} {}
  double x() const { return c[0]; }
  double y() const { return c[1]; }
  Vec2 operator-(const Vec2& o) const { return Vec2(c[0] - o.c[0], c[1] - o.c[1]); }
};

struct Vec3 {
  double c[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : c{x, y, z} {}
  double x() const { return c[0]; }
  double y() const { return c[1]; }
  double z() const { return c[2]; }
};

}  // namespace stereoscan
