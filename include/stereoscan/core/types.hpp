// Eigen-free core types of the B200 stereo path.
// Mirrors /root/reference/proj/include/stereoscan/core/types.hpp:16-40
// (Error, CameraIntrinsics, StereoRig). Vec2 / Vec3 replace Eigen::Vector2d /
// Vector3d with PODs exposing the accessors the stereo and feature paths use; RigidPose and
// the rest of the SLAM types are out of scope.
#pragma once

#include <cmath>
#include <stdexcept>
#include <string>

namespace stereoscan {

// Runtime failures carry a human-readable message (types.hpp:16-21).
// Contract violations throw std::invalid_argument instead.
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct Vec2 {
  double v[2] = {0.0, 0.0};
  Vec2() = default;
  Vec2(double x, double y) : v{x, y} {}
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  Vec2 operator-(const Vec2& o) const { return Vec2(v[0] - o.v[0], v[1] - o.v[1]); }
  bool operator==(const Vec2& o) const { return v[0] == o.v[0] && v[1] == o.v[1]; }
};

struct Vec3 {
  double v[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
  double& operator()(int i) { return v[i]; }
  double operator()(int i) const { return v[i]; }
  double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
  double norm() const { return std::sqrt(dot(*this)); }
};

struct CameraIntrinsics {
  double fx = 0.0;  // focal lengths, pixels
  double fy = 0.0;
  double cx = 0.0;  // principal point, pixels
  double cy = 0.0;
  int width = 0;
  int height = 0;

  // Throws Error naming the first violated field (geometry.cpp:7-14).
  void validate() const;
};

struct StereoRig {
  CameraIntrinsics intrinsics;  // shared by both rectified cameras
  double baseline_mm = 0.0;

  void validate() const;  // geometry.cpp:16-19
};

}  // namespace stereoscan
