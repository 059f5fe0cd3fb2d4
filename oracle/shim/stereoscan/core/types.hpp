// ORACLE BUILD SHIM — test infrastructure only, never part of the product.
//
// The reference's real core/types.hpp pulls in Eigen (absent on this machine,
// see SURVEY.md fact 3). The four hot-path translation units
// (matcher.cpp, reference.cpp, cleanup.cpp, smoothing.cpp) only need
// stereoscan::Error from it (via stereo/params.hpp:3), so this shim provides
// exactly that and nothing else. It is placed ahead of the reference include
// directory by oracle/Makefile.
//
// Mirrors /root/reference/proj/include/stereoscan/core/types.hpp:16-21.
#pragma once

#include <stdexcept>
#include <string>

namespace stereoscan {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

}  // namespace stereoscan
