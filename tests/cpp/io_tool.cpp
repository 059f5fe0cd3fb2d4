// Test driver for include/stereoscan/io/io.hpp (tests/test_io.py calls it).
//   io_tool calib <path>                -> "fx fy cx cy width height baseline" or "ERROR <msg>"
//   io_tool png <path>                  -> "w h sum" (sum of all RGB bytes) or "ERROR <msg>"
//   io_tool pngsave <path> <w> <h>      -> writes a deterministic gradient RGB PNG
//   io_tool pgm <path>                  -> writes a 4x2 map: 7.0, 7.5, -1, 300, invalid(9), 0.001, 255.998, 0
//   io_tool ply <path> <n>              -> writes n points (i, 2i, 3i), normal (0,0,-1), colour white
//   io_tool stereo <calib> <dir> <frame> <out_prefix> <d_min> <d_max>  (GPU) -> "points <n>"
#include <cstdio>
#include <cstdlib>
#include <string>

#include "stereoscan/io/io.hpp"

using namespace stereoscan;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string cmd = argv[1], path = argv[2];
  try {
    if (cmd == "calib") {
      const StereoRig r = io::load_calibration(path);
      std::printf("%.17g %.17g %.17g %.17g %d %d %.17g\n", r.intrinsics.fx, r.intrinsics.fy,
                  r.intrinsics.cx, r.intrinsics.cy, r.intrinsics.width, r.intrinsics.height,
                  r.baseline_mm);
    } else if (cmd == "png") {
      const ColorImage im = io::load_png(path);
      unsigned long long s = 0;
      for (uint8_t b : im.pixels) s += b;
      std::printf("%d %d %llu\n", im.width, im.height, s);
    } else if (cmd == "pngsave") {
      ColorImage im(std::atoi(argv[3]), std::atoi(argv[4]));
      for (size_t i = 0; i < im.pixels.size(); ++i) im.pixels[i] = static_cast<uint8_t>(i * 7 % 251);
      io::save_png(path, im);
    } else if (cmd == "pgm") {
      DisparityMap m(4, 2);
      const float d[8] = {7.0f, 7.5f, -1.0f, 300.0f, 9.0f, 0.001f, 255.998f, 0.0f};
      for (int i = 0; i < 8; ++i) {
        m.disparity[i] = d[i];
        m.valid[i] = i == 4 ? 0 : 1;
      }
      io::write_disparity_pgm16(path, m);
    } else if (cmd == "ply") {
      StereoCloud c;
      const int n = std::atoi(argv[3]);
      for (int i = 0; i < n; ++i) {
        c.points.push_back(Vec3(i, 2.0 * i, 3.0 * i));
        c.normals.push_back(Vec3(0, 0, -1));
        c.colors.push_back({255, 255, 255});
      }
      io::export_ply(path, c);
    } else if (cmd == "stereo") {
      StereoParams p;
      p.d_min = std::atoi(argv[6]);
      p.d_max = std::atoi(argv[7]);
      const int n = io::run_stereo_only(path, argv[3], std::atoi(argv[4]), p, argv[5]);
      std::printf("points %d\n", n);
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
  }
  return 0;
}
