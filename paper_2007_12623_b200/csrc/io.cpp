// io formats around the stereo path (include/stereoscan/io/io.hpp; SPEC.md
// [MODULE] io and run_stereo_only). Host code: a minimal PNG codec on zlib,
// line-oriented calibration parsing, 16-bit PGM and binary PLY writers.
#include "stereoscan/io/io.hpp"

#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <vector>

#include "stereoscan/stereo/cleanup.hpp"
#include "stereoscan/stereo/matcher.hpp"
#include "stereoscan/stereo/smoothing.hpp"

namespace stereoscan::io {

namespace {

std::vector<uint8_t> read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error("cannot open " + path);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const std::string& bytes) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Error("cannot write " + path);
  f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!f) throw Error("cannot write " + path);
}

uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}
void put_be32(std::string& s, uint32_t x) {
  for (int k = 3; k >= 0; --k) s.push_back(static_cast<char>((x >> (8 * k)) & 0xFF));
}

int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

void png_chunk(std::string& out, const char* type, const std::string& data) {
  put_be32(out, static_cast<uint32_t>(data.size()));
  std::string td(type, 4);
  td += data;
  out += td;
  put_be32(out, static_cast<uint32_t>(crc32(0L, reinterpret_cast<const Bytef*>(td.data()),
                                            static_cast<uInt>(td.size()))));
}

}  // namespace

StereoRig load_calibration(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error("cannot open calibration file: " + path);
  static const char* kKeys[] = {"fx", "fy", "cx", "cy", "baseline_mm", "width", "height"};
  std::map<std::string, double> kv;
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    const size_t eq = line.find('=');
    auto trim = [](std::string s) {
      const size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
      return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
    };
    const std::string where = path + ":" + std::to_string(no);
    if (eq == std::string::npos) throw Error(where + ": expected 'key = value'");
    const std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
    if (std::find_if(std::begin(kKeys), std::end(kKeys),
                     [&](const char* k) { return key == k; }) == std::end(kKeys))
      throw Error(where + ": unknown key \"" + key + "\"");
    char* end = nullptr;
    const double x = std::strtod(val.c_str(), &end);
    if (val.empty() || end == val.c_str() || *end != '\0' || !std::isfinite(x))
      throw Error(where + ": non-numeric value for \"" + key + "\"");
    kv[key] = x;
  }
  for (const char* k : kKeys)
    if (!kv.count(k)) throw Error(path + ": missing key \"" + std::string(k) + "\"");
  for (const char* k : {"width", "height"})
    if (kv[k] != std::floor(kv[k])) throw Error(path + ": \"" + std::string(k) + "\" must be an integer");
  StereoRig rig;
  rig.intrinsics.fx = kv["fx"];
  rig.intrinsics.fy = kv["fy"];
  rig.intrinsics.cx = kv["cx"];
  rig.intrinsics.cy = kv["cy"];
  rig.intrinsics.width = static_cast<int>(kv["width"]);
  rig.intrinsics.height = static_cast<int>(kv["height"]);
  rig.baseline_mm = kv["baseline_mm"];
  rig.validate();  // names the violated field (geometry.cpp:7-19)
  return rig;
}

ColorImage load_png(const std::string& path) {
  const std::vector<uint8_t> f = read_file(path);
  static const uint8_t kSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1A, '\n'};
  if (f.size() < 8 || std::memcmp(f.data(), kSig, 8) != 0) throw Error(path + ": not a PNG file");
  uint32_t w = 0, h = 0;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<uint8_t> idat;
  for (size_t p = 8; p + 12 <= f.size();) {
    const uint32_t len = be32(&f[p]);
    if (p + 12 + len > f.size()) throw Error(path + ": truncated chunk");
    const std::string type(reinterpret_cast<const char*>(&f[p + 4]), 4);
    const uint8_t* d = &f[p + 8];
    if (type == "IHDR") {
      w = be32(d);
      h = be32(d + 4);
      depth = d[8];
      ctype = d[9];
      interlace = d[12];
    } else if (type == "IDAT") {
      idat.insert(idat.end(), d, d + len);
    } else if (type == "IEND") {
      break;
    }
    p += 12 + len;
  }
  const int ch = ctype == 0 ? 1 : ctype == 2 ? 3 : ctype == 4 ? 2 : ctype == 6 ? 4 : 0;
  if (depth != 8 || ch == 0 || interlace != 0)
    throw Error(path + ": unsupported PNG (8-bit grey/RGB(A), non-interlaced only)");
  if (w == 0 || h == 0 || w > 65535 || h > 65535) throw Error(path + ": bad PNG size");
  const size_t stride = static_cast<size_t>(w) * ch;
  std::vector<uint8_t> raw((stride + 1) * h);
  uLongf rawlen = static_cast<uLongf>(raw.size());
  if (uncompress(raw.data(), &rawlen, idat.data(), static_cast<uLong>(idat.size())) != Z_OK ||
      rawlen != raw.size())
    throw Error(path + ": corrupt PNG image data");
  std::vector<uint8_t> px(stride * h);
  for (uint32_t y = 0; y < h; ++y) {
    const uint8_t ft = raw[y * (stride + 1)];
    const uint8_t* src = &raw[y * (stride + 1) + 1];
    uint8_t* dst = &px[y * stride];
    const uint8_t* up = y ? &px[(y - 1) * stride] : nullptr;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= static_cast<size_t>(ch) ? dst[i - ch] : 0, b = up ? up[i] : 0,
                c = (up && i >= static_cast<size_t>(ch)) ? up[i - ch] : 0;
      int pred = 0;
      switch (ft) {
        case 0: pred = 0; break;
        case 1: pred = a; break;
        case 2: pred = b; break;
        case 3: pred = (a + b) / 2; break;
        case 4: pred = paeth(a, b, c); break;
        default: throw Error(path + ": bad PNG filter");
      }
      dst[i] = static_cast<uint8_t>(src[i] + pred);
    }
  }
  ColorImage img(static_cast<int>(w), static_cast<int>(h));
  for (size_t i = 0; i < static_cast<size_t>(w) * h; ++i) {
    const uint8_t* s = &px[i * ch];
    const bool grey = ch < 3;
    img.pixels[3 * i] = s[0];
    img.pixels[3 * i + 1] = grey ? s[0] : s[1];
    img.pixels[3 * i + 2] = grey ? s[0] : s[2];
  }
  return img;
}

void save_png(const std::string& path, const ColorImage& img) {
  const size_t stride = static_cast<size_t>(img.width) * 3;
  std::string raw;
  raw.reserve((stride + 1) * img.height);
  for (int y = 0; y < img.height; ++y) {
    raw.push_back(0);  // filter: none
    raw.append(reinterpret_cast<const char*>(&img.pixels[y * stride]), stride);
  }
  uLongf zlen = compressBound(static_cast<uLong>(raw.size()));
  std::string z(zlen, '\0');
  if (compress2(reinterpret_cast<Bytef*>(&z[0]), &zlen, reinterpret_cast<const Bytef*>(raw.data()),
                static_cast<uLong>(raw.size()), 6) != Z_OK)
    throw Error(path + ": PNG compression failed");
  z.resize(zlen);
  std::string out("\x89PNG\r\n\x1a\n", 8), ihdr;
  put_be32(ihdr, static_cast<uint32_t>(img.width));
  put_be32(ihdr, static_cast<uint32_t>(img.height));
  ihdr += std::string("\x08\x02\x00\x00\x00", 5);  // 8-bit RGB, deflate, no filter set, no interlace
  png_chunk(out, "IHDR", ihdr);
  png_chunk(out, "IDAT", z);
  png_chunk(out, "IEND", "");
  write_file(path, out);
}

std::pair<ColorImage, ColorImage> load_frame_pair(const std::string& dir, int index,
                                                  const StereoRig& rig) {
  char name[32];
  std::snprintf(name, sizeof(name), "%06d.png", index);
  const std::string lp = dir + "/left_" + name, rp = dir + "/right_" + name;
  ColorImage l = load_png(lp), r = load_png(rp);
  for (const auto* pr : {&lp, &rp}) {
    const ColorImage& im = pr == &lp ? l : r;
    if (im.width != rig.intrinsics.width || im.height != rig.intrinsics.height)
      throw Error(*pr + ": " + std::to_string(im.width) + "x" + std::to_string(im.height) +
                  " does not match the calibration's " + std::to_string(rig.intrinsics.width) +
                  "x" + std::to_string(rig.intrinsics.height));
  }
  return {std::move(l), std::move(r)};
}

void write_disparity_pgm16(const std::string& path, const DisparityMap& map) {
  std::string out = "P5\n" + std::to_string(map.width) + " " + std::to_string(map.height) +
                    "\n65535\n";
  const size_t n = static_cast<size_t>(map.width) * map.height;
  out.reserve(out.size() + 2 * n);
  for (size_t i = 0; i < n; ++i) {
    long q = 0;
    if (map.valid[i]) q = std::clamp<long>(std::lround(256.0 * map.disparity[i]), 0, 65535);
    out.push_back(static_cast<char>((q >> 8) & 0xFF));
    out.push_back(static_cast<char>(q & 0xFF));
  }
  write_file(path, out);
}

std::vector<uint16_t> read_pgm16(const std::string& path, int* width, int* height) {
  const std::vector<uint8_t> f = read_file(path);
  std::string head(f.begin(), f.begin() + std::min<size_t>(f.size(), 64));
  std::istringstream hs(head);
  std::string magic;
  int w = 0, h = 0, mx = 0;
  if (!(hs >> magic >> w >> h >> mx) || magic != "P5" || mx != 65535 || w < 0 || h < 0)
    throw Error(path + ": not a 16-bit binary PGM");
  const size_t off = static_cast<size_t>(hs.tellg()) + 1;
  const size_t n = static_cast<size_t>(w) * h;
  if (f.size() < off + 2 * n) throw Error(path + ": truncated PGM");
  std::vector<uint16_t> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = static_cast<uint16_t>((f[off + 2 * i] << 8) | f[off + 2 * i + 1]);
  *width = w;
  *height = h;
  return v;
}

void export_ply(const std::string& path, const StereoCloud& cloud) {
  const size_t n = cloud.points.size();
  std::string out = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) +
                    "\nproperty float x\nproperty float y\nproperty float z\n"
                    "property float nx\nproperty float ny\nproperty float nz\n"
                    "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n";
  const size_t head = out.size();
  out.resize(head + 27 * n);
  char* p = &out[head];
  for (size_t i = 0; i < n; ++i) {
    const float v[6] = {static_cast<float>(cloud.points[i].x()), static_cast<float>(cloud.points[i].y()),
                        static_cast<float>(cloud.points[i].z()), static_cast<float>(cloud.normals[i].x()),
                        static_cast<float>(cloud.normals[i].y()), static_cast<float>(cloud.normals[i].z())};
    std::memcpy(p, v, 24);  // little-endian host (x86-64 / aarch64)
    std::memcpy(p + 24, cloud.colors[i].data(), 3);
    p += 27;
  }
  write_file(path, out);
}

int run_stereo_only(const std::string& calibration, const std::string& dir, int index,
                    const StereoParams& params, const std::string& out_prefix) {
  const StereoRig rig = load_calibration(calibration);
  const auto [left, right] = load_frame_pair(dir, index, rig);
  const GrayImage gl = to_gray(left), gr = to_gray(right);
  DisparityMap m = compute_disparity(gl, gr, params);
  m = cleanup_pass(m, params);
  m = refine_disparities(m, gl, gr, params);
  const StereoCloud cloud = disparity_to_cloud(m, left, rig);
  export_ply(out_prefix + ".ply", cloud);
  write_disparity_pgm16(out_prefix + "_disparity.pgm", m);
  return static_cast<int>(cloud.points.size());
}

}  // namespace stereoscan::io
