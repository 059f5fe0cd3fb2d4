// In-process frame sharding across GPUs: one ss_ctx and one
// host worker thread per device entry. A batch of n pairs splits into
// contiguous frame blocks (sizes differ by at most one, the same partition as
// paper_2007_12623_b200/shard.py); every worker runs the pipelined host batch
// API on its block and writes its outputs straight into the caller's
// frame-ordered host arrays — the host-side gather of the per-frame clouds,
// with no collective and no copy between GPUs. Device entries may repeat (two
// contexts on one GPU), which is how the logic is tested on a one-GPU box.
#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ss_stereo.h"

struct ss_multi {
  std::vector<ss_ctx*> ctx;
  std::vector<int32_t> device;
};

namespace {

thread_local std::string tl_multi_err;

void frame_block(int32_t n, int32_t k, int32_t parts, int32_t* start, int32_t* count) {
  const int32_t base = n / parts, extra = n % parts;
  *start = k * base + std::min(k, extra);
  *count = base + (k < extra ? 1 : 0);
}

}  // namespace

extern "C" {

ss_status ss_multi_create(int32_t n_devices, const int32_t* devices, int32_t max_w, int32_t max_h,
                          int32_t max_batch, const ss_stereo_params* p, const ss_stereo_rig* rig,
                          ss_multi** out) {
  if (!out || n_devices <= 0 || !devices) return SS_EINVAL;
  *out = nullptr;
  auto m = std::make_unique<ss_multi>();
  for (int32_t k = 0; k < n_devices; ++k) {
    ss_ctx* c = nullptr;
    const ss_status st = ss_ctx_create(devices[k], max_w, max_h, max_batch, p, rig, &c);
    if (st != SS_OK) {
      for (ss_ctx* x : m->ctx) ss_ctx_destroy(x);
      return st;
    }
    m->ctx.push_back(c);
    m->device.push_back(devices[k]);
  }
  *out = m.release();
  return SS_OK;
}

ss_status ss_multi_destroy(ss_multi* m) {
  if (!m) return SS_OK;
  ss_status st = SS_OK;
  for (ss_ctx* c : m->ctx) {
    const ss_status s = ss_ctx_destroy(c);
    if (st == SS_OK) st = s;
  }
  delete m;
  return st;
}

int32_t ss_multi_size(const ss_multi* m) { return m ? static_cast<int32_t>(m->ctx.size()) : 0; }

ss_ctx* ss_multi_ctx(ss_multi* m, int32_t k) {
  return (m && k >= 0 && k < static_cast<int32_t>(m->ctx.size())) ? m->ctx[k] : nullptr;
}

ss_status ss_multi_set_lr_check(ss_multi* m, int32_t enable, int32_t max_diff) {
  if (!m) return SS_EINVAL;
  for (ss_ctx* c : m->ctx) {
    const ss_status st = ss_ctx_set_lr_check(c, enable, max_diff);
    if (st != SS_OK) return st;
  }
  return SS_OK;
}

ss_status ss_multi_stereo_batch(ss_multi* m, int32_t n, int32_t w, int32_t h, int32_t in_format,
                                const uint8_t* left, const uint8_t* right, uint32_t out_flags,
                                const ss_batch_out* out) {
  if (!m || !out || n < 0 || w <= 0 || h <= 0) return SS_EINVAL;
  const int32_t parts = static_cast<int32_t>(m->ctx.size());
  const long N = static_cast<long>(w) * h;
  const long in_bytes = (in_format == SS_IN_RGB ? 3 : 1) * N;
  std::vector<ss_status> status(parts, SS_OK);
  std::vector<std::string> msg(parts);
  auto work = [&](int32_t k) {
    int32_t f0 = 0, cnt = 0;
    frame_block(n, k, parts, &f0, &cnt);
    if (cnt == 0) return;
    ss_batch_out o{};
    o.disparity = out->disparity ? out->disparity + f0 * N : nullptr;
    o.valid = out->valid ? out->valid + f0 * N : nullptr;
    o.index = out->index ? out->index + f0 * N : nullptr;
    o.points = out->points ? out->points + f0 * N * 3 : nullptr;
    o.normals = out->normals ? out->normals + f0 * N * 3 : nullptr;
    o.colors = out->colors ? out->colors + f0 * N * 3 : nullptr;
    o.n_points = out->n_points ? out->n_points + f0 : nullptr;
    status[k] = ss_stereo_batch(m->ctx[k], cnt, w, h, in_format, left + f0 * in_bytes,
                                right + f0 * in_bytes, out_flags, &o);
    if (status[k] != SS_OK) msg[k] = ss_last_error();
  };
  std::vector<std::thread> th;
  for (int32_t k = 1; k < parts; ++k) th.emplace_back(work, k);
  work(0);  // the calling thread serves the first device
  for (auto& t : th) t.join();
  for (int32_t k = 0; k < parts; ++k)
    if (status[k] != SS_OK) {
      tl_multi_err = "device " + std::to_string(m->device[k]) + ": " + msg[k];
      return status[k];
    }
  return SS_OK;
}

const char* ss_multi_last_error(void) { return tl_multi_err.c_str(); }

}  // extern "C"
