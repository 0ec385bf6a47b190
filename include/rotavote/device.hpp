// Per-thread device context for the C++ drop-in API. The reference estimator is stateless
// and safe for concurrent calls; each host thread gets its own rv_context
// (stream + buffers) on device ROTAVOTE_DEVICE (default 0). There is no CPU fallback: without
// a CUDA device every device-backed call throws rotavote::DeviceError.
#pragma once

#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "../rotavote_b200.h"
#include "errors.hpp"

namespace rotavote {
namespace detail {

struct ContextDeleter {
  void operator()(rv_context* c) const { rv_context_destroy(c); }
};

inline rv_context* context() {
  thread_local std::unique_ptr<rv_context, ContextDeleter> ctx;
  if (!ctx) {
    const char* env = std::getenv("ROTAVOTE_DEVICE");
    rv_context* c = nullptr;
    const rv_status st = rv_context_create(env ? std::atoi(env) : 0, &c);
    if (st != RV_OK) throw_status(st, std::string("rotavote device context: ") + rv_status_string(st));
    ctx.reset(c);
  }
  return ctx.get();
}

// Multi-GPU: ROTAVOTE_DEVICES="0,1,2,3" (a list of device ids) routes
// estimate_single and accumulate through one rv_multi per host thread -- contiguous shards, one
// per device, u32 grids summed by an NCCL all-reduce, the sharded finish; results are identical to
// the single-device path (a one-id list runs the same sharded code on one device). Unset: the
// per-thread single-device context above.
struct MultiDeleter {
  void operator()(rv_multi* m) const { rv_multi_destroy(m); }
};

inline rv_multi* multi() {
  thread_local std::unique_ptr<rv_multi, MultiDeleter> m;
  thread_local bool probed = false;
  if (!probed) {
    probed = true;
    const char* env = std::getenv("ROTAVOTE_DEVICES");
    std::vector<int32_t> devs;
    for (const char* p = env; p && *p;) {
      char* end = nullptr;
      const long v = std::strtol(p, &end, 10);
      if (end == p) break;
      devs.push_back(static_cast<int32_t>(v));
      p = *end == ',' ? end + 1 : end;
    }
    if (!devs.empty()) {
      rv_multi* h = nullptr;
      const rv_status st = rv_multi_create(devs.data(), static_cast<int32_t>(devs.size()), &h);
      if (st != RV_OK) throw_status(st, std::string("rotavote multi-GPU context: ") + rv_status_string(st));
      m.reset(h);
    }
  }
  return m.get();
}

inline void check_multi(rv_status st) {
  if (st != RV_OK) throw_status(st, std::string(rv_status_string(st)) + ": " + rv_multi_last_error(multi()));
}

inline void check(rv_status st) {
  if (st != RV_OK) throw_status(st, std::string(rv_status_string(st)) + ": " + rv_context_last_error(context()));
}

}  // namespace detail
}  // namespace rotavote
