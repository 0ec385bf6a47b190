// Per-thread device context for the C++ drop-in API. The reference estimator is stateless
// and safe for concurrent calls; each host thread gets its own rv_context
// (stream + buffers) on device ROTAVOTE_DEVICE (default 0). There is no CPU fallback: without
// a CUDA device every device-backed call throws rotavote::DeviceError.
#pragma once

#include <cstdlib>
#include <memory>
#include <string>

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

inline void check(rv_status st) {
  if (st != RV_OK) throw_status(st, std::string(rv_status_string(st)) + ": " + rv_context_last_error(context()));
}

}  // namespace detail
}  // namespace rotavote
