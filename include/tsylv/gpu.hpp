// tsylv drop-in (B200 build) — bridge from the header API to the C-ABI
// (include/tsylv_gpu.h): one lazily created context per host thread (the
// reference API is context-free and re-entrant), and the
// status-code -> exception mapping of the boundary contract.
#pragma once
#include <stdexcept>
#include <string>

#include "tsylv/errors.hpp"
#include "tsylv_gpu.h"

namespace tsylv::gpu {

struct ContextHolder {
  tsg_ctx* ctx = nullptr;
  ~ContextHolder() {
    if (ctx) tsg_destroy(ctx);
  }
};

inline tsg_ctx* context() {
  thread_local ContextHolder h;
  if (!h.ctx) {
    const int dev = 0;
    if (tsg_create(1, &dev, &h.ctx) != TSG_OK)
      throw std::runtime_error("tsylv: cannot create GPU context (no CUDA device?)");
  }
  return h.ctx;
}

// Status -> reference exception type (errors.hpp:13-62).
inline void check(int rc, const char* who) {
  if (rc == TSG_OK) return;
  std::string msg = std::string(who) + ": " + tsg_last_error(context());
  switch (rc) {
    case TSG_EDIM:
      throw dimension_error(msg);
    case TSG_ESINGULAR:
      throw singular_error(msg);
    case TSG_EFACT:
      throw factorization_error(msg);
    case TSG_EINVAL:
      throw std::invalid_argument(msg);
    default:
      throw std::runtime_error(msg);
  }
}

}  // namespace tsylv::gpu
