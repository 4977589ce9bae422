// Status codes, thread-local error text and CUDA error plumbing shared by the
// runtime and the C ABI (include/tilerun_b200.h).
#pragma once

#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/tilerun_b200.h"

namespace tr {

// Exception carrying a tr_status; the C ABI catches it and returns the code.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(int status, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(status, buf);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) fail(TR_ERR_CUDA, "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
}

#define TR_CUDA(call) ::tr::cuda_check((call), #call, __FILE__, __LINE__)

void set_last_error(const char* msg);

// NVTX range on the calling thread (products, device jobs, tasks, fills): named
// host-side intervals for nsys / Nsight timelines; a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, long long a) {
    char buf[96];
    snprintf(buf, sizeof(buf), fmt, a);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace tr
