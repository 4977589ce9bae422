// Process-wide cache of large device allocations (tile slabs, staging buffers).
//
// A reference-style one-shot run() creates and destroys a session per product;
// freeing and re-allocating several GiB of HBM each time costs up to seconds
// (cudaFree of a multi-GiB range is slow and synchronising).  Sessions return
// their buffers here instead, and the next session on the same GPU reuses any
// cached block that is large enough (best fit).  tr_release_cached_memory()
// hands everything back to CUDA.
#pragma once

#include <cstddef>
#include <map>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

namespace tr {

class DevPool {
 public:
  static DevPool& get();
  // Allocates >= bytes on `gpu` (current device must be `gpu`); returns the
  // block's real capacity in *cap.
  cudaError_t alloc(int gpu, size_t bytes, void** out, size_t* cap);
  void release(int gpu, void* p, size_t cap);
  void trim();  // cudaFree every cached block
  size_t cached_bytes();
  // Free HBM on the current device `gpu` (cudaMemGetInfo), re-queried at most
  // once per `max_age_s`: the query occasionally stalls for tens of ms, which a
  // one-shot run() per product would otherwise pay on every call.
  cudaError_t free_bytes(int gpu, size_t* out, double max_age_s = 10.0);

 private:
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void*>> free_;  // gpu -> size -> ptr
  struct FreeInfo {
    size_t bytes = 0;
    double when = -1e30;
  };
  std::map<int, FreeInfo> free_info_;
};

}  // namespace tr
