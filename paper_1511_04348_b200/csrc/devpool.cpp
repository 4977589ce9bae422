#include "devpool.h"

#include <chrono>

namespace tr {

DevPool& DevPool::get() {
  static DevPool* p = new DevPool();  // intentionally leaked: outlives static destructors
  return *p;
}

cudaError_t DevPool::alloc(int gpu, size_t bytes, void** out, size_t* cap) {
  {
    std::lock_guard<std::mutex> g(mu_);
    auto& m = free_[gpu];
    auto it = m.lower_bound(bytes);
    // reuse a block that is large enough but not wastefully so (<= 2x)
    if (it != m.end() && it->first <= 2 * bytes + (64u << 20)) {
      *out = it->second;
      *cap = it->first;
      m.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(out, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    trim();  // give cached blocks back and retry once
    e = cudaMalloc(out, bytes);
  }
  if (e == cudaSuccess) {
    *cap = bytes;
    std::lock_guard<std::mutex> g(mu_);
    auto it = free_info_.find(gpu);
    if (it != free_info_.end()) it->second.bytes -= std::min(it->second.bytes, bytes);  // keep the cached view honest
  }
  return e;
}

cudaError_t DevPool::free_bytes(int gpu, size_t* out, double max_age_s) {
  const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  {
    std::lock_guard<std::mutex> g(mu_);
    auto it = free_info_.find(gpu);
    if (it != free_info_.end() && now - it->second.when < max_age_s) {
      *out = it->second.bytes;
      return cudaSuccess;
    }
  }
  size_t f = 0, t = 0;
  cudaError_t e = cudaMemGetInfo(&f, &t);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu_);
  free_info_[gpu] = FreeInfo{f, now};
  *out = f;
  return cudaSuccess;
}

void DevPool::release(int gpu, void* p, size_t cap) {
  if (!p) return;
  std::lock_guard<std::mutex> g(mu_);
  free_[gpu].emplace(cap, p);
}

void DevPool::trim() {
  std::lock_guard<std::mutex> g(mu_);
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& kv : free_) {
    cudaSetDevice(kv.first);
    for (auto& b : kv.second) cudaFree(b.second);
    kv.second.clear();
  }
  free_info_.clear();  // free memory changed: re-query next time
  if (prev >= 0) cudaSetDevice(prev);
}

size_t DevPool::cached_bytes() {
  std::lock_guard<std::mutex> g(mu_);
  size_t s = 0;
  for (auto& kv : free_)
    for (auto& b : kv.second) s += b.first;
  return s;
}

}  // namespace tr
