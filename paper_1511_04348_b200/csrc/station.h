// Reservation stations and work stealing (scheduler.py:200-249).
//
// A station holds the task ids a device has reserved.  The owner serves them
// FIFO from the front, a thief removes from the back, and one lock makes every
// operation atomic so each task is obtained by exactly one party
// (scheduler.py:200-236).  In a GPU session each station entry is backed by a
// CUDA stream: the device thread moves ids from here onto idle streams.
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <mutex>
#include <utility>
#include <vector>

#include "msqueue.h"

namespace tr {

class Station {
 public:
  Station(int owner, int width) : owner_(owner), width_(width) {}
  int owner() const { return owner_; }
  int width() const { return width_; }

  // scheduler.py:214-224 — pull from the global queue until `limit` ids are reserved.
  std::vector<uint64_t> refill(MSQueue& q, int limit) {
    std::vector<uint64_t> pulled;
    std::lock_guard<std::mutex> g(mu_);
    while (static_cast<int>(slots_.size()) < limit) {
      uint64_t v;
      if (!q.dequeue(&v)) break;
      slots_.push_back(v);
      pulled.push_back(v);
    }
    return pulled;
  }
  // scheduler.py:226-228
  bool pop_for_run(uint64_t* tid) {
    std::lock_guard<std::mutex> g(mu_);
    if (slots_.empty()) return false;
    *tid = slots_.front();
    slots_.pop_front();
    return true;
  }
  // Priority pop (B200 addition): the reserved id with the highest score,
  // ties to the front (FIFO); with a constant score this is pop_for_run.
  template <typename Score>
  bool pop_best(uint64_t* tid, Score score) {
    std::lock_guard<std::mutex> g(mu_);
    if (slots_.empty()) return false;
    size_t best = 0;
    int best_score = score(slots_[0]);
    for (size_t i = 1; i < slots_.size(); ++i) {
      const int sc = score(slots_[i]);
      if (sc > best_score) {
        best = i;
        best_score = sc;
      }
    }
    *tid = slots_[best];
    slots_.erase(slots_.begin() + static_cast<std::ptrdiff_t>(best));
    return true;
  }
  // scheduler.py:230-232
  bool try_steal(uint64_t* tid) {
    std::lock_guard<std::mutex> g(mu_);
    if (slots_.empty()) return false;
    *tid = slots_.back();
    slots_.pop_back();
    return true;
  }
  // The id the owner would pop next, without popping it.
  bool peek_front(uint64_t* tid) {
    std::lock_guard<std::mutex> g(mu_);
    if (slots_.empty()) return false;
    *tid = slots_.front();
    return true;
  }
  int reserved_count() {
    std::lock_guard<std::mutex> g(mu_);
    return static_cast<int>(slots_.size());
  }
  // Snapshot of the reserved ids, front first (for fetch-ahead).
  std::vector<uint64_t> peek() {
    std::lock_guard<std::mutex> g(mu_);
    return std::vector<uint64_t>(slots_.begin(), slots_.end());
  }
  void clear() {
    std::lock_guard<std::mutex> g(mu_);
    slots_.clear();
  }

 private:
  int owner_, width_;
  std::mutex mu_;
  std::deque<uint64_t> slots_;
};

// scheduler.py:239-249 — victim is the most-loaded station, ties to the lowest id.
inline bool steal_task(int thief, Station* const* stations, int n, uint64_t* tid, int* victim) {
  std::vector<std::pair<int, int>> counts;  // (-count, id)
  for (int d = 0; d < n; ++d)
    if (stations[d]->owner() != thief) counts.emplace_back(-stations[d]->reserved_count(), stations[d]->owner());
  std::sort(counts.begin(), counts.end());
  for (const auto& cv : counts) {
    if (cv.first == 0) break;
    for (int d = 0; d < n; ++d) {
      if (stations[d]->owner() != cv.second) continue;
      if (stations[d]->try_steal(tid)) {
        *victim = cv.second;
        return true;
      }
    }
  }
  return false;
}

}  // namespace tr
