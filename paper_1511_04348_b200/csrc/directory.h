// The two-level tile-cache directory (L1 = own HBM, L2 = a peer's HBM, else host).
//
// Semantics follow the reference CacheDirectory exactly (coherence.py:86-313):
// one residency map key -> owner set, a per-device LRU (or FIFO) order, per-device
// pin counts, eviction of the oldest UNPINNED tiles only, CapacityError leaving the
// directory unchanged, exact hit/byte counters, and one lock that makes every
// composite operation (acquire_input = lookup + accounting + admit + pin)
// linearizable (coherence.py:202-209).
//
// The B200 build adds one thing the reference does not need: every resident
// INPUT tile is bound to a physical slot of the device's HBM slab.  Slots are
// handed out on admission and returned on eviction, so slot reuse is decided by
// the same LRU/pin rules the counters follow.
#pragma once

#include <chrono>
#include <cstdint>
#include <list>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/tilerun_b200.h"

namespace tr {

// The directory lock, instrumented: total time held, time callers waited for it,
// acquisitions and the longest hold (tr_session_lock_stats).  Two steady_clock
// reads per acquisition.
class DirMutex {
 public:
  void lock() {
    const auto t0 = std::chrono::steady_clock::now();
    m_.lock();
    t_lock_ = std::chrono::steady_clock::now();
    wait_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(t_lock_ - t0).count();
    count_ += 1;
  }
  void unlock() {
    const int64_t held =
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_lock_).count();
    hold_ns_ += held;
    if (held > max_hold_ns_) max_hold_ns_ = held;
    m_.unlock();
  }
  // snapshot / reset (caller does not hold the lock)
  void stats(int64_t* hold_ns, int64_t* wait_ns, int64_t* count, int64_t* max_hold_ns) {
    std::lock_guard<std::mutex> g(m_);
    *hold_ns = hold_ns_;
    *wait_ns = wait_ns_;
    *count = count_;
    *max_hold_ns = max_hold_ns_;
  }
  void reset() {
    std::lock_guard<std::mutex> g(m_);
    hold_ns_ = wait_ns_ = count_ = max_hold_ns_ = 0;
  }

 private:
  std::mutex m_;
  std::chrono::steady_clock::time_point t_lock_;
  int64_t hold_ns_ = 0, wait_ns_ = 0, count_ = 0, max_hold_ns_ = 0;  // written under m_
};
using DirLock = std::lock_guard<DirMutex>;

struct TileKey {
  uint64_t matrix;
  int64_t row, col;
  bool operator==(const TileKey& o) const { return matrix == o.matrix && row == o.row && col == o.col; }
};

struct TileKeyHash {
  size_t operator()(const TileKey& k) const {
    uint64_t h = k.matrix * 0x9E3779B97F4A7C15ull;
    h ^= static_cast<uint64_t>(k.row) + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2);
    h ^= static_cast<uint64_t>(k.col) + 0x85EBCA77C2B2AE63ull + (h << 6) + (h >> 2);
    return static_cast<size_t>(h);
  }
};

enum HitLevel : int32_t { HIT_L1 = TR_HIT_L1, HIT_L2 = TR_HIT_L2, HIT_MISS = TR_HIT_MISS };

struct Acquired {
  HitLevel level;
  int32_t source;  // device id the bytes came from, or TR_SOURCE_HOST
  int64_t nbytes;
  int32_t slot;    // physical slot on the requester (-1: none / bypass)
  std::vector<TileKey> evicted;
  bool prefetched = false;  // counted as `level` but already resident (filled ahead of the request)
  // Physical source of the bytes when the requester is not resident: a device id
  // (peer copy) or TR_SOURCE_HOST.  Differs from `source` only when the tile is
  // counted as a host fetch but another device already holds a fetch-ahead copy.
  int32_t phys_source = TR_SOURCE_HOST;
};

class Directory {
 public:
  Directory(int n_devices, const std::vector<int64_t>& capacity, const std::vector<bool>& host_worker,
            const std::vector<int64_t>& hops, bool enabled, int policy, bool debug);

  int n_devices() const { return n_; }
  bool enabled() const { return enabled_; }

  // ---- public, self-locking API (mirrors coherence.py method by method)
  HitLevel lookup(int requester, const TileKey& key, int32_t* owner);
  std::vector<TileKey> admit(int device, const TileKey& key);
  void pin(int device, const TileKey& key);
  void unpin(int device, const TileKey& key);
  bool is_pinned(int device, const TileKey& key);
  std::vector<TileKey> residents(int device);
  int64_t used_tiles(int device);
  Acquired acquire_input(int requester, const TileKey& key, int64_t nbytes);
  void release_input(int device, const TileKey& key);
  std::vector<TileKey> admit_output(int device, const TileKey& key);
  void release_output(int device, const TileKey& key, int64_t nbytes);
  tr_cache_stats stats();
  std::vector<tr_cache_stats> stats_per_device();
  void check_invariants();

  // ---- for the session: caller holds `mu`
  DirMutex mu;
  HitLevel lookup_locked(int requester, const TileKey& key, int32_t* owner);
  std::vector<TileKey> admit_locked(int device, const TileKey& key, bool input, int32_t* slot_out);
  Acquired acquire_input_locked(int requester, const TileKey& key, int64_t nbytes);
  void release_input_locked(int device, const TileKey& key);
  std::vector<TileKey> admit_output_locked(int device, const TileKey& key);
  // Fetch-ahead: make `key` resident on `device` before any task requests it,
  // WITHOUT counting anything and without evicting (returns false when the tile
  // is already resident, the device is full, or coherence is off).  The first
  // acquire_input of the tile on `device` is then counted exactly as it would
  // have been without the prefetch (host fetch, or L2 hit), so every counter
  // keeps the reference's meaning: requests classify against COUNTED owners
  // only.  *phys_source says where to copy from (a device id or host).
  bool prefetch_locked(int device, const TileKey& key, int32_t* slot, int32_t* phys_source, bool host_only = false);
  void release_output_locked(int device, const TileKey& key, int64_t nbytes);
  // Drop every unpinned resident tile of matrix `uid` on every device (the
  // content is dead, e.g. a retired weight version).  Not an eviction; no
  // counters change.  Returns the number of tiles dropped.
  int64_t forget_locked(uint64_t uid);
  void check_invariants_locked();
  // Out-of-core support (HBM slab smaller than the working set, logical capacity
  // unbounded): the remaining requests of every input tile in the current job.
  // While set, a physically full device evicts a DEAD tile (no remaining
  // request) before any live one, and fetch-ahead may replace dead tiles.
  // Logical (capacity_tiles) evictions keep the reference's LRU/FIFO order.
  void set_future_locked(std::unordered_map<TileKey, int64_t, TileKeyHash> future);
  void clear_future_locked();
  int32_t slot_of_locked(int device, const TileKey& key) const;
  // Physical source of an L2 fill of `key` into `requester` on a uniform
  // (NVSwitch) fabric: among the other owners with the fewest hops, the one
  // with the least `load` (copies it has served in this job), ties to the lowest
  // id.  The reference's closest_owner (devices.py:285-291) sends every fill to
  // the lowest-id owner; counters do not depend on the choice.  -1: no owner.
  int32_t balanced_source_locked(int requester, const TileKey& key, const std::vector<int64_t>& load) const;
  // Owners of `key` (bitmask over device ids).
  uint64_t owners_locked(const TileKey& key) const;
  // Bind device `d` to `n_slots` physical slots [0, n_slots).  May be called again to grow.
  void attach_slots(int device, int32_t n_slots);
  int32_t attached_slots(int device) const { return static_cast<int32_t>(slot_total_[device]); }
  int64_t capacity(int device) const { return capacity_[device]; }

 private:
  struct Entry {
    std::list<TileKey>::iterator pos;
    int32_t slot;
    int8_t pending = 0;  // 1: fetched ahead, not yet requested on this device (uncounted)
  };
  struct Dev {
    std::list<TileKey> order;  // LRU order, most recent at the back
    std::unordered_map<TileKey, Entry, TileKeyHash> entries;
    std::unordered_map<TileKey, int64_t, TileKeyHash> pins;
    std::vector<int32_t> free_slots;
    tr_cache_stats stats{};
  };

  int closest_owner(int requester, uint64_t owners) const;
  bool dead_locked(const TileKey& key) const;  // no remaining request in the current job
  bool physical_victim_locked(int device, TileKey* victim, bool dead_only) const;
  void unpin_locked(int device, const TileKey& key);
  void drop_locked(int device, const TileKey& key);  // remove residency (no counters)

  int n_;
  std::vector<int64_t> capacity_;  // -1 = unbounded
  std::vector<bool> host_worker_;
  std::vector<int64_t> hops_;
  bool enabled_;
  int policy_;  // TR_POLICY_LRU / TR_POLICY_FIFO
  bool debug_;
  std::vector<Dev> dev_;
  std::vector<int64_t> slot_total_;
  std::unordered_map<TileKey, uint64_t, TileKeyHash> residency_;
  std::unordered_map<TileKey, int64_t, TileKeyHash> future_;
  bool future_on_ = false;
  tr_cache_stats stats_{};
};

void add_stats(tr_cache_stats* into, const tr_cache_stats& s);
tr_cache_stats sub_stats(const tr_cache_stats& a, const tr_cache_stats& b);

}  // namespace tr
