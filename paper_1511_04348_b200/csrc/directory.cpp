// Tile-cache directory; see directory.h.  Each method cites the reference
// behaviour it restates (coherence.py line numbers).
#include "directory.h"

#include "common.h"

namespace tr {

void add_stats(tr_cache_stats* into, const tr_cache_stats& s) {
  into->l1_hits += s.l1_hits;
  into->l2_hits += s.l2_hits;
  into->host_fetches += s.host_fetches;
  into->bytes_host += s.bytes_host;
  into->bytes_peer += s.bytes_peer;
  into->evictions += s.evictions;
  into->writebacks += s.writebacks;
  into->bytes_writeback += s.bytes_writeback;
}

tr_cache_stats sub_stats(const tr_cache_stats& a, const tr_cache_stats& b) {
  tr_cache_stats r;
  r.l1_hits = a.l1_hits - b.l1_hits;
  r.l2_hits = a.l2_hits - b.l2_hits;
  r.host_fetches = a.host_fetches - b.host_fetches;
  r.bytes_host = a.bytes_host - b.bytes_host;
  r.bytes_peer = a.bytes_peer - b.bytes_peer;
  r.evictions = a.evictions - b.evictions;
  r.writebacks = a.writebacks - b.writebacks;
  r.bytes_writeback = a.bytes_writeback - b.bytes_writeback;
  return r;
}

Directory::Directory(int n_devices, const std::vector<int64_t>& capacity, const std::vector<bool>& host_worker,
                     const std::vector<int64_t>& hops, bool enabled, int policy, bool debug)
    : n_(n_devices),
      capacity_(capacity),
      host_worker_(host_worker),
      hops_(hops),
      enabled_(enabled),
      policy_(policy),
      debug_(debug),
      dev_(n_devices),
      slot_total_(n_devices, 0) {
  if (n_devices < 1 || n_devices > 64) fail(TR_ERR_CONFIG, "directory supports 1..64 devices, got %d", n_devices);
  if (policy != TR_POLICY_LRU && policy != TR_POLICY_FIFO) fail(TR_ERR_VALUE, "unknown eviction policy %d", policy);
  if (static_cast<int>(capacity_.size()) != n_ || static_cast<int>(host_worker_.size()) != n_ ||
      static_cast<int64_t>(hops_.size()) != static_cast<int64_t>(n_) * n_)
    fail(TR_ERR_CONFIG, "directory: per-device arrays do not match n_devices");
}

// devices.py:285-291: fewest hops, ties to the lowest device id.
int Directory::closest_owner(int requester, uint64_t owners) const {
  int best = -1;
  int64_t best_h = 0;
  for (int o = 0; o < n_; ++o) {
    if (!(owners >> o & 1)) continue;
    const int64_t h = hops_[static_cast<int64_t>(requester) * n_ + o];
    if (best < 0 || h < best_h) {
      best = o;
      best_h = h;
    }
  }
  return best;
}

int32_t Directory::balanced_source_locked(int requester, const TileKey& key, const std::vector<int64_t>& load) const {
  auto it = residency_.find(key);
  const uint64_t owners = (it == residency_.end() ? 0 : it->second) & ~(1ull << requester);
  int best = -1;
  int64_t best_h = 0, best_l = 0;
  for (int o = 0; o < n_; ++o) {
    if (!(owners >> o & 1)) continue;
    const int64_t h = hops_[static_cast<int64_t>(requester) * n_ + o];
    const int64_t l = o < static_cast<int>(load.size()) ? load[o] : 0;
    if (best < 0 || h < best_h || (h == best_h && l < best_l)) {
      best = o;
      best_h = h;
      best_l = l;
    }
  }
  return best;
}

void Directory::attach_slots(int device, int32_t n_slots) {
  Dev& d = dev_[device];
  // stack: the lowest new index is handed out first
  for (int32_t s = n_slots - 1; s >= static_cast<int32_t>(slot_total_[device]); --s) d.free_slots.push_back(s);
  if (n_slots > slot_total_[device]) slot_total_[device] = n_slots;
}

int32_t Directory::slot_of_locked(int device, const TileKey& key) const {
  auto it = dev_[device].entries.find(key);
  return it == dev_[device].entries.end() ? -1 : it->second.slot;
}

uint64_t Directory::owners_locked(const TileKey& key) const {
  auto it = residency_.find(key);
  return it == residency_.end() ? 0 : it->second;
}

// coherence.py:118-134
HitLevel Directory::lookup_locked(int requester, const TileKey& key, int32_t* owner) {
  if (owner) *owner = -1;
  auto it = residency_.find(key);
  const uint64_t owners = it == residency_.end() ? 0 : it->second;
  if (owners >> requester & 1) {
    if (policy_ == TR_POLICY_LRU) {
      Dev& d = dev_[requester];
      Entry& e = d.entries.at(key);
      d.order.splice(d.order.end(), d.order, e.pos);
    }
    return HIT_L1;
  }
  if (owners) {
    if (owner) *owner = closest_owner(requester, owners);
    return HIT_L2;
  }
  return HIT_MISS;
}

void Directory::drop_locked(int device, const TileKey& key) {
  Dev& d = dev_[device];
  auto it = d.entries.find(key);
  if (it->second.slot >= 0) d.free_slots.push_back(it->second.slot);
  d.order.erase(it->second.pos);
  d.entries.erase(it);
  auto r = residency_.find(key);
  r->second &= ~(1ull << device);
  if (!r->second) residency_.erase(r);
}

// coherence.py:147-174
std::vector<TileKey> Directory::admit_locked(int device, const TileKey& key, bool input, int32_t* slot_out) {
  Dev& d = dev_[device];
  if (d.entries.count(key)) fail(TR_ERR_VALUE, "tile (%llu,%lld,%lld) already resident on device %d",
                                 (unsigned long long)key.matrix, (long long)key.row, (long long)key.col, device);
  std::vector<TileKey> evicted;
  const int64_t cap = capacity_[device];
  if (cap >= 0 && static_cast<int64_t>(d.order.size()) >= cap) {
    const int64_t need = static_cast<int64_t>(d.order.size()) + 1 - cap;
    std::vector<TileKey> victims;
    for (const TileKey& k : d.order) {
      if (static_cast<int64_t>(victims.size()) >= need) break;
      auto p = d.pins.find(k);
      if (p == d.pins.end() || p->second == 0) victims.push_back(k);
    }
    if (static_cast<int64_t>(victims.size()) < need)
      fail(TR_ERR_CAPACITY, "device %d: capacity %lld exhausted and all resident tiles pinned; working set does not fit",
           device, (long long)cap);
    for (const TileKey& v : victims) {
      drop_locked(device, v);
      evicted.push_back(v);
    }
    stats_.evictions += static_cast<int64_t>(victims.size());
    d.stats.evictions += static_cast<int64_t>(victims.size());
  }
  int32_t slot = -1;
  if (input && slot_total_[device] > 0) {
    if (d.free_slots.empty()) {
      // Physical pool smaller than the logical capacity (HBM budget): evict a
      // dead tile if the job's future is known, else the LRU unpinned one.
      TileKey victim{};
      const bool found = physical_victim_locked(device, &victim, false);
      if (!found)
        fail(TR_ERR_CAPACITY, "device %d: HBM slab exhausted (%lld slots, %zu resident) and all resident tiles pinned",
             device, (long long)slot_total_[device], d.order.size());
      drop_locked(device, victim);
      evicted.push_back(victim);
      stats_.evictions += 1;
      d.stats.evictions += 1;
    }
    slot = d.free_slots.back();
    d.free_slots.pop_back();
  }
  d.order.push_back(key);
  d.entries[key] = Entry{std::prev(d.order.end()), slot, 0};
  residency_[key] |= 1ull << device;
  if (slot_out) *slot_out = slot;
  if (debug_) check_invariants_locked();
  return evicted;
}

void Directory::unpin_locked(int device, const TileKey& key) {
  auto& pins = dev_[device].pins;
  auto it = pins.find(key);
  if (it == pins.end() || it->second < 1)
    fail(TR_ERR_VALUE, "unpin below zero for tile (%llu,%lld,%lld) on device %d", (unsigned long long)key.matrix,
         (long long)key.row, (long long)key.col, device);
  if (--it->second == 0) pins.erase(it);
}

// coherence.py:210-246
Acquired Directory::acquire_input_locked(int requester, const TileKey& key, int64_t nbytes) {
  Dev& d = dev_[requester];
  tr_cache_stats& ds = d.stats;
  Acquired r{HIT_MISS, TR_SOURCE_HOST, 0, -1, {}};
  if (host_worker_[requester]) {
    stats_.host_fetches += 1;
    ds.host_fetches += 1;
    return r;
  }
  if (!enabled_) {
    stats_.host_fetches += 1;
    ds.host_fetches += 1;
    stats_.bytes_host += nbytes;
    ds.bytes_host += nbytes;
    r.nbytes = nbytes;
    return r;
  }
  if (future_on_) {
    auto f = future_.find(key);
    if (f != future_.end()) f->second -= 1;
  }
  // Classification (coherence.py:124-134) over COUNTED owners: a tile some device
  // holds only as an unclaimed fetch-ahead is, for the counters, not resident yet
  // -- exactly as in a run without fetch-ahead.
  auto it = residency_.find(key);
  const uint64_t owners = it == residency_.end() ? 0 : it->second;
  uint64_t counted = 0;
  for (int o = 0; o < n_; ++o)
    if ((owners >> o & 1) && !dev_[o].entries.at(key).pending) counted |= 1ull << o;
  const uint64_t others = counted & ~(1ull << requester);
  if (owners >> requester & 1) {
    Entry& e = d.entries.at(key);
    if (policy_ == TR_POLICY_LRU) d.order.splice(d.order.end(), d.order, e.pos);
    d.pins[key] += 1;
    r.slot = e.slot;
    if (!e.pending) {
      stats_.l1_hits += 1;
      ds.l1_hits += 1;
      r.level = HIT_L1;
      r.source = requester;
      return r;
    }
    // first request of a fetched-ahead tile: count it as the request would have
    // been counted without the fetch-ahead (peer copy if a counted owner exists)
    r.prefetched = true;
    r.nbytes = nbytes;
    e.pending = 0;
    if (others) {
      stats_.l2_hits += 1;
      ds.l2_hits += 1;
      stats_.bytes_peer += nbytes;
      ds.bytes_peer += nbytes;
      r.level = HIT_L2;
      r.source = closest_owner(requester, others);
    } else {
      stats_.host_fetches += 1;
      ds.host_fetches += 1;
      stats_.bytes_host += nbytes;
      ds.bytes_host += nbytes;
      r.level = HIT_MISS;
    }
    return r;
  }
  if (others) {
    // counters before admit, as coherence.py:233-237 does
    stats_.l2_hits += 1;
    ds.l2_hits += 1;
    stats_.bytes_peer += nbytes;
    ds.bytes_peer += nbytes;
    r.evicted = admit_locked(requester, key, true, &r.slot);
    d.pins[key] += 1;
    r.level = HIT_L2;
    r.source = closest_owner(requester, others);
    r.phys_source = r.source;
    r.nbytes = nbytes;
    return r;
  }
  stats_.host_fetches += 1;
  ds.host_fetches += 1;
  stats_.bytes_host += nbytes;
  ds.bytes_host += nbytes;
  r.evicted = admit_locked(requester, key, true, &r.slot);
  d.pins[key] += 1;
  r.nbytes = nbytes;
  // counted as a host fetch; physically, another device's in-flight fetch-ahead
  // copy (if any) is closer than the host
  const uint64_t pend = owners & ~(1ull << requester);
  if (pend) r.phys_source = closest_owner(requester, pend);
  return r;
}

bool Directory::physical_victim_locked(int device, TileKey* victim, bool dead_only) const {
  const Dev& d = dev_[device];
  const TileKey* lru = nullptr;
  for (const TileKey& k : d.order) {
    auto e = d.entries.find(k);
    if (e->second.slot < 0) continue;
    auto p = d.pins.find(k);
    if (p != d.pins.end() && p->second > 0) continue;
    if (!future_on_ || dead_locked(k)) {
      *victim = k;
      return true;
    }
    if (!lru && !e->second.pending) lru = &k;  // live: only if nothing is dead
  }
  if (dead_only || !lru) return false;
  *victim = *lru;
  return true;
}

bool Directory::dead_locked(const TileKey& key) const {
  auto it = future_.find(key);
  return it != future_.end() && it->second <= 0;
}

void Directory::set_future_locked(std::unordered_map<TileKey, int64_t, TileKeyHash> future) {
  future_ = std::move(future);
  future_on_ = true;
}

void Directory::clear_future_locked() {
  future_.clear();
  future_on_ = false;
}

bool Directory::prefetch_locked(int device, const TileKey& key, int32_t* slot, int32_t* phys_source, bool host_only) {
  if (!enabled_ || host_worker_[device]) return false;
  Dev& d = dev_[device];
  if (d.entries.count(key)) return false;
  if (capacity_[device] >= 0 && static_cast<int64_t>(d.order.size()) >= capacity_[device]) return false;
  if (slot_total_[device] > 0 && d.free_slots.empty()) {
    // out-of-core: a dead tile's slot may take the prefetch (never a live one)
    TileKey victim{};
    if (!future_on_ || !physical_victim_locked(device, &victim, true)) return false;
    drop_locked(device, victim);
    stats_.evictions += 1;
    d.stats.evictions += 1;
  }
  auto it = residency_.find(key);
  const uint64_t owners = it == residency_.end() ? 0 : it->second;
  if (host_only && owners) return false;
  *phys_source = owners ? closest_owner(device, owners) : TR_SOURCE_HOST;
  admit_locked(device, key, true, slot);  // cannot evict: checked above
  d.entries.at(key).pending = 1;
  return true;
}

// coherence.py:248-252
void Directory::release_input_locked(int device, const TileKey& key) {
  if (!enabled_ || host_worker_[device]) return;
  unpin_locked(device, key);
}

// coherence.py:254-261
std::vector<TileKey> Directory::admit_output_locked(int device, const TileKey& key) {
  if (!enabled_ || host_worker_[device]) return {};
  auto ev = admit_locked(device, key, false, nullptr);
  dev_[device].pins[key] += 1;
  return ev;
}

// coherence.py:263-280
void Directory::release_output_locked(int device, const TileKey& key, int64_t nbytes) {
  if (!enabled_ || host_worker_[device]) return;
  unpin_locked(device, key);
  if (!dev_[device].entries.count(key))  // the reference raises KeyError here (after the unpin)
    fail(TR_ERR_VALUE, "tile (%llu,%lld,%lld) is not resident on device %d", (unsigned long long)key.matrix,
         (long long)key.row, (long long)key.col, device);
  drop_locked(device, key);
  stats_.writebacks += 1;
  stats_.bytes_writeback += nbytes;
  dev_[device].stats.writebacks += 1;
  dev_[device].stats.bytes_writeback += nbytes;
  if (debug_) check_invariants_locked();
}

int64_t Directory::forget_locked(uint64_t uid) {
  int64_t n = 0;
  for (int d = 0; d < n_; ++d) {
    Dev& dv = dev_[d];
    std::vector<TileKey> dead;
    for (const auto& e : dv.entries) {
      if (e.first.matrix != uid) continue;
      auto p = dv.pins.find(e.first);
      if (p == dv.pins.end() || p->second == 0) dead.push_back(e.first);
    }
    for (const TileKey& k : dead) drop_locked(d, k);
    n += static_cast<int64_t>(dead.size());
  }
  if (debug_) check_invariants_locked();
  return n;
}

// coherence.py:300-313
void Directory::check_invariants_locked() {
  std::vector<int64_t> per_dev(n_, 0);
  for (const auto& kv : residency_) {
    if (!kv.second) fail(TR_ERR_INTERNAL, "invariant: tile has an empty owner set");
    for (int d = 0; d < n_; ++d) {
      if (!(kv.second >> d & 1)) continue;
      per_dev[d] += 1;
      if (!dev_[d].entries.count(kv.first)) fail(TR_ERR_INTERNAL, "invariant: tile in residency but not in order[%d]", d);
    }
  }
  for (int d = 0; d < n_; ++d) {
    const Dev& dv = dev_[d];
    if (static_cast<int64_t>(dv.order.size()) != per_dev[d] || dv.order.size() != dv.entries.size())
      fail(TR_ERR_INTERNAL, "invariant: order/residency disagree on device %d", d);
    if (capacity_[d] >= 0 && static_cast<int64_t>(dv.order.size()) > capacity_[d])
      fail(TR_ERR_INTERNAL, "invariant: device %d over capacity", d);
    for (const auto& p : dv.pins) {
      if (p.second <= 0) fail(TR_ERR_INTERNAL, "invariant: non-positive pin count on device %d", d);
      if (!dv.entries.count(p.first)) fail(TR_ERR_INTERNAL, "invariant: pinned tile not resident on device %d", d);
    }
    if (slot_total_[d] > 0) {
      std::vector<char> used(static_cast<size_t>(slot_total_[d]), 0);
      for (const auto& e : dv.entries) {
        if (e.second.slot < 0) continue;
        if (used[e.second.slot]) fail(TR_ERR_INTERNAL, "invariant: slot %d bound twice on device %d", e.second.slot, d);
        used[e.second.slot] = 1;
      }
      for (int32_t s : dv.free_slots) {
        if (used[s]) fail(TR_ERR_INTERNAL, "invariant: slot %d both free and bound on device %d", s, d);
        used[s] = 1;
      }
    }
  }
}

// ---- self-locking wrappers
HitLevel Directory::lookup(int requester, const TileKey& key, int32_t* owner) {
  DirLock g(mu);
  return lookup_locked(requester, key, owner);
}
std::vector<TileKey> Directory::admit(int device, const TileKey& key) {
  DirLock g(mu);
  return admit_locked(device, key, false, nullptr);
}
void Directory::pin(int device, const TileKey& key) {
  DirLock g(mu);
  if (!dev_[device].entries.count(key))
    fail(TR_ERR_VALUE, "cannot pin tile (%llu,%lld,%lld): not resident on device %d", (unsigned long long)key.matrix,
         (long long)key.row, (long long)key.col, device);
  dev_[device].pins[key] += 1;
}
void Directory::unpin(int device, const TileKey& key) {
  DirLock g(mu);
  unpin_locked(device, key);
}
bool Directory::is_pinned(int device, const TileKey& key) {
  DirLock g(mu);
  auto it = dev_[device].pins.find(key);
  return it != dev_[device].pins.end() && it->second > 0;
}
std::vector<TileKey> Directory::residents(int device) {
  DirLock g(mu);
  return std::vector<TileKey>(dev_[device].order.begin(), dev_[device].order.end());
}
int64_t Directory::used_tiles(int device) {
  DirLock g(mu);
  return static_cast<int64_t>(dev_[device].order.size());
}
Acquired Directory::acquire_input(int requester, const TileKey& key, int64_t nbytes) {
  DirLock g(mu);
  return acquire_input_locked(requester, key, nbytes);
}
void Directory::release_input(int device, const TileKey& key) {
  DirLock g(mu);
  release_input_locked(device, key);
}
std::vector<TileKey> Directory::admit_output(int device, const TileKey& key) {
  DirLock g(mu);
  return admit_output_locked(device, key);
}
void Directory::release_output(int device, const TileKey& key, int64_t nbytes) {
  DirLock g(mu);
  release_output_locked(device, key, nbytes);
}
tr_cache_stats Directory::stats() {
  DirLock g(mu);
  return stats_;
}
std::vector<tr_cache_stats> Directory::stats_per_device() {
  DirLock g(mu);
  std::vector<tr_cache_stats> out;
  for (const Dev& d : dev_) out.push_back(d.stats);
  return out;
}
void Directory::check_invariants() {
  DirLock g(mu);
  check_invariants_locked();
}

}  // namespace tr
