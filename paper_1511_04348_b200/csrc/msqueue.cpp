// Lock-free Michael-Scott queue; see msqueue.h.
#include "msqueue.h"

#include <new>

namespace tr {

MSQueue::MSQueue() {
  chunks_ = new std::atomic<Node*>[kMaxChunks];
  for (int i = 0; i < kMaxChunks; ++i) chunks_[i].store(nullptr, std::memory_order_relaxed);
  free_head_.store(pack(NIL, 0));
  const uint32_t dummy = alloc_node();
  node(dummy).next.store(pack(NIL, 0));
  head_.store(pack(dummy, 0));
  tail_.store(pack(dummy, 0));
}

MSQueue::~MSQueue() {
  for (int i = 0; i < kMaxChunks; ++i) delete[] chunks_[i].load();
  delete[] chunks_;
}

uint32_t MSQueue::alloc_node() {
  // Reuse a retired node first (tagged Treiber pop).
  uint64_t h = free_head_.load(std::memory_order_acquire);
  while (idx_of(h) != NIL) {
    const uint32_t nxt = node(idx_of(h)).free_next.load(std::memory_order_relaxed);
    if (free_head_.compare_exchange_weak(h, pack(nxt, tag_of(h) + 1), std::memory_order_acq_rel,
                                         std::memory_order_acquire))
      return idx_of(h);
  }
  const uint32_t i = n_fresh_.fetch_add(1, std::memory_order_relaxed);
  const uint32_t c = i >> kChunkBits;
  if (c >= static_cast<uint32_t>(kMaxChunks)) throw std::bad_alloc();
  if (chunks_[c].load(std::memory_order_acquire) == nullptr) {
    std::lock_guard<std::mutex> g(grow_mu_);
    if (chunks_[c].load(std::memory_order_relaxed) == nullptr) {
      Node* fresh = new Node[kChunk];
      for (uint32_t k = 0; k < kChunk; ++k) {
        fresh[k].next.store(pack(NIL, 0), std::memory_order_relaxed);
        fresh[k].value.store(0, std::memory_order_relaxed);
        fresh[k].free_next.store(NIL, std::memory_order_relaxed);
      }
      chunks_[c].store(fresh, std::memory_order_release);
    }
  }
  return i;
}

void MSQueue::free_node(uint32_t i) {
  uint64_t h = free_head_.load(std::memory_order_acquire);
  do {
    node(i).free_next.store(idx_of(h), std::memory_order_relaxed);
  } while (!free_head_.compare_exchange_weak(h, pack(i, tag_of(h) + 1), std::memory_order_acq_rel,
                                             std::memory_order_acquire));
}

void MSQueue::enqueue(uint64_t v) {
  const uint32_t n = alloc_node();
  Node& nn = node(n);
  nn.value.store(v, std::memory_order_relaxed);
  // Re-arm the link with a fresh tag so a stale enqueuer's CAS on a recycled
  // node cannot succeed (ABA on next).
  const uint64_t old = nn.next.load(std::memory_order_relaxed);
  nn.next.store(pack(NIL, tag_of(old) + 1), std::memory_order_release);
  uint64_t tail;
  for (;;) {
    tail = tail_.load(std::memory_order_acquire);
    uint64_t next = node(idx_of(tail)).next.load(std::memory_order_acquire);
    if (tail != tail_.load(std::memory_order_acquire)) continue;
    if (idx_of(next) == NIL) {
      if (node(idx_of(tail)).next.compare_exchange_weak(next, pack(n, tag_of(next) + 1), std::memory_order_acq_rel,
                                                        std::memory_order_acquire))
        break;
    } else {
      tail_.compare_exchange_weak(tail, pack(idx_of(next), tag_of(tail) + 1), std::memory_order_acq_rel,
                                  std::memory_order_acquire);
    }
  }
  tail_.compare_exchange_strong(tail, pack(n, tag_of(tail) + 1), std::memory_order_acq_rel,
                                std::memory_order_acquire);
}

bool MSQueue::dequeue(uint64_t* out) {
  uint64_t head;
  uint64_t v;
  for (;;) {
    head = head_.load(std::memory_order_acquire);
    uint64_t tail = tail_.load(std::memory_order_acquire);
    uint64_t next = node(idx_of(head)).next.load(std::memory_order_acquire);
    if (head != head_.load(std::memory_order_acquire)) continue;
    if (idx_of(head) == idx_of(tail)) {
      if (idx_of(next) == NIL) return false;
      tail_.compare_exchange_weak(tail, pack(idx_of(next), tag_of(tail) + 1), std::memory_order_acq_rel,
                                  std::memory_order_acquire);
    } else {
      v = node(idx_of(next)).value.load(std::memory_order_acquire);
      if (head_.compare_exchange_weak(head, pack(idx_of(next), tag_of(head) + 1), std::memory_order_acq_rel,
                                      std::memory_order_acquire))
        break;
    }
  }
  free_node(idx_of(head));  // the old dummy retires; `next` is the new dummy
  *out = v;
  return true;
}

bool MSQueue::is_empty() const {
  for (;;) {
    const uint64_t head = head_.load(std::memory_order_acquire);
    const uint64_t next = node(idx_of(head)).next.load(std::memory_order_acquire);
    if (head == head_.load(std::memory_order_acquire)) return idx_of(next) == NIL;
  }
}

}  // namespace tr
