// Lock-free Michael-Scott MPMC FIFO of 64-bit task ids.
//
// Replaces the reference's two-lock queue (msqueue.py:28-67; the paper, PAPER.md:40,
// asks for the lock-free variant).  Same contract (msqueue.py:9-12): every enqueued
// value is dequeued exactly once or is still queued, values from one producer
// come out in order, and is_empty() is exact once producers have quiesced.
//
// ABA safety uses the original paper's counted pointers: every link is a 64-bit
// word {node index : 32, tag : 32} and every successful CAS bumps the tag.  Nodes
// live in a chunked pool that is never returned to the OS, so a stale reader can
// always dereference an index; its CAS then fails on the tag.  Retired nodes go to
// a tagged Treiber free list.
#pragma once

#include <atomic>
#include <cstdint>
#include <mutex>

namespace tr {

class MSQueue {
 public:
  MSQueue();
  ~MSQueue();
  MSQueue(const MSQueue&) = delete;
  MSQueue& operator=(const MSQueue&) = delete;

  void enqueue(uint64_t v);
  bool dequeue(uint64_t* out);  // false when empty
  bool is_empty() const;

 private:
  static constexpr uint32_t NIL = 0xFFFFFFFFu;
  static constexpr int kChunkBits = 12;
  static constexpr uint32_t kChunk = 1u << kChunkBits;
  static constexpr int kMaxChunks = 1 << 16;  // 2^28 nodes max

  struct Node {
    std::atomic<uint64_t> next;
    std::atomic<uint64_t> value;
    std::atomic<uint32_t> free_next;
  };

  static uint64_t pack(uint32_t idx, uint32_t tag) { return (static_cast<uint64_t>(tag) << 32) | idx; }
  static uint32_t idx_of(uint64_t w) { return static_cast<uint32_t>(w & 0xFFFFFFFFu); }
  static uint32_t tag_of(uint64_t w) { return static_cast<uint32_t>(w >> 32); }

  Node& node(uint32_t i) const { return chunks_[i >> kChunkBits].load(std::memory_order_acquire)[i & (kChunk - 1)]; }
  uint32_t alloc_node();
  void free_node(uint32_t i);

  std::atomic<Node*>* chunks_;
  std::atomic<uint32_t> n_fresh_{0};
  std::mutex grow_mu_;
  alignas(64) std::atomic<uint64_t> free_head_;
  alignas(64) std::atomic<uint64_t> head_;
  alignas(64) std::atomic<uint64_t> tail_;
};

}  // namespace tr
