// ThreadSanitizer stress of the runtime's host-side concurrency (SURVEY.md §5
// "race detection": TSAN on the C++ units).  Built and run by
// tests/test_native_tsan.py with g++ -fsanitize=thread; exits non-zero on a
// contract violation, and TSAN aborts the process on a data race.
//
//  1. MSQueue (msqueue.cpp): 4 producers x 4 consumers; every value dequeued
//     exactly once, each producer's values in order (msqueue.py:9-12).
//  2. Global queue + reservation stations (station.h): 8 owners refill, pop and
//     steal from each other; every task id obtained exactly once
//     (scheduler.py:200-249).
//  3. Directory (directory.cpp) with debug invariants: 8 device threads run the
//     _execute_task protocol (admit_output, acquire/release A and B per k-step,
//     release_output; scheduler.py:371-410) on a shared key space, so L1 hits,
//     L2 hits, host fetches and evictions interleave; the counters must add up
//     (l1 + l2 + host == input requests, writebacks == tasks).
#include <atomic>
#include <chrono>
#include <memory>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "directory.h"
#include "msqueue.h"
#include "station.h"

namespace {

int failures = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

void queue_stress() {
  tr::MSQueue q;
  const int P = 4, C = 4, per = 50000;
  std::atomic<int> done{0};
  std::vector<std::vector<uint64_t>> got(C);
  std::vector<std::thread> th;
  for (int p = 0; p < P; ++p)
    th.emplace_back([&, p] {
      for (int i = 0; i < per; ++i) q.enqueue((static_cast<uint64_t>(p) << 32) | static_cast<uint64_t>(i));
      done.fetch_add(1);
    });
  for (int c = 0; c < C; ++c)
    th.emplace_back([&, c] {
      uint64_t v;
      while (true) {
        if (q.dequeue(&v)) {
          got[c].push_back(v);
        } else if (done.load() == P && q.is_empty()) {
          break;
        }
      }
    });
  for (auto& t : th) t.join();
  std::vector<int> seen(static_cast<size_t>(P) * per, 0);
  for (int c = 0; c < C; ++c) {
    std::vector<int64_t> last(P, -1);
    for (uint64_t v : got[c]) {
      const int p = static_cast<int>(v >> 32), i = static_cast<int>(v & 0xFFFFFFFFu);
      CHECK(i > last[p]);  // per-producer FIFO as seen by one consumer
      last[p] = i;
      seen[static_cast<size_t>(p) * per + i] += 1;
    }
  }
  for (int s : seen) CHECK(s == 1);
  CHECK(q.is_empty());
}

void station_stress() {
  tr::MSQueue q;
  const int N = 8, tasks = 20000;
  for (int t = 0; t < tasks; ++t) q.enqueue(static_cast<uint64_t>(t));
  std::vector<std::unique_ptr<tr::Station>> sp;
  for (int d = 0; d < N; ++d) sp.emplace_back(new tr::Station(d, 4));
  auto st = [&](int d) -> tr::Station& { return *sp[d]; };
  std::vector<std::atomic<int>> taken(tasks);
  for (auto& a : taken) a.store(0);
  std::atomic<int> steals{0};
  std::vector<std::thread> th;
  for (int d = 0; d < N; ++d)
    th.emplace_back([&, d] {
      std::mt19937 rng(static_cast<unsigned>(d));
      uint64_t tid;
      while (true) {
        st(d).refill(q, 4);
        if (st(d).pop_for_run(&tid)) {
          taken[tid].fetch_add(1);
          // two slow owners: their reserved ids are left for the others to steal
          if (d < 2) std::this_thread::sleep_for(std::chrono::microseconds(50));
          continue;
        }
        // queue empty and own station empty: steal from the others (scheduler.py:239-249)
        bool got = false;
        for (int k = 1; k < N && !got; ++k) {
          const int v = (d + k + static_cast<int>(rng() % N)) % N;
          if (v != d && st(v).try_steal(&tid)) {
            taken[tid].fetch_add(1);
            steals.fetch_add(1);
            got = true;
          }
        }
        if (!got && q.is_empty()) {
          bool all_empty = true;
          for (int v = 0; v < N; ++v) {
            uint64_t x;
            if (st(v).peek_front(&x)) all_empty = false;
          }
          if (all_empty) break;
        }
      }
    });
  for (auto& t : th) t.join();
  for (auto& a : taken) CHECK(a.load() == 1);
  std::printf("stations: %d tasks, %d steals\n", tasks, steals.load());
  // deterministic stealing: an owner reserves ids and never runs them; seven
  // thieves race to steal them from the back -- each id is taken exactly once
  tr::MSQueue q2;
  for (int t = 0; t < 64; ++t) q2.enqueue(static_cast<uint64_t>(t));
  tr::Station owner(0, 64);
  CHECK(static_cast<int>(owner.refill(q2, 64).size()) == 64);
  std::vector<std::atomic<int>> got(64);
  for (auto& a : got) a.store(0);
  std::vector<std::thread> thieves;
  for (int d = 1; d < N; ++d)
    thieves.emplace_back([&] {
      uint64_t tid;
      while (owner.try_steal(&tid)) got[tid].fetch_add(1);
    });
  for (auto& t : thieves) t.join();
  for (auto& a : got) CHECK(a.load() == 1);
}

void directory_stress() {
  const int N = 8, g = 6, tasks_per_dev = 200;
  const int64_t tile_bytes = 4096;
  std::vector<int64_t> cap(N, 16), hops(N * N, 1);
  for (int d = 0; d < N; ++d) hops[d * N + d] = 0;
  tr::Directory dir(N, cap, std::vector<bool>(N, false), hops, true, TR_POLICY_LRU, /*debug=*/true);
  std::atomic<int64_t> requests{0};
  std::vector<std::thread> th;
  for (int d = 0; d < N; ++d)
    th.emplace_back([&, d] {
      std::mt19937 rng(static_cast<unsigned>(100 + d));
      for (int t = 0; t < tasks_per_dev; ++t) {
        const int64_t i = rng() % g, j = rng() % g;
        const tr::TileKey ck{3, static_cast<int64_t>(d) * 1000 + t, 0};  // outputs are unique per task
        dir.admit_output(d, ck);
        for (int64_t k = 0; k < g; ++k) {
          const tr::TileKey ak{1, i, k}, bk{2, k, j};
          dir.acquire_input(d, ak, tile_bytes);
          dir.acquire_input(d, bk, tile_bytes);
          requests.fetch_add(2);
          dir.release_input(d, ak);
          dir.release_input(d, bk);
        }
        dir.release_output(d, ck, tile_bytes);
      }
    });
  for (auto& t : th) t.join();
  dir.check_invariants();
  const tr_cache_stats s = dir.stats();
  CHECK(s.l1_hits + s.l2_hits + s.host_fetches == requests.load());
  CHECK(s.writebacks == static_cast<int64_t>(N) * tasks_per_dev);
  CHECK(s.bytes_host == s.host_fetches * tile_bytes && s.bytes_peer == s.l2_hits * tile_bytes);
  CHECK(s.l1_hits > 0 && s.l2_hits > 0 && s.evictions > 0);
  std::printf("directory: l1 %lld l2 %lld host %lld evictions %lld writebacks %lld\n",
              static_cast<long long>(s.l1_hits), static_cast<long long>(s.l2_hits),
              static_cast<long long>(s.host_fetches), static_cast<long long>(s.evictions),
              static_cast<long long>(s.writebacks));
}

}  // namespace

namespace tr {
void set_last_error(const char*) {}
}  // namespace tr

int main() {
  queue_stress();
  station_stress();
  directory_stress();
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("tsan stress ok\n");
  return 0;
}
