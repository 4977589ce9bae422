// The simulated engine (TR_FLAG_SIM): the reference's sim event loop and cost
// model replayed natively; see session.h and DESIGN.md section 6.
#include "session.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>
#include <utility>
#include <vector>

#include "common.h"

namespace tr {

// ---------------------------------------------------------------- simulated engine
// The reference's sim engine (scheduler.py:432-464) with its cost model
// (devices.py:255-283), replayed natively: devices are served in order of their
// compute clock (ties to the lower id), each refills its station, pops (or,
// after observing an empty queue, steals), and runs the whole task's directory
// sequence at once; fetch k+1 overlaps compute k, the writeback waits for the
// last accumulate.  Every double is formed in the reference's operation order,
// so makespans match the reference bit for bit.
double Session::sim_now() const {
  double t = 0.0;
  for (const SimClock& c : clocks_) t = std::max(t, std::max(c.compute, c.transfer));
  return t;
}

double Session::xfer_cost(int src, int dst, int64_t nbytes) const {
  if (src == dst) return 0.0;
  if (src == TR_SOURCE_HOST || dst == TR_SOURCE_HOST) {
    const int dev = src == TR_SOURCE_HOST ? dst : src;
    if (host_worker_[dev]) return 0.0;
    return static_cast<double>(nbytes) / host_bw_[dev] + latency_;
  }
  return static_cast<double>(nbytes) / peer_bw_[static_cast<size_t>(src) * n_devices() + dst] + latency_;
}

void Session::sim_task(int d, Job& job, int64_t gtid, double t) {
  int64_t tid = 0;
  const Product& p = job.prod_of(gtid, &tid);
  const int64_t T = tile_;
  const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
  const int64_t mt = std::min(T, p.M - i * T);
  const int64_t nt = std::min(T, p.N - j * T);
  const TileKey c_key{p.c_uid, i, j};
  std::vector<std::pair<double, double>> steps;
  steps.reserve(static_cast<size_t>(p.k_steps));
  {
    DirLock g(dir_->mu);
    dir_->admit_output_locked(d, c_key);  // scheduler.py:390
    for (int64_t k = 0; k < p.k_steps; ++k) {
      const int64_t ar = p.ta ? k : i, ac = p.ta ? i : k;
      const int64_t br = p.tb ? j : k, bc = p.tb ? k : j;
      const int64_t na = std::min(T, p.a.rows - ar * T) * std::min(T, p.a.cols - ac * T) * element_bytes_;
      const int64_t nb = std::min(T, p.b.rows - br * T) * std::min(T, p.b.cols - bc * T) * element_bytes_;
      const TileKey ka{p.a_uid, ar, ac}, kb{p.b_uid, br, bc};
      const Acquired ra = dir_->acquire_input_locked(d, ka, na);
      const Acquired rb = dir_->acquire_input_locked(d, kb, nb);
      const double fetch = xfer_cost(ra.source, d, ra.nbytes) + xfer_cost(rb.source, d, rb.nbytes);
      const int64_t kt = std::min(T, p.K - k * T);
      const double compute = 2.0 * static_cast<double>(mt) * static_cast<double>(kt) * static_cast<double>(nt) / flops_[d];
      dir_->release_input_locked(d, ka);
      dir_->release_input_locked(d, kb);
      steps.emplace_back(fetch, compute);
    }
    const int64_t wb_bytes = mt * nt * element_bytes_;
    const double wb = xfer_cost(d, TR_SOURCE_HOST, wb_bytes);
    dir_->release_output_locked(d, c_key, wb_bytes);
    SimClock& eng = clocks_[d];
    double tr = std::max(eng.transfer, t);  // transfers for this task cannot predate claiming it
    double co = eng.compute;
    for (const auto& st : steps) {
      tr += st.first;
      co = std::max(co, tr) + st.second;  // fetch k+1 overlaps compute k
    }
    tr = std::max(tr, co) + wb;  // the writeback waits for the last accumulate
    eng.transfer = tr;
    eng.compute = co;
  }
  job.mark(gtid);
  devs_[d].stats.tasks_completed += 1;
  devs_[d].stats.macs += job.task_macs(gtid, tile_);
}

void Session::run_sim(Job& job) {
  using Ev = std::pair<double, int>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap;
  for (int d = 0; d < n_devices(); ++d) heap.emplace(clocks_[d].compute, d);
  while (!heap.empty()) {
    const Ev top = heap.top();
    heap.pop();
    const double t = top.first;
    const int d = top.second;
    Station& st = *devs_[d].station;
    job.claimed.fetch_add(static_cast<int64_t>(st.refill(job.queue, st.width()).size()));
    uint64_t tid = 0;
    if (!st.pop_for_run(&tid)) {
      int victim = -1;
      bool got = false;
      if (steal_ && job.queue.is_empty())
        got = steal_task(d, station_ptrs_.data(), static_cast<int>(station_ptrs_.size()), &tid, &victim);
      if (!got) continue;  // queue drained and nothing stealable: the device retires
      job.steals.push_back(tr_steal_event{d, victim, static_cast<int64_t>(tid), t});
      devs_[d].stats.steals_performed += 1;
      devs_[victim].stats.steals_suffered += 1;
    }
    sim_task(d, job, static_cast<int64_t>(tid), t);
    heap.emplace(clocks_[d].compute, d);
  }
}

}  // namespace tr
