// The k-panel schedule for cold (host-resident) single-device products; see
// session.h and DESIGN.md section 4.
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

namespace {
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
}  // namespace

// ---------------------------------------------------------------- k-panel schedule
// A cold product on one device is bound by the host link (H2D of A and B), and
// the GPU can only compute what has arrived.  Whole-task launches need a task's
// full A row panel and B column panel first, so in the first half of a cold run
// the tensor cores starve (shell s makes (2s+1) tasks runnable per 2·k tiles)
// and the backlog becomes the tail.  The k-panel schedule streams the first P
// k-panels in k-major order instead -- panel p (A[:,p] and B[p,:], 2g tiles)
// makes ONE k-step of every task runnable (g² units: as much compute as the
// panel took to copy) -- then finishes the tasks in shells order over the
// remaining k-panels, so C tiles complete (and are written back) progressively.
// Every task keeps its own C accumulator in HBM between its units.  Directory
// sequence per task: admit C, then per unit acquire A then B per k-step and
// release; release C after the last unit -- the reference's operations, so all
// counters keep the reference's values.  Fills are issued up front in arrival
// order (uncounted, like fetch-ahead); each unit's launch waits for its tiles.
bool Session::panels_apply(const Job& job) const {
  if (dryrun_ || sim_ || exact_ || !coherence_ || n_devices() != 1 || devs_[0].capacity >= 0 || job.prods.size() != 1)
    return false;
  if (!(order_ == -1 || order_ == 4) || (flags_ & TR_FLAG_NO_PREFETCH)) return false;
  const Product& p = job.prods[0];
  if (p.a.location != TR_LOC_HOST || p.b.location != TR_LOC_HOST || p.c.location != TR_LOC_HOST) return false;
  if (p.post != POST_NONE || p.k_steps < 2 || p.k_steps > kMaxKSteps) return false;
  if (small_gemm_enabled() && (tile_ <= kSmallMaxN || p.N <= kSmallMaxN)) return false;  // CUDA-core tasks
  if (order_ == -1 && job.n_tasks < 16) return false;  // small products gain nothing
  // in-core, or out-of-core with the future-aware directory (blocks, see run_panels)
  const int64_t T = tile_;
  const int64_t in_tiles = ceil_div(p.a.rows, T) * ceil_div(p.a.cols, T) + ceil_div(p.b.rows, T) * ceil_div(p.b.cols, T);
  return job.out_of_core || dir_->used_tiles(0) + in_tiles <= devs_[0].max_slots;
}

bool Session::run_panels(Job& job) {
  NvtxRange nv("tr.k_panels");
  const int d = 0;
  DeviceCtx& dc = devs_[d];
  const Product& p = job.prods[0];
  const int64_t T = tile_, ks = p.k_steps;
  const std::vector<int64_t>& order = job.order;  // planned tasks: shells, or blocks walked in shells
  const size_t nt_tasks = order.size();
  const int W = dc.width;
  const int G = std::max(1, std::min(max_group_, kMaxGroup));
  const int64_t ces = p.c.esize();
  std::vector<int64_t> ti(nt_tasks), tj(nt_tasks);
  for (size_t q = 0; q < nt_tasks; ++q) {
    int64_t tid = 0;
    job.prod_of(order[q], &tid);
    ti[q] = tid / p.grid_cols;
    tj[q] = tid % p.grid_cols;
  }
  // Task blocks: in-core, all tasks; out-of-core, the blocked order's b x b task
  // blocks (their panels fit the slab), scheduled one after another -- the next
  // block's fills take the slots of the previous block's dead tiles as soon as
  // the kernels reading them are done.
  std::vector<std::pair<size_t, size_t>> blocks;
  if (job.out_of_core) {
    const int64_t bsz = std::max<int64_t>(1, (static_cast<int64_t>(dc.max_slots) - 8) / (2 * ks));
    size_t b0 = 0;
    for (size_t q = 1; q <= nt_tasks; ++q)
      if (q == nt_tasks || ti[q] / bsz != ti[b0] / bsz || tj[q] / bsz != tj[b0] / bsz) {
        blocks.emplace_back(b0, q);
        b0 = q;
      }
  } else {
    blocks.emplace_back(0, nt_tasks);
  }
  size_t max_block = 0;
  for (const auto& b : blocks) max_block = std::max(max_block, b.second - b.first);
  // ---- 0. C accumulators in HBM for one block's tasks (reused block to block);
  //         without room, the caller runs the ordinary task path (nothing touched yet)
  struct CbufGuard {
    int gpu;
    void* p = nullptr;
    size_t cap = 0;
    ~CbufGuard() {
      if (p) DevPool::get().release(gpu, p, cap);
    }
  } guard{dc.gpu};
  const size_t ctile = static_cast<size_t>(T * T * ces);
  if (DevPool::get().alloc(dc.gpu, ctile * max_block, &guard.p, &guard.cap) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  std::vector<EvRef> cbuf_free(max_block);  // D2H of the accumulator's previous task done
  std::vector<EvRef> task_last(nt_tasks);   // completion of each task's previous unit
  int64_t P = std::max<int64_t>(1, ks / 4);  // measured best on cfg2 (tools/probe_panels.py)
  if (const char* e = getenv("TR_PANELS")) P = std::max<int64_t>(0, std::min<int64_t>(ks, atoi(e)));
  // k-steps per finishing unit: a unit starts as soon as ITS tiles are in, so
  // short units let the last shell's compute follow its tiles in
  int64_t F = ks;
  if (const char* e = getenv("TR_PANEL_FINISH")) F = std::max<int64_t>(1, atoi(e));
  int gb = 1;  // tasks per finishing launch: each starts as soon as its own tiles are in
  if (const char* e = getenv("TR_PANEL_GROUP")) gb = std::max(1, std::min(G, atoi(e)));
  auto a_key = [&](int64_t i, int64_t k) { return p.ta ? std::make_pair(k, i) : std::make_pair(i, k); };
  auto b_key = [&](int64_t k, int64_t j) { return p.tb ? std::make_pair(j, k) : std::make_pair(k, j); };
  auto tall = [&](size_t q) { return group_uses_pairs(static_cast<int>(std::min(T, p.M - ti[q] * T))); };
  struct Unit {
    size_t q;
    int64_t k0, k1;
    int64_t launch;  // units with the same launch id form one grouped launch
  };
  int64_t li = 0;  // launches so far (stream rotation)
  for (const auto& blk : blocks) {
    // ---- 1. the block's units: the first P k-panels k-major in groups of G
    //         tasks, then one finishing unit per task (k = P..ks-1)
    std::vector<Unit> units;
    int64_t launch = 0;
    auto add_grouped = [&](int64_t k0, int64_t k1, int gsz) {
      size_t in_launch = 0;
      for (size_t q = blk.first; q < blk.second; ++q) {
        if (in_launch > 0 && (static_cast<int>(in_launch) == gsz || tall(q) != tall(units.back().q))) {
          ++launch;
          in_launch = 0;
        }
        units.push_back(Unit{q, k0, k1, launch});
        ++in_launch;
      }
      ++launch;
    };
    for (int64_t k = 0; k < P; ++k) add_grouped(k, k + 1, G);
    if (P < ks && F >= ks - P) {
      add_grouped(P, ks, gb);
    } else if (P < ks) {  // finishing in chunks of F k-steps, task by task (same fill order)
      for (size_t q = blk.first; q < blk.second; ++q)
        for (int64_t k0 = P; k0 < ks; k0 += F) units.push_back(Unit{q, k0, std::min(ks, k0 + F), launch++});
    }
    // ---- 2. fills in first-need order (uncounted, like fetch-ahead; the unit's acquire counts them)
    for (const Unit& u : units)
      for (int64_t k = u.k0; k < u.k1; ++k)
        for (int which = 0; which < 2; ++which) {
          const auto rc = which == 0 ? a_key(ti[u.q], k) : b_key(k, tj[u.q]);
          const Mat& m = which == 0 ? p.a : p.b;
          const uint64_t uid = which == 0 ? p.a_uid : p.b_uid;
          DirLock g(dir_->mu);
          int32_t slot = -1, source = TR_SOURCE_HOST;
          const TileKey key{uid, rc.first, rc.second};
          if (!dir_->prefetch_locked(d, key, &slot, &source, false)) continue;
          load_slot(d, W, phys_of(d, slot), source >= 0 ? HIT_L2 : HIT_MISS, source, key, m, rc.first, rc.second,
                    job);
        }
    // ---- 3. launches: a task's units are ordered by events, launches rotate over the streams
    std::vector<int64_t> units_left(nt_tasks, 0);
    for (const Unit& u : units) units_left[u.q] += 1;
    for (size_t b = 0; b < units.size();) {
      size_t e = b;
      while (e < units.size() && units[e].launch == units[b].launch) ++e;
      const int s = static_cast<int>(li++ % W);
      StreamCtx& sc = dc.streams[s];
      GemmGroup grp;
      grp.n_tasks = static_cast<int32_t>(e - b);
      grp.k_split = 1;
      std::vector<TileKey> used;
      std::vector<int32_t> used_phys;
      for (size_t x = b; x < e; ++x) {
        const Unit& u = units[x];
        const size_t cq = u.q - blk.first;  // accumulator slot
        const int64_t i = ti[u.q], j = tj[u.q];
        const int64_t mt = std::min(T, p.M - i * T), nt = std::min(T, p.N - j * T);
        if (u.k0 == 0) {
          DirLock lk(dir_->mu);
          dir_->admit_output_locked(d, TileKey{p.c_uid, i, j});  // scheduler.py:390
          wait_on(d, s, cbuf_free[cq]);
        }
        wait_on(d, s, task_last[u.q]);
        GemmArgs& a = grp.task[x - b];
        std::memset(&a, 0, sizeof(a));
        a.m_valid = static_cast<int32_t>(mt);
        a.n_valid = static_cast<int32_t>(nt);
        a.n_ksteps = static_cast<int32_t>(u.k1 - u.k0);
        a.planes = planes_;
        a.c = static_cast<char*>(guard.p) + cq * ctile;
        a.ldc = nt;
        a.c_f64 = p.c.dtype == TR_DTYPE_F64;
        a.epilogue = u.k0 == 0 ? EPI_STORE : EPI_ACCUMULATE;
        a.seg_kb = seg_kb_for(planes_);
        a.k_split = 1;
        for (int64_t k = u.k0; k < u.k1; ++k) {
          const auto ak = a_key(i, k), bk = b_key(k, j);
          const int32_t pa = acquire(d, s, job, p.a, p.a_uid, p.ta, ak.first, ak.second, 0);
          const int32_t pb = acquire(d, s, job, p.b, p.b_uid, p.tb, bk.first, bk.second, 1);
          a.a_z[k - u.k0] = pa * planes_;
          a.b_z[k - u.k0] = pb * planes_;
          a.k_len[k - u.k0] = static_cast<int32_t>(std::min(T, p.K - k * T));
          used.push_back(TileKey{p.a_uid, ak.first, ak.second});
          used.push_back(TileKey{p.b_uid, bk.first, bk.second});
          used_phys.push_back(pa);
          used_phys.push_back(pb);
        }
      }
      BoxKind ba, bb;
      gemm_boxes(p.ta, p.tb, grp.task[0].m_valid, &ba, &bb, /*grouped=*/true);
      TimedLaunch tl = timing_pair(d);
      TR_CUDA(cudaEventRecord(tl.start, sc.stream));
      // non-persistent: the schedule keeps several launches in flight on its streams
      TR_CUDA(launch_tile_gemm_group(dc.tmap[ba], dc.tmap[bb], grp, p.ta, p.tb, /*persistent=*/false, sc.stream));
      TR_CUDA(cudaEventRecord(tl.end, sc.stream));
      dc.timed.push_back(tl);
      if (tracing_)
        for (size_t x = b; x < e; ++x) {
          TraceRec rec;
          rec.ev = tr_trace_event{d, TR_TRACE_GEMM, s, order[units[x].q], static_cast<uint64_t>(dc.timed.size() - 1),
                                  ti[units[x].q], tj[units[x].q], 0.0, 0.0};
          rec.t = TimedLaunch{nullptr, nullptr};
          dc.trace.push_back(rec);
        }
      job.launches.fetch_add(1);
      {
        DirLock lk(dir_->mu);
        const EvRef ev = record(d, s);
        for (int32_t ph : used_phys) note_use(dc.slots[ph], ev);
        for (const TileKey& key : used) dir_->release_input_locked(d, key);
        for (size_t x = b; x < e; ++x) task_last[units[x].q] = ev;
      }
      // finished tasks: one pitched D2H each on the writeback stream (so the
      // compute stream's next launch does not queue behind it), then release C
      const int wb = W + 2;
      for (size_t x = b; x < e; ++x) {
        const size_t q = units[x].q;
        if (--units_left[q] != 0) continue;
        const int64_t i = ti[q], j = tj[q];
        const int64_t mt = std::min(T, p.M - i * T), nt = std::min(T, p.N - j * T);
        char* dst = const_cast<char*>(static_cast<const char*>(p.c.ptr)) + (i * T * p.c.ld + j * T) * ces;
        wait_on(d, wb, task_last[q]);
        TimedLaunch tw{};
        trace_begin(d, wb, &tw);
        TR_CUDA(cudaMemcpy2DAsync(dst, p.c.ld * ces, static_cast<char*>(guard.p) + (q - blk.first) * ctile, nt * ces,
                                  nt * ces, mt, cudaMemcpyDeviceToHost, dc.streams[wb].stream));
        trace_end(d, wb, tw, TR_TRACE_D2H, order[q], p.c_uid, i, j);
        DirLock lk(dir_->mu);
        cbuf_free[q - blk.first] = record(d, wb);
        dir_->release_output_locked(d, TileKey{p.c_uid, i, j}, mt * nt * element_bytes_);  // coherence.py:263-280
      }
      b = e;
    }
  }
  // ---- 4. completion
  for (auto& sc : dc.streams) TR_CUDA(cudaStreamSynchronize(sc.stream));
  for (int64_t gt : order) {
    job.mark(gt);
    dc.stats.tasks_completed += 1;
    dc.stats.macs += job.task_macs(gt, tile_);
  }
  return true;
}

}  // namespace tr
