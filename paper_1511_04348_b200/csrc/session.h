// The GPU runtime session: Runtime (scheduler.py:522-621) re-designed for B200.
//
//   reference (Python, simulated devices)        this build
//   ------------------------------------------   ------------------------------------------------
//   one Python thread per device (467-516)       one pinned C++ thread per logical device
//   ReservationStation width 4 (200-236)         station entries feed CUDA streams (one per entry)
//   _execute_task k-loop (371-410)               async issue: acquire tiles -> fills on the
//                                                task's stream -> ONE tcgen05 GEMM launch over
//                                                all k-steps -> D2H writeback of C
//   CacheDirectory (coherence.py)                same directory + physical HBM slab slots;
//                                                L2 hit = cudaMemcpyPeerAsync from the owner,
//                                                miss = pinned-host H2D + split/convert (K2)
//   instantaneous copies under one lock          copies are async; ordering is enforced with
//                                                CUDA events: a slot is refilled only after every
//                                                stream that read it has passed its last use
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "devpool.h"
#include "directory.h"
#include "msqueue.h"
#include "station.h"
#include "tile_gemm.h"

namespace tr {

constexpr int64_t kTaskNone = -1;    // StreamCtx::task: idle
constexpr int64_t kTaskMarked = -2;  // StreamCtx::task: a stream-ordered launch in flight, counted at enqueue


struct Mat {
  const void* ptr = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  int32_t dtype = TR_DTYPE_F32;
  int32_t location = TR_LOC_HOST;
  int64_t esize() const { return dtype == TR_DTYPE_F64 ? 8 : 4; }
};

class Session;

// One product of a job (a batch of independent products may share a job).
struct Product {
  Mat a, b, c;
  bool ta = false, tb = false;
  uint64_t a_uid = 0, b_uid = 0, c_uid = 0;
  int64_t M = 0, N = 0, K = 0;
  int64_t grid_rows = 0, grid_cols = 0, k_steps = 0;
  int64_t base = 0;  // first global task id of this product
  // fused epilogue post-op (tile_gemm.h PostOp), device float32 outputs only
  int32_t post = 0, act = 0;
  const float* bias = nullptr;
  const float* aux = nullptr;
  int64_t ldaux = 0;
  uint64_t cache_as = 0;  // write-through: the output's tiles enter the cache under this uid
  bool axpy = false;      // C += alpha * A.B (every k-chunk accumulates)
  float alpha = 1.f;
  float* colsum = nullptr;  // 32-row block column sums of the final output (tr_product.colsum)
};

struct Job {
  std::vector<Product> prods;
  int64_t total = 0;    // global task ids [0, total)
  int64_t n_tasks = 0;  // planned tasks (shard)
  MSQueue queue;
  std::vector<std::atomic<uint8_t>> done;  // exactly-once bitmap over ALL global task ids
  std::atomic<int64_t> done_count{0};
  std::atomic<bool> abort{false};
  std::mutex mu;  // errors + steal log
  int err_status = 0;
  std::string err_msg;
  std::vector<tr_steal_event> steals;
  std::atomic<int64_t> launches{0};
  std::vector<int64_t> order;          // planned global task ids in enqueue order
  std::atomic<int64_t> claimed{0};     // tasks pulled from the queue so far (all devices)
  bool async = false;                  // stream-ordered: tasks complete in stream order, no host wait
  bool out_of_core = false;            // inputs exceed the HBM slab (future-aware eviction on)

  explicit Job(int64_t total_ids) : total(total_ids), done(static_cast<size_t>(total_ids)) {
    for (auto& d : done) d.store(0);
  }
  // product owning global task id g; *tid = its task id within the product
  const Product& prod_of(int64_t g, int64_t* tid) const {
    size_t lo = 0, hi = prods.size();
    while (hi - lo > 1) {
      const size_t mid = (lo + hi) / 2;
      if (prods[mid].base <= g) lo = mid;
      else hi = mid;
    }
    *tid = g - prods[lo].base;
    return prods[lo];
  }
  void mark(int64_t tid);  // scheduler.py:78-83
  // rows x cols x K of global task g (its share of the work)
  int64_t task_macs(int64_t g, int64_t tile) const {
    int64_t t = 0;
    const Product& p = prod_of(g, &t);
    const int64_t i = t / p.grid_cols, j = t % p.grid_cols;
    const int64_t mt = p.M - i * tile < tile ? p.M - i * tile : tile;
    const int64_t nt = p.N - j * tile < tile ? p.N - j * tile : tile;
    return mt * nt * p.K;
  }
  bool all_done() const { return done_count.load() == n_tasks; }
  void set_error(int status, const std::string& msg);
};

// Tasks per grouped K1 launch for sessions created from now on (1 disables);
// default 4, or TR_GROUP=<n> in the environment.
int task_group_max();
void set_task_group_max(int n);
int split_factor(int64_t ctas, int total_kb, int64_t sms);

class Session {
 public:
  Session(const tr_machine& m, int32_t tile, int32_t precision, uint32_t flags, int64_t hbm_budget);
  ~Session();

  Directory& directory() { return *dir_; }
  int n_devices() const { return static_cast<int>(devs_.size()); }
  // Runs one product (scheduler.py:559-612); fills `rep`.
  void gemm(const Mat& a, uint64_t a_uid, bool ta, const Mat& b, uint64_t b_uid, bool tb, const Mat& c,
            uint64_t c_uid, int64_t task_offset, int64_t task_stride, tr_gemm_report* rep);
  // A batch of independent products scheduled as one job (their tasks interleave).
  void run_products(std::vector<Product> prods, int64_t task_offset, int64_t task_stride, tr_gemm_report* rep);
  void kernel_ms(double* out) const;
  void span_ms(double* out) const;
  void set_inflight(int n);
  void set_order(int order) { order_ = order; }
  void set_external_stream(cudaStream_t s, bool on) {
    ext_stream_ = on ? s : nullptr;
    ext_on_ = on;
  }
  void set_async(bool on) { async_ = on; }
  double sim_now() const;
  const std::vector<tr_trace_event>& trace() const { return last_trace_; }

 private:
  static constexpr int kStage = 4;  // H2D staging ring depth per device

  // A point on a stream.  Events are recycled only after they completed, so a
  // reference whose generation no longer matches its event names a point that
  // is known to be complete (waiting on it is a no-op).
  struct EvRef {
    int32_t gs = -1;   // global stream id (device * 64 + stream); -1 = none
    int32_t idx = -1;  // index in that stream's event pool
    uint64_t gen = 0;  // generation of the recording
  };
  struct SlotState {
    EvRef ready;              // fill (convert or peer copy) of the current content
    std::vector<EvRef> uses;  // last read of the slot by each stream (kernels, peer copies)
  };
  struct StreamCtx {
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> evs;   // event pool, recycled in recording order once complete
    std::vector<uint64_t> gen;
    std::deque<int32_t> fifo;
    cudaEvent_t done = nullptr;
    int64_t task = -1;      // in-flight task id; kTaskNone idle, kTaskMarked stream-ordered (already counted)
    std::vector<int64_t> group_rest;  // further tasks of an in-flight grouped launch
    uint64_t seq = 0;       // issue order
    void* staging = nullptr;  // host-tile landing zone (T*T*8 bytes)
    void* outbuf = nullptr;   // C tile for host outputs (T*T*8 bytes)
    size_t staging_cap = 0, outbuf_cap = 0;
    float* ws = nullptr;      // split-K partial sums (grown on demand)
    size_t ws_cap = 0;
    void* gout = nullptr;     // C tiles of a grouped launch with host outputs (grown on demand)
    size_t gout_cap = 0;
    EvRef gout_free;          // the writeback stream's D2H of gout's previous contents
  };
  struct TimedLaunch {
    cudaEvent_t start, end;
  };
  struct TraceRec {
    tr_trace_event ev;
    TimedLaunch t;
  };
  struct DeviceCtx {
    int id = 0, gpu = 0, width = 4, max_inflight = 2;
    int sms = 148;  // multiprocessors this device runs on (split-K sizing, persistent grids)
    bool host_fills = false;  // the current job still fills tiles from host memory (see run_job)
    CUgreenCtx green = nullptr;  // sm_count > 0: the green context holding its SMs
    int green_sms = 0;
    int64_t capacity = -1;
    uint16_t* slab = nullptr;
    size_t slab_cap = 0;
    int32_t slab_slots = 0;  // directory slots allocated (physical = slab_slots + scratch)
    int32_t max_slots = 0;
    CUtensorMap tmap[4];
    std::vector<SlotState> slots;  // indexed by physical slot
    // [0, width): task streams (station entries); [width]: fill (convert) stream,
    // highest priority; [width+1]: copy stream (H2D into the staging ring, peer copies)
    std::vector<StreamCtx> streams;
    void* stage[kStage] = {};
    size_t stage_cap[kStage] = {};
    EvRef stage_free[kStage];
    uint64_t stage_next = 0;    std::unique_ptr<Station> station;
    tr_device_stats stats{};
    std::vector<TimedLaunch> timed, timed_pool;
    std::vector<TraceRec> trace;
    double last_kernel_ms = 0;
    int64_t pending_prefetch = 0;  // fetched-ahead tiles not yet claimed (this job)
    int64_t last_launches = 0;
    double last_span_ms = 0;
    cudaEvent_t span_start = nullptr, span_end = nullptr;
    std::thread worker;
  };

  // worker-side
  void worker_main(int d);
  void run_job(int d, Job& job);
  void issue(int d, Job& job, int64_t tid, int s);
  // simulated engine (TR_FLAG_SIM)
  void run_sim(Job& job);
  void sim_task(int d, Job& job, int64_t gtid, double t);
  double xfer_cost(int src, int dst, int64_t nbytes) const;
  void plan_split_k(int d, StreamCtx& sc, GemmArgs& args);
  void plan_split_small(int d, StreamCtx& sc, GemmArgs& args);
  bool plan_narrow(int d, StreamCtx& sc, GemmArgs& args, GemmArgs& t);
  void use_workspace(int d, StreamCtx& sc, GemmArgs& args, int splits, int64_t ws_ld);
  float* workspace(int d, StreamCtx& sc, size_t bytes);
  bool group_outbuf(int d, int s, size_t bytes);
  int group_split(int d, const GemmGroup& grp, bool pair) const;
  // write-through: reserve the cache slot for output tile (i, j) of p and point
  // args at its planes; returns the physical slot (-1: not written through)
  int32_t write_through(int d, int s, const Product& p, int64_t i, int64_t j, GemmArgs& args);
  // grouped launches: several ready tasks of one product in one K1 launch
  bool groupable(int d, Job& job, int64_t gtid);
  void issue_group(int d, Job& job, const std::vector<int64_t>& gtids, int s);
  // cold single-device products: k-panel schedule (see run_panels)
  bool panels_apply(const Job& job) const;
  bool run_panels(Job& job);  // false: no HBM for the C accumulators (nothing done)
  int max_group_ = -1;  // tasks per grouped launch (TR_GROUP env, default 4; 1 disables)
  int32_t acquire(int d, int s, Job& job, const Mat& src, uint64_t uid, bool transposed, int64_t r, int64_t c,
                  int scratch);
  void fill_slot(int d, int s, int32_t phys, const Mat& src, int64_t r, int64_t c);
  void load_slot(int d, int s, int32_t phys, HitLevel level, int32_t source, const TileKey& key, const Mat& src,
                 int64_t r, int64_t c, Job& job);
  void fetch_ahead(int d, Job& job, std::vector<uint8_t>& seen, std::vector<uint8_t>& seen_global,
                   int64_t& pending);
  bool prefetch_task(int d, Job& job, int64_t tid, bool host_only, int64_t& pending, int64_t budget);
  void wait_slot_free(int d, int s, int32_t phys);
  void wait_on(int d, int s, const EvRef& r);  // stream (d, s) waits for point r (unless same stream / complete)
  EvRef record(int d, int s);
  void note_use(SlotState& st, const EvRef& r);
  int32_t gs_of(int d, int s) const { return d * 64 + s; }
  void reap(int d, Job& job, bool block_oldest);
  // tracing (TR_FLAG_TRACE): bracket an async operation with timing events
  TimedLaunch timing_pair(int d);
  void trace_begin(int d, int s, TimedLaunch* t);
  void trace_end(int d, int s, TimedLaunch t, int kind, int64_t task, uint64_t uid, int64_t r, int64_t c);

  // session-side
  void ensure_slab(int d, int64_t needed);
  void build_tmaps(int d);
  void* lazy_tile(int d, void** p, size_t* cap);
  bool fuse_colsum(const Product& p, int64_t i, int64_t j, GemmArgs& args, bool small = false) const;
  void colsum_pass(const Product& p, int64_t i, int64_t j, cudaStream_t s);
  uint16_t* slot_ptr(int d, int32_t phys) const {
    return devs_[d].slab + static_cast<int64_t>(phys) * slot_elems_;
  }
  int32_t scratch_phys(int s, int which) const { return 2 * s + which; }
  int32_t phys_of(int d, int32_t dir_slot) const { return dir_slot + 2 * devs_[d].width; }

  int32_t tile_;
  int32_t precision_;
  bool exact_ = false;  // TR_PREC_EXACT: float64 tiles, the KX kernel only
  int planes_;
  int64_t ld_, plane_elems_, slot_elems_;
  uint32_t flags_;
  bool dryrun_, steal_, coherence_;
  int32_t element_bytes_;
  int64_t hbm_budget_;
  int order_ = -1;  // task enqueue order: 0 row-major, 1 banded, 2 shells, 3 blocked, 4 k-panels, -1 auto
  cudaStream_t ext_stream_ = nullptr;  // products start after the work queued here
  bool ext_on_ = false;                // ext_stream_ set (nullptr = the legacy default stream)
  bool async_ = false;                 // device-resident products return once enqueued (see run_products)
  // simulated engine: reference cost model (devices.py:255-283) and per-device
  // compute / transfer clocks that persist across calls (scheduler.py:416-429)
  bool sim_ = false;
  struct SimClock {
    double compute = 0.0, transfer = 0.0;
  };
  std::vector<SimClock> clocks_;
  std::vector<double> flops_, host_bw_, peer_bw_;
  std::vector<bool> host_worker_;
  double latency_ = 0.0;
  double last_makespan_ = 0.0;
  cudaEvent_t ext_ready_ = nullptr;
  bool tracing_ = false;
  std::vector<tr_trace_event> last_trace_;
  std::unique_ptr<Directory> dir_;
  std::vector<DeviceCtx> devs_;
  std::vector<Station*> station_ptrs_;
  std::vector<int64_t> peer_served_;  // L2 fills each device sourced in the current job (under dir_->mu)

  // worker coordination
  std::mutex mu_;
  std::condition_variable cv_;
  std::condition_variable cv_done_;
  uint64_t generation_ = 0;
  int workers_done_ = 0;
  bool shutdown_ = false;
  Job* job_ = nullptr;
};

}  // namespace tr
