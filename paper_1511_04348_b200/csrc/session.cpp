// GPU runtime session; see session.h for the mapping onto the reference.
#include "session.h"

#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <functional>
#include <queue>
#include <string>

#include "common.h"
#include "mlp_kernels.h"

namespace tr {

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// CPUs of the NUMA node the GPU's PCIe root hangs off (sysfs), empty when
// unknown (numa_node -1: one node, or a VM that hides it).
std::vector<int> gpu_local_cpus(int gpu) {
  std::vector<int> out;
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), gpu) != cudaSuccess) {
    cudaGetLastError();
    return out;
  }
  for (char* p = bus; *p; ++p) *p = static_cast<char>(tolower(*p));
  int node = -1;
  if (FILE* f = fopen((std::string("/sys/bus/pci/devices/") + bus + "/numa_node").c_str(), "r")) {
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
  }
  if (node < 0) return out;
  char list[4096] = {0};
  if (FILE* f = fopen(("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist").c_str(), "r")) {
    if (!fgets(list, sizeof(list), f)) list[0] = 0;
    fclose(f);
  }
  for (char* tok = strtok(list, ",\n"); tok; tok = strtok(nullptr, ",\n")) {  // "0-15,32-47"
    int a = -1, b = -1;
    if (sscanf(tok, "%d-%d", &a, &b) == 2)
      for (int c = a; c <= b; ++c) out.push_back(c);
    else if (sscanf(tok, "%d", &a) == 1)
      out.push_back(a);
  }
  return out;
}

// Pin device `index`'s worker to one core: of the GPU's NUMA node when sysfs
// names one (its host copies stay on the local memory controller), else of the
// whole allowed set; core 0 of the set stays with the calling (Python) thread.
void pin_thread_to_core(int index, int gpu) {
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof(allowed), &allowed) != 0) return;
  std::vector<int> cores, local;
  for (int c = 0; c < CPU_SETSIZE; ++c)
    if (CPU_ISSET(c, &allowed)) cores.push_back(c);
  if (gpu >= 0)
    for (int c : gpu_local_cpus(gpu))
      if (c < CPU_SETSIZE && CPU_ISSET(c, &allowed) && c != cores.front()) local.push_back(c);
  int core = -1;
  if (!local.empty()) core = local[static_cast<size_t>(index) % local.size()];
  else if (cores.size() >= 2) core = cores[1 + index % static_cast<int>(cores.size() - 1)];
  if (core < 0) return;
  cpu_set_t one;
  CPU_ZERO(&one);
  CPU_SET(core, &one);
  pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
}

// Driver entry points for green contexts (the library links the static runtime,
// not libcuda; cuTensorMapEncodeTiled is reached the same way).
template <typename Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    fail(TR_ERR_CUDA, "driver entry point %s unavailable", name);
  }
  return reinterpret_cast<Fn>(p);
}

void check_cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(TR_ERR_CUDA, "%s failed (CUresult %d)", what, static_cast<int>(r));
}

}  // namespace

void Job::mark(int64_t tid) {
  if (done[static_cast<size_t>(tid)].exchange(1) != 0) fail(TR_ERR_RUNTIME, "task %lld executed twice", (long long)tid);
  done_count.fetch_add(1);
}

void Job::set_error(int status, const std::string& msg) {
  std::lock_guard<std::mutex> g(mu);
  if (err_status == 0) {
    err_status = status;
    err_msg = msg;
  }
  abort.store(true);
}

// ---------------------------------------------------------------- construction
Session::Session(const tr_machine& m, int32_t tile, int32_t precision, uint32_t flags, int64_t hbm_budget)
    : tile_(tile), precision_(precision), flags_(flags), hbm_budget_(hbm_budget) {
  if (tile < 1) fail(TR_ERR_SHAPE, "tile_size must be >= 1, got %d", tile);
  if (precision != TR_PREC_BF16 && precision != TR_PREC_FP32ACC && precision != TR_PREC_EXACT &&
      precision != TR_PREC_FP32HI)
    fail(TR_ERR_VALUE, "unknown precision %d", precision);
  if (m.n_devices < 1 || m.n_devices > 64) fail(TR_ERR_CONFIG, "machine needs 1..64 devices, got %d", m.n_devices);
  sim_ = flags & TR_FLAG_SIM;
  max_group_ = task_group_max();
  // Inhomogeneous devices (green contexts of different sizes): smaller groups keep
  // a slow device from holding several tasks at once (tools/green/probe_green_1234.py).
  for (int d = 1; d < m.n_devices; ++d)
    if (m.devices[d].sm_count != m.devices[0].sm_count) max_group_ = std::min(max_group_, 2);
  dryrun_ = (flags & TR_FLAG_DRYRUN) || sim_;
  steal_ = flags & TR_FLAG_STEAL;
  coherence_ = flags & TR_FLAG_COHERENCE;
  tracing_ = (flags & TR_FLAG_TRACE) && !(flags & TR_FLAG_DRYRUN);
  element_bytes_ = m.element_bytes > 0 ? m.element_bytes : 8;
  // bf16: one bf16 plane; fp32acc: hi/lo planes; exact: the tile as float64 (4 planes' worth)
  exact_ = precision == TR_PREC_EXACT;
  planes_ = exact_ ? 4 : precision == TR_PREC_FP32HI ? 3 : precision == TR_PREC_FP32ACC ? 2 : 1;
  ld_ = ceil_div(tile, 8) * 8;
  plane_elems_ = static_cast<int64_t>(tile) * ld_;
  slot_elems_ = planes_ * plane_elems_;

  const int n = m.n_devices;
  std::vector<int64_t> caps(n), hops(static_cast<size_t>(n) * n);
  std::vector<bool> hw(n, false);
  for (int d = 0; d < n; ++d) {
    const tr_device_spec& ds = m.devices[d];
    if (ds.device_id != d) fail(TR_ERR_CONFIG, "device ids must be 0..%d in order", n - 1);
    if (ds.kind != TR_KIND_ACCELERATOR && !sim_)
      fail(TR_ERR_CONFIG, "device %d is a host-worker: the B200 runtime has no CPU compute path", d);
    hw[d] = ds.kind == TR_KIND_HOST_WORKER;
    if (ds.slots < 1 || ds.slots > 32) fail(TR_ERR_CONFIG, "device %d: slots must be in 1..32", d);
    caps[d] = ds.capacity_tiles;
    if (caps[d] >= 0 && caps[d] < 3) fail(TR_ERR_CONFIG, "capacity_tiles must be >= 3 (A+B+C working set)");
  }
  for (int64_t i = 0; i < static_cast<int64_t>(n) * n; ++i) hops[i] = m.hops ? m.hops[i] : (i % (n + 1) ? 1 : 0);
  if (sim_) {
    clocks_.assign(n, SimClock{});
    host_worker_ = hw;
    latency_ = m.transfer_latency;
    for (int d = 0; d < n; ++d) {
      const tr_device_spec& ds = m.devices[d];
      if (!(ds.flops_per_unit > 0) || (!hw[d] && !(ds.host_bandwidth > 0)))
        fail(TR_ERR_CONFIG, "device %d: flops_per_unit and host_bandwidth must be > 0", d);
      flops_.push_back(ds.flops_per_unit);
      host_bw_.push_back(ds.host_bandwidth);
    }
    peer_bw_.assign(static_cast<size_t>(n) * n, 0.0);
    for (int64_t i = 0; i < static_cast<int64_t>(n) * n; ++i) peer_bw_[i] = m.peer_bandwidth ? m.peer_bandwidth[i] : 0.0;
  }
  dir_ = std::make_unique<Directory>(n, caps, hw, hops, coherence_, (flags & TR_FLAG_FIFO) ? TR_POLICY_FIFO : TR_POLICY_LRU,
                                     (flags & TR_FLAG_DEBUG) != 0);

  int n_gpus = 0;
  if (!dryrun_) {
    cudaError_t e = cudaGetDeviceCount(&n_gpus);
    if (e != cudaSuccess || n_gpus < 1) {
      cudaGetLastError();
      fail(TR_ERR_NODEVICE, "no CUDA device available (%s): the tile GEMM runs only on the GPU",
           e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    }
  }
  devs_.resize(n);
  std::vector<int> per_gpu(std::max(n_gpus, 1), 0);
  for (int d = 0; d < n; ++d) {
    DeviceCtx& dc = devs_[d];
    dc.id = d;
    dc.width = m.devices[d].slots;
    dc.max_inflight = std::min(dc.width, 2);
    dc.capacity = caps[d];
    dc.gpu = dryrun_ ? 0 : (m.devices[d].gpu >= 0 ? m.devices[d].gpu : d % n_gpus);
    if (!dryrun_ && dc.gpu >= n_gpus) fail(TR_ERR_CONFIG, "device %d maps to GPU %d but only %d visible", d, dc.gpu, n_gpus);
    per_gpu[dc.gpu] += 1;
    dc.station = std::make_unique<Station>(d, dc.width);
    station_ptrs_.push_back(dc.station.get());
  }
  const bool tdebug = getenv("TR_TIMING") != nullptr;  // session set-up timing on stderr
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  if (!dryrun_) {
    // Inhomogeneous devices: a logical device with sm_count > 0 runs on a green
    // context holding that many SMs of its GPU.  A GPU's SMs are split once into
    // groups of the hardware granularity (8 SMs on B200; the remainder of a
    // split cannot be split again), and its such devices take ceil(count / 8)
    // consecutive groups each, in device-id order -- disjoint SM sets.
    constexpr unsigned kSmGroup = 8;
    std::vector<std::vector<CUdevResource>> sm_groups(static_cast<size_t>(std::max(n_gpus, 1)));
    std::vector<size_t> sm_next(sm_groups.size(), 0);
    for (int d = 0; d < n; ++d) {
      const int want = m.devices[d].sm_count;
      if (want <= 0) continue;
      DeviceCtx& dc = devs_[d];
      TR_CUDA(cudaSetDevice(dc.gpu));
      TR_CUDA(cudaFree(nullptr));  // the primary context exists before the green one
      CUdevice cudev;
      check_cu(driver_fn<decltype(&cuDeviceGet)>("cuDeviceGet")(&cudev, dc.gpu), "cuDeviceGet");
      auto& pool = sm_groups[dc.gpu];
      if (pool.empty()) {
        CUdevResource all, rest;
        check_cu(driver_fn<decltype(&cuDeviceGetDevResource)>("cuDeviceGetDevResource")(cudev, &all,
                                                                                       CU_DEV_RESOURCE_TYPE_SM),
                 "cuDeviceGetDevResource");
        unsigned n_groups = all.sm.smCount / kSmGroup;
        pool.resize(n_groups);
        check_cu(driver_fn<decltype(&cuDevSmResourceSplitByCount)>("cuDevSmResourceSplitByCount")(
                     pool.data(), &n_groups, &all, &rest, 0, kSmGroup),
                 "cuDevSmResourceSplitByCount");
        pool.resize(n_groups);
      }
      const size_t take = (static_cast<size_t>(want) + kSmGroup - 1) / kSmGroup;
      if (sm_next[dc.gpu] + take > pool.size())
        fail(TR_ERR_CONFIG, "device %d: GPU %d has only %zu of the %zu SM groups of %u requested", d, dc.gpu,
             pool.size() - sm_next[dc.gpu], take, kSmGroup);
      CUdevResourceDesc desc;
      check_cu(driver_fn<decltype(&cuDevResourceGenerateDesc)>("cuDevResourceGenerateDesc")(
                   &desc, pool.data() + sm_next[dc.gpu], static_cast<unsigned>(take)),
               "cuDevResourceGenerateDesc");
      dc.green_sms = 0;
      for (size_t k = 0; k < take; ++k) dc.green_sms += static_cast<int>(pool[sm_next[dc.gpu] + k].sm.smCount);
      sm_next[dc.gpu] += take;
      check_cu(driver_fn<decltype(&cuGreenCtxCreate)>("cuGreenCtxCreate")(&dc.green, desc, cudev,
                                                                           CU_GREEN_CTX_DEFAULT_STREAM),
               "cuGreenCtxCreate");
    }
    for (int d = 0; d < n; ++d) {
      DeviceCtx& dc = devs_[d];
      const auto q0 = tnow();
      TR_CUDA(cudaSetDevice(dc.gpu));
      TR_CUDA(cudaDeviceGetAttribute(&dc.sms, cudaDevAttrMultiProcessorCount, dc.gpu));
      if (dc.green) dc.sms = dc.green_sms;
      die_map_prepare(dc.gpu);  // once per GPU and process: K1's die-aware unit order
      size_t free_b = 0;
      TR_CUDA(DevPool::get().free_bytes(dc.gpu, &free_b));
      const double reusable = static_cast<double>(free_b) + static_cast<double>(DevPool::get().cached_bytes());
      int64_t budget = hbm_budget_ > 0 ? hbm_budget_ : static_cast<int64_t>(0.8 * reusable);
      budget /= per_gpu[dc.gpu];
      const int64_t tile_bytes = static_cast<int64_t>(tile) * tile * 8;
      const int64_t slot_bytes = slot_elems_ * 2;
      // stage ring + lazy tiles + the grouped launches' host-output buffers (one per
      // concurrently used compute stream, max_group fp32 tiles each)
      const int64_t gout_bytes = static_cast<int64_t>(std::min(dc.width, 2)) * std::min(max_group_, kMaxGroup) *
                                 static_cast<int64_t>(tile) * tile * 4;
      int64_t avail = budget - static_cast<int64_t>(kStage + 2) * tile_bytes - gout_bytes;
      int64_t slots = avail / slot_bytes - 2 * dc.width;
      slots = std::min<int64_t>(slots, int64_t(1) << 22);
      if (dc.capacity >= 0) slots = std::min<int64_t>(slots, dc.capacity);
      if (slots < 2) fail(TR_ERR_CAPACITY, "device %d: HBM budget too small for tile size %d", d, tile);
      dc.max_slots = static_cast<int32_t>(slots);
      const auto q1 = tnow();
      // + fill (convert) stream [width] + copy stream [width+1] + writeback stream [width+2]
      dc.streams.resize(dc.width + 3);
      TR_CUDA(cudaEventCreate(&dc.span_start));
      TR_CUDA(cudaEventCreate(&dc.span_end));
      int prio_low = 0, prio_high = 0;
      TR_CUDA(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
      for (size_t si = 0; si < dc.streams.size(); ++si) {
        StreamCtx& sc = dc.streams[si];
        // the fill stream runs at the highest priority: its split/convert kernels
        // must not queue behind GEMM CTAs that occupy every SM
        const int prio = static_cast<int>(si) == dc.width ? prio_high : prio_low;
        if (dc.green) {
          CUstream cs;
          check_cu(driver_fn<decltype(&cuGreenCtxStreamCreate)>("cuGreenCtxStreamCreate")(
                       &cs, dc.green, CU_STREAM_NON_BLOCKING, prio), "cuGreenCtxStreamCreate");
          sc.stream = reinterpret_cast<cudaStream_t>(cs);
        } else {
          TR_CUDA(cudaStreamCreateWithPriority(&sc.stream, cudaStreamNonBlocking, prio));
        }
        TR_CUDA(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming));
        // per-stream staging / output tiles are allocated on first use (lazy_tile):
        // bypass-mode fills and host outputs of single-task launches only
      }
      if (tdebug)
        fprintf(stderr, "[tr] session dev %d: meminfo %.2f ms, streams+buffers %.2f ms, budget %.2f GB, max slots %d\n", d,
                tms(q0, q1), tms(q1, tnow()), budget / 1e9, dc.max_slots);
    }
    // Peer access between every pair of distinct GPUs in use (NVLink / NVSwitch).
    for (int d = 0; d < n; ++d) {
      for (int o = 0; o < n; ++o) {
        const int g = devs_[d].gpu, h = devs_[o].gpu;
        if (g == h) continue;
        int can = 0;
        TR_CUDA(cudaDeviceCanAccessPeer(&can, g, h));
        if (!can) continue;
        TR_CUDA(cudaSetDevice(g));
        cudaError_t e = cudaDeviceEnablePeerAccess(h, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else TR_CUDA(e);
      }
    }
  }
  const auto q2 = tnow();
  for (int d = 0; d < n; ++d) devs_[d].worker = std::thread(&Session::worker_main, this, d);
  if (tdebug) fprintf(stderr, "[tr] session threads %.2f ms\n", tms(q2, tnow()));
}

Session::~Session() {
  {
    std::lock_guard<std::mutex> g(mu_);
    shutdown_ = true;
  }
  cv_.notify_all();
  for (auto& dc : devs_)
    if (dc.worker.joinable()) dc.worker.join();
  if (dryrun_) return;
  for (auto& dc : devs_) {
    cudaSetDevice(dc.gpu);
    cudaDeviceSynchronize();
    for (auto& sc : dc.streams) {
      for (auto& ev : sc.evs) cudaEventDestroy(ev);
      cudaEventDestroy(sc.done);
      DevPool::get().release(dc.gpu, sc.staging, sc.staging_cap);
      DevPool::get().release(dc.gpu, sc.outbuf, sc.outbuf_cap);
      if (sc.ws) DevPool::get().release(dc.gpu, sc.ws, sc.ws_cap);
      if (sc.gout) DevPool::get().release(dc.gpu, sc.gout, sc.gout_cap);
      cudaStreamDestroy(sc.stream);
    }
    for (auto& t : dc.timed) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.end);
    }
    for (auto& t : dc.timed_pool) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.end);
    }
    if (dc.green) driver_fn<decltype(&cuGreenCtxDestroy)>("cuGreenCtxDestroy")(dc.green);  // after its streams
    DevPool::get().release(dc.gpu, dc.slab, dc.slab_cap);
    for (int k = 0; k < kStage; ++k) DevPool::get().release(dc.gpu, dc.stage[k], dc.stage_cap[k]);
    cudaEventDestroy(dc.span_start);
    cudaEventDestroy(dc.span_end);
  }
  if (ext_ready_) cudaEventDestroy(ext_ready_);
}

// A tile-sized device buffer (T x T doubles), allocated on first use.
void* Session::lazy_tile(int d, void** p, size_t* cap) {
  if (!*p) TR_CUDA(DevPool::get().alloc(devs_[d].gpu, static_cast<size_t>(tile_) * tile_ * 8, p, cap));
  return *p;
}

// ---------------------------------------------------------------- HBM slab
void Session::build_tmaps(int d) {
  DeviceCtx& dc = devs_[d];
  PlaneGeom g;
  g.base = dc.slab;
  g.cols = tile_;
  g.rows = tile_;
  g.nplanes = static_cast<int64_t>(dc.slab_slots + 2 * dc.width) * planes_;
  g.ld = ld_;
  g.plane_stride = plane_elems_;
  for (int b = 0; b < 4; ++b) {
    const int r = make_plane_tmap(&dc.tmap[b], g, static_cast<BoxKind>(b));
    if (r != 0) fail(TR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for device %d", r, d);
  }
}

void Session::ensure_slab(int d, int64_t needed) {
  DeviceCtx& dc = devs_[d];
  const int64_t target = std::min<int64_t>(dc.max_slots, std::max<int64_t>(needed, 1));
  if (target <= dc.slab_slots) return;
  int64_t grow = std::min<int64_t>(dc.max_slots, std::max<int64_t>(target, 2 * static_cast<int64_t>(dc.slab_slots)));
  const int64_t scratch = 2 * dc.width;
  TR_CUDA(cudaSetDevice(dc.gpu));
  TR_CUDA(cudaDeviceSynchronize());
  uint16_t* nb = nullptr;
  size_t cap = 0;
  cudaError_t e = DevPool::get().alloc(dc.gpu, static_cast<size_t>((grow + scratch) * slot_elems_ * 2),
                                       reinterpret_cast<void**>(&nb), &cap);
  if (e != cudaSuccess && grow > target) {
    grow = target;
    e = DevPool::get().alloc(dc.gpu, static_cast<size_t>((grow + scratch) * slot_elems_ * 2),
                             reinterpret_cast<void**>(&nb), &cap);
  }
  // HBM taken since the budget was set (other logical devices of this GPU, the
  // caller's tensors): settle for the largest growth that still fits
  for (int64_t lo = dc.slab_slots; e != cudaSuccess && grow - lo > 8;) {
    grow = lo + (grow - lo) / 2;
    e = DevPool::get().alloc(dc.gpu, static_cast<size_t>((grow + scratch) * slot_elems_ * 2),
                             reinterpret_cast<void**>(&nb), &cap);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    // a slab that cannot grow still serves the job: the directory evicts into it
    if (dc.slab_slots >= 3) {
      if (getenv("TR_TIMING"))
        fprintf(stderr, "[tr] device %d: slab stays at %d slots (growth to %lld failed: %s)\n", d, dc.slab_slots,
                (long long)grow, cudaGetErrorString(e));
      return;
    }
    fail(TR_ERR_CAPACITY, "device %d: cannot allocate a %lld-slot tile slab (%s)", d, (long long)grow,
         cudaGetErrorString(e));
  }
  if (dc.slab) {
    TR_CUDA(cudaMemcpy(nb, dc.slab, static_cast<size_t>((dc.slab_slots + scratch) * slot_elems_ * 2),
                       cudaMemcpyDeviceToDevice));
    DevPool::get().release(dc.gpu, dc.slab, dc.slab_cap);
  }
  dc.slab_cap = cap;
  dc.slab = nb;
  dc.slab_slots = static_cast<int32_t>(grow);
  dc.slots.resize(static_cast<size_t>(grow + scratch));
  {
    DirLock g(dir_->mu);
    dir_->attach_slots(d, dc.slab_slots);
  }
  build_tmaps(d);
}

// ---------------------------------------------------------------- events / ordering
Session::EvRef Session::record(int d, int s) {
  StreamCtx& sc = devs_[d].streams[s];
  int32_t idx = -1;
  if (!sc.fifo.empty()) {
    const cudaError_t q = cudaEventQuery(sc.evs[sc.fifo.front()]);
    if (q == cudaSuccess) {
      idx = sc.fifo.front();
      sc.fifo.pop_front();
    } else if (q != cudaErrorNotReady) {
      TR_CUDA(q);
    }
  }
  if (idx < 0) {
    cudaEvent_t ev;
    TR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    idx = static_cast<int32_t>(sc.evs.size());
    sc.evs.push_back(ev);
    sc.gen.push_back(0);
  }
  sc.gen[idx] += 1;
  TR_CUDA(cudaEventRecord(sc.evs[idx], sc.stream));
  sc.fifo.push_back(idx);
  return EvRef{gs_of(d, s), idx, sc.gen[idx]};
}

void Session::wait_on(int d, int s, const EvRef& r) {
  if (r.gs < 0 || r.gs == gs_of(d, s)) return;  // none, or same stream: already ordered
  StreamCtx& src = devs_[r.gs / 64].streams[r.gs % 64];
  if (src.gen[r.idx] != r.gen) return;  // the event was recycled: that point completed
  TR_CUDA(cudaStreamWaitEvent(devs_[d].streams[s].stream, src.evs[r.idx], 0));
}

Session::TimedLaunch Session::timing_pair(int d) {
  DeviceCtx& dc = devs_[d];
  TimedLaunch tl;
  if (!dc.timed_pool.empty()) {
    tl = dc.timed_pool.back();
    dc.timed_pool.pop_back();
  } else {
    TR_CUDA(cudaEventCreate(&tl.start));
    TR_CUDA(cudaEventCreate(&tl.end));
  }
  return tl;
}

void Session::trace_begin(int d, int s, TimedLaunch* t) {
  if (!tracing_) return;
  *t = timing_pair(d);
  TR_CUDA(cudaEventRecord(t->start, devs_[d].streams[s].stream));
}

void Session::trace_end(int d, int s, TimedLaunch t, int kind, int64_t task, uint64_t uid, int64_t r, int64_t c) {
  if (!tracing_) return;
  TR_CUDA(cudaEventRecord(t.end, devs_[d].streams[s].stream));
  TraceRec rec;
  rec.ev = tr_trace_event{d, kind, s, task, uid, r, c, 0.0, 0.0};
  rec.t = t;
  devs_[d].trace.push_back(rec);
}

void Session::note_use(SlotState& st, const EvRef& r) {
  for (auto& u : st.uses)
    if (u.gs == r.gs) {
      u = r;
      return;
    }
  st.uses.push_back(r);
}

// Before overwriting physical slot `phys` of device d from stream s: every other
// stream that read it (kernels, peer copies) or is still filling it must be done.
void Session::wait_slot_free(int d, int s, int32_t phys) {
  SlotState& st = devs_[d].slots[phys];
  wait_on(d, s, st.ready);
  for (auto& u : st.uses) wait_on(d, s, u);
}

// Miss path: host (pinned) -> staging -> split/convert into the slot, or
// device matrix -> split/convert directly.
void Session::fill_slot(int d, int s, int32_t phys, const Mat& src, int64_t r, int64_t c) {
  DeviceCtx& dc = devs_[d];
  StreamCtx& sc = dc.streams[s];
  const int64_t T = tile_;
  const int64_t tr_ = std::min(T, src.rows - r * T);
  const int64_t tc = std::min(T, src.cols - c * T);
  const int64_t es = src.esize();
  const char* base = static_cast<const char*>(src.ptr) + (r * T * src.ld + c * T) * es;
  const void* conv_src = base;
  int64_t conv_ld = src.ld;
  if (src.location == TR_LOC_HOST) {
    lazy_tile(d, &sc.staging, &sc.staging_cap);
    TR_CUDA(cudaMemcpy2DAsync(sc.staging, tc * es, base, src.ld * es, tc * es, tr_, cudaMemcpyHostToDevice, sc.stream));
    conv_src = sc.staging;
    conv_ld = tc;
  }
  TR_CUDA(launch_split_convert(conv_src, src.dtype == TR_DTYPE_F64, conv_ld, tr_, tc, slot_ptr(d, phys), ld_, T,
                               plane_elems_, planes_, sc.stream));
}

// One input tile for device d, task stream s: directory accounting exactly as
// coherence.py:210-246, then the physical action for the hit level.
int32_t Session::acquire(int d, int s, Job& job, const Mat& src, uint64_t uid, bool transposed, int64_t r,
                         int64_t c, int scratch) {
  // r, c are STORED coordinates of the tile (Operand.key, scheduler.py:132-134)
  (void)transposed;
  const int64_t T = tile_;
  const int64_t nbytes = std::min(T, src.rows - r * T) * std::min(T, src.cols - c * T) * element_bytes_;
  const TileKey key{uid, r, c};
  const int32_t gs = gs_of(d, s);
  DirLock g(dir_->mu);
  Acquired a = dir_->acquire_input_locked(d, key, nbytes);
  if (dryrun_) return a.slot;
  if (!coherence_) {
    // bypass (coherence.py:220-225): every request is a host fetch into a per-stream scratch slot
    const int32_t phys = scratch_phys(s, scratch);
    fill_slot(d, s, phys, src, r, c);
    job.launches.fetch_add(1);
    return phys;
  }
  DeviceCtx& dc = devs_[d];
  const int32_t phys = phys_of(d, a.slot);
  SlotState& st = dc.slots[phys];
  if (a.prefetched && dc.pending_prefetch > 0) dc.pending_prefetch -= 1;  // claimed a fetched-ahead tile
  if (a.level == HIT_L1 || a.prefetched) {
    // resident (possibly still being filled ahead of time on another stream)
    wait_on(d, s, st.ready);
    return phys;
  }
  // every fill runs on the device's fill/copy streams; the task's stream waits for it
  load_slot(d, dc.width, phys, a.phys_source >= 0 ? HIT_L2 : HIT_MISS, a.phys_source, key, src, r, c, job);
  wait_on(d, s, st.ready);
  return phys;
}

// Physical side of an L2 hit (peer copy of the converted planes) or a miss
// (host H2D + split/convert, or device-matrix split/convert) into slot `phys`
// of device d, on stream s.  Caller holds the directory lock.
void Session::load_slot(int d, int /*task stream*/, int32_t phys, HitLevel level, int32_t source,
                        const TileKey& key, const Mat& src, int64_t r, int64_t c, Job& job) {
  NvtxRange nv(level == HIT_L2 ? "tr.fill peer" : "tr.fill host");
  DeviceCtx& dc = devs_[d];
  SlotState& st = dc.slots[phys];
  const int F = dc.width;      // high-priority convert stream (writes slots)
  const int X = dc.width + 1;  // copy stream (DMA only)
  if (level == HIT_L2) {
    // peer copy of the already-converted planes, on the copy stream
    wait_slot_free(d, X, phys);
    // load-aware source: the directory's closest owner (the reference's choice)
    // unless another equally close owner has served fewer copies in this job
    int o = dir_->balanced_source_locked(d, key, peer_served_);
    if (o < 0) o = source;
    peer_served_[o] += 1;
    devs_[o].stats.peer_copies_served += 1;
    const int32_t src_phys = phys_of(o, dir_->slot_of_locked(o, key));
    SlotState& ss = devs_[o].slots[src_phys];
    wait_on(d, X, ss.ready);
    const size_t bytes = static_cast<size_t>(slot_elems_ * 2);
    cudaStream_t xs = dc.streams[X].stream;
    TimedLaunch tt{};
    trace_begin(d, X, &tt);
    // TR_FORCE_PEER_COPY=1: the cross-GPU call even between logical devices of one
    // GPU, so single-GPU tests exercise the multi-GPU fill path
    static const bool force_peer = getenv("TR_FORCE_PEER_COPY") && getenv("TR_FORCE_PEER_COPY")[0] == '1';
    if (devs_[o].gpu == dc.gpu && !force_peer) {
      TR_CUDA(cudaMemcpyAsync(slot_ptr(d, phys), slot_ptr(o, src_phys), bytes, cudaMemcpyDeviceToDevice, xs));
    } else {
      TR_CUDA(cudaMemcpyPeerAsync(slot_ptr(d, phys), dc.gpu, slot_ptr(o, src_phys), devs_[o].gpu, bytes, xs));
    }
    trace_end(d, X, tt, TR_TRACE_PEER, -1, key.matrix, key.row, key.col);
    const EvRef ev = record(d, X);
    note_use(ss, ev);  // the source cannot be refilled under the copy
    st.ready = ev;
    st.uses.clear();
    return;
  }
  const int64_t T = tile_;
  const int64_t tr_ = std::min(T, src.rows - r * T);
  const int64_t tc = std::min(T, src.cols - c * T);
  const int64_t es = src.esize();
  const char* base = static_cast<const char*>(src.ptr) + (r * T * src.ld + c * T) * es;
  cudaStream_t fs = dc.streams[F].stream;
  wait_slot_free(d, F, phys);
  if (src.location == TR_LOC_HOST) {
    // H2D into the next staging buffer of the ring on the copy stream; the
    // convert follows on the fill stream.  The DMA engine runs up to kStage
    // tiles ahead of the converts (which may wait for SMs busy with GEMMs).
    const int k = static_cast<int>(dc.stage_next++ % kStage);
    lazy_tile(d, &dc.stage[k], &dc.stage_cap[k]);
    cudaStream_t xs = dc.streams[X].stream;
    wait_on(d, X, dc.stage_free[k]);
    TimedLaunch tc1{}, tc2{};
    trace_begin(d, X, &tc1);
    TR_CUDA(cudaMemcpy2DAsync(dc.stage[k], tc * es, base, src.ld * es, tc * es, tr_, cudaMemcpyHostToDevice, xs));
    trace_end(d, X, tc1, TR_TRACE_H2D, -1, key.matrix, key.row, key.col);
    wait_on(d, F, record(d, X));  // convert after the copy landed
    trace_begin(d, F, &tc2);
    TR_CUDA(launch_split_convert(dc.stage[k], src.dtype == TR_DTYPE_F64, tc, tr_, tc, slot_ptr(d, phys), ld_, T,
                                 plane_elems_, planes_, fs));
    trace_end(d, F, tc2, TR_TRACE_CONVERT, -1, key.matrix, key.row, key.col);
    dc.stage_free[k] = record(d, F);
  } else {
    TimedLaunch tc2{};
    trace_begin(d, F, &tc2);
    TR_CUDA(launch_split_convert(base, src.dtype == TR_DTYPE_F64, src.ld, tr_, tc, slot_ptr(d, phys), ld_, T,
                                 plane_elems_, planes_, fs));
    trace_end(d, F, tc2, TR_TRACE_CONVERT, -1, key.matrix, key.row, key.col);
  }
  job.launches.fetch_add(1);
  st.ready = record(d, F);
  st.uses.clear();
}

// Prefetch every input tile of task `tid` that is not yet resident on device d
// (see fetch_ahead).  host_only: only tiles resident nowhere (another device
// holding a tile serves it over NVLink when actually needed).  Stops once
// `pending` reaches `budget`.
bool Session::prefetch_task(int d, Job& job, int64_t gtid, bool host_only, int64_t& pending, int64_t budget) {
  const int s = devs_[d].width;  // the fill stream
  int64_t tid = 0;
  const Product& p = job.prod_of(gtid, &tid);
  const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
  for (int64_t k = 0; k < p.k_steps; ++k) {
    for (int which = 0; which < 2; ++which) {
      if (pending >= budget) return false;
      const Mat& m = which == 0 ? p.a : p.b;
      const uint64_t uid = which == 0 ? p.a_uid : p.b_uid;
      const bool t = which == 0 ? p.ta : p.tb;
      const int64_t r = which == 0 ? (t ? k : i) : (t ? j : k);
      const int64_t c = which == 0 ? (t ? i : k) : (t ? k : j);
      const TileKey key{uid, r, c};
      DirLock g(dir_->mu);
      int32_t slot = -1, source = TR_SOURCE_HOST;
      if (!dir_->prefetch_locked(d, key, &slot, &source, host_only)) continue;
      load_slot(d, s, phys_of(d, slot), source >= 0 ? HIT_L2 : HIT_MISS, source, key, m, r, c, job);
      ++pending;
    }
  }
  return true;
}

// Fetch-ahead ("threaded fetch-ahead", absent from the
// reference's code).  Two windows: (1) every input tile of the tasks this device
// has RESERVED; (2) a bounded lookahead over the planned order just past the
// queue head, for tiles resident nowhere -- this keeps the H2D engine busy
// through the first-touch phase, when each new task needs several new panels.
// Directory::prefetch_locked never evicts and never counts, so the counters are
// exactly the reference's.  `pending` counts this device's fetched-ahead tiles
// not yet claimed by one of its tasks.
void Session::fetch_ahead(int d, Job& job, std::vector<uint8_t>& seen, std::vector<uint8_t>& seen_global,
                          int64_t& pending) {
  DeviceCtx& dc = devs_[d];
  // unclaimed prefetched tiles per device / tasks looked ahead past the queue
  // head; out-of-core jobs look further (the next task block's panels).  Long
  // contractions (cfg4: 32 k-steps) need two tasks' panels in flight: a new
  // shell's first task brings a whole row panel (k tiles) before it can run.
  int64_t max_ks = 0;
  for (const Product& p : job.prods) max_ks = std::max<int64_t>(max_ks, p.k_steps);
  // never more than a third of the device's slab: unclaimed tiles cannot be evicted
  const int64_t kBudget = std::min<int64_t>(std::max<int64_t>(job.out_of_core ? 96 : 32, 4 * max_ks),
                                            std::max<int64_t>(1, dc.slab_slots / 3));
  const int64_t kLookahead = job.out_of_core ? 48 : 16;
  for (uint64_t tid : dc.station->peek()) {
    if (seen[tid]) continue;
    if (!prefetch_task(d, job, static_cast<int64_t>(tid), false, pending, kBudget)) return;
    seen[tid] = 1;
  }
  const int64_t head = job.claimed.load();
  const int64_t end = std::min<int64_t>(static_cast<int64_t>(job.order.size()), head + kLookahead);
  for (int64_t pos = head; pos < end; ++pos) {
    const int64_t tid = job.order[static_cast<size_t>(pos)];
    if (seen_global[tid]) continue;
    if (!prefetch_task(d, job, tid, true, pending, kBudget)) return;
    seen_global[tid] = 1;
  }
}

// ---------------------------------------------------------------- split-K
// A launch whose output tile has fewer 128 x 256 blocks than the GPU has SMs
// (skinny MLP layers: N = 10, K = 784 edges) is split along K so that about
// two waves of CTAs run; partials go to the stream's workspace and a reduction
// kernel sums them in a fixed order (deterministic) and applies the epilogue.
// K-splits for a launch of `ctas` output blocks over `total_kb` k-blocks: about
// two waves of CTAs, at most splitk_max(), each split >= 8 k-blocks; 1 = no split.
int split_factor(int64_t ctas, int total_kb, int64_t sms) {
  const int smax = splitk_max();
  if (smax < 2 || ctas >= sms) return 1;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({2 * sms / ctas, smax, total_kb / 8})));
}

void Session::plan_split_k(int d, StreamCtx& sc, GemmArgs& args) {
  args.k_split = 1;
  int total_kb = 0;
  for (int k = 0; k < args.n_ksteps; ++k) total_kb += (args.k_len[k] + 63) / 64;
  const int64_t ctas = ((args.m_valid + 127) / 128) * static_cast<int64_t>((args.n_valid + 255) / 256);
  const int s = split_factor(ctas, total_kb, devs_[d].sms);
  if (s >= 2) use_workspace(d, sc, args, s, (args.n_valid + 255) / 256 * 256);
}

// A narrow task on the tensor cores (tile_gemm.h, narrow_tc): t is the
// transposed product P = Bᵀ·Aᵀ (operand planes swapped, raw fp32 out) split
// along k to about two waves of CTAs; args gets P's partials (args.ws, ws_ld,
// ws_zstride, k_split) for launch_splitk_reduce_t.  False without workspace.
bool Session::plan_narrow(int d, StreamCtx& sc, GemmArgs& args, GemmArgs& t) {
  t = args;
  t.m_valid = args.n_valid;
  t.n_valid = args.m_valid;
  int kb = 0;
  for (int k = 0; k < args.n_ksteps; ++k) {
    t.a_z[k] = args.b_z[k];
    t.b_z[k] = args.a_z[k];
    kb += (args.k_len[k] + 63) / 64;
  }
  t.c_f64 = 0;
  t.epilogue = EPI_STORE;
  t.post = POST_NONE;
  t.scaled = 0;
  t.bias = nullptr;
  t.aux = nullptr;
  t.wt = nullptr;
  const int64_t ctas = ceil_div(t.n_valid, 256);  // P has <= 32 rows: one 128-row block
  // narrow tiles split up to 16 ways; a lower TR_SPLITK / set_splitk limit is honoured
  const int64_t cap = splitk_max() >= 8 ? 16 : splitk_max();
  int splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({ceil_div(2 * devs_[d].sms, ctas), cap, kb / 8})));
  const int64_t ws_ld = (t.n_valid + 255) / 256 * 256;
  const int64_t zstride = static_cast<int64_t>(t.m_valid) * ws_ld;
  float* ws = workspace(d, sc, static_cast<size_t>(splits * zstride) * sizeof(float));
  if (!ws) return false;
  if (splits > 1) {
    t.k_split = splits;
    t.ws = ws;
    t.ws_ld = ws_ld;
    t.ws_zstride = zstride;
    t.c = nullptr;
  } else {  // one share: P is stored straight into the workspace
    t.k_split = 1;
    t.c = ws;
    t.ldc = ws_ld;
  }
  args.k_split = splits;
  args.ws = ws;
  args.ws_ld = ws_ld;
  args.ws_zstride = zstride;
  return true;
}

// The CUDA-core kernel's split: ~4 CTAs per SM for a narrow tile's long k.
void Session::plan_split_small(int d, StreamCtx& sc, GemmArgs& args) {
  args.k_split = 1;
  const int s = small_gemm_split(args, static_cast<int>(devs_[d].sms));
  if (s >= 2) use_workspace(d, sc, args, s, (args.n_valid + 15) / 16 * 16);
}

// Points args at stream s's split-K workspace (grown on demand) for `splits`
// partials of ws_ld-wide rows; leaves the launch unsplit when HBM is short.
void Session::use_workspace(int d, StreamCtx& sc, GemmArgs& args, int splits, int64_t ws_ld) {
  const int64_t zstride = static_cast<int64_t>(args.m_valid) * ws_ld;
  float* ws = workspace(d, sc, static_cast<size_t>(splits * zstride) * sizeof(float));
  if (!ws) return;  // no room: run unsplit
  args.k_split = splits;
  args.ws = ws;
  args.ws_ld = ws_ld;
  args.ws_zstride = zstride;
}

// Stream s's split-K workspace, grown to >= bytes (nullptr when HBM is short).
float* Session::workspace(int d, StreamCtx& sc, size_t bytes) {
  if (bytes > sc.ws_cap) {
    DeviceCtx& dc = devs_[d];
    if (sc.ws) {
      TR_CUDA(cudaStreamSynchronize(sc.stream));  // the old workspace may still be read
      DevPool::get().release(dc.gpu, sc.ws, sc.ws_cap);
      sc.ws = nullptr;
      sc.ws_cap = 0;
    }
    void* p = nullptr;
    size_t cap = 0;
    if (DevPool::get().alloc(dc.gpu, bytes, &p, &cap) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    sc.ws = static_cast<float*>(p);
    sc.ws_cap = cap;
  }
  return sc.ws;
}

// Stream s's C tiles for a grouped launch with host outputs, grown to >= bytes
// (false when HBM is short: the tasks then run one launch each).
bool Session::group_outbuf(int d, int s, size_t bytes) {
  StreamCtx& sc = devs_[d].streams[s];
  if (bytes <= sc.gout_cap) return true;
  DeviceCtx& dc = devs_[d];
  if (sc.gout) {
    // earlier launches (this stream) and their writebacks (the writeback stream) may
    // still use it; other logical devices sharing the GPU are not stalled
    TR_CUDA(cudaStreamSynchronize(sc.stream));
    TR_CUDA(cudaStreamSynchronize(dc.streams[dc.width + 2].stream));
    DevPool::get().release(dc.gpu, sc.gout, sc.gout_cap);
    sc.gout = nullptr;
    sc.gout_cap = 0;
  }
  if (DevPool::get().alloc(dc.gpu, bytes, &sc.gout, &sc.gout_cap) != cudaSuccess) {
    cudaGetLastError();
    sc.gout = nullptr;
    sc.gout_cap = 0;
    return false;
  }
  return true;
}

// Split-K for a grouped launch: the k-share count s that minimises the
// estimated time -- the persistent grid's waves (tiles * s units over the
// device's CTA (pair) slots, each 1/s of the k-loop) plus the partials'
// round trip through HBM (written by the kernel, read by the reduction: 2 * s
// fp32 output tiles) -- when that beats the unsplit launch by 10 %.
int Session::group_split(int d, const GemmGroup& grp, bool pair) const {
  const int smax = splitk_max();
  if (smax < 2) return 1;
  const int cg = pair ? 2 : 1;
  int64_t tiles = 0;
  double out_bytes = 0;
  int kb = 1 << 30;
  for (int t = 0; t < grp.n_tasks; ++t) {
    const GemmArgs& a = grp.task[t];
    tiles += ceil_div(a.m_valid, 128 * cg) * ceil_div(a.n_valid, 256);
    out_bytes += 4.0 * a.m_valid * ((a.n_valid + 255) / 256 * 256);
    int k = 0;
    for (int q = 0; q < a.n_ksteps; ++q) k += (a.k_len[q] + 63) / 64;
    kb = std::min(kb, k);
  }
  const int64_t slots = std::max<int64_t>(1, devs_[d].sms / cg);
  // time of one unit's full k-loop (µs; ~1.35 µs per split-bf16x3 k-block under
  // the power cap, a third of that in bf16) and the partials' HBM round trip
  // at ~5 TB/s (µs per byte)
  const double unit_us = kb * 0.45 * (grp.task[0].planes == 3 ? 6 : grp.task[0].planes == 2 ? 3 : 1);
  const double us_per_byte = 1.0 / 5e6;
  const bool with_reduce = !(getenv("TR_SPLIT_REDUCE_COST") && getenv("TR_SPLIT_REDUCE_COST")[0] == '0');
  const double base = static_cast<double>(ceil_div(tiles, slots)) * unit_us;
  double best = base;
  int best_s = 1;
  for (int sp = 2; sp <= smax && kb / sp >= 8; ++sp) {
    const double cost = static_cast<double>(ceil_div(tiles * sp, slots)) / sp * unit_us +
                        (with_reduce ? 2.0 * sp * out_bytes * us_per_byte : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      best_s = sp;
    }
  }
  return best <= 0.9 * base ? best_s : 1;
}

// ---------------------------------------------------------------- grouped issue
static std::atomic<int> g_task_group{-1};

int task_group_max() {
  int v = g_task_group.load();
  if (v < 0) {
    const char* e = getenv("TR_GROUP");
    v = e ? std::max(1, std::min(kMaxGroup, atoi(e))) : 4;
    g_task_group.store(v);
  }
  return v;
}

void set_task_group_max(int n) { g_task_group.store(std::max(1, std::min(kMaxGroup, n))); }

// A task qualifies for a grouped launch when it runs as ONE launch (coherence on,
// capacity unbounded) and would not be split along K.  Host outputs land in the
// stream's group buffer and are written back on the writeback stream.
bool Session::groupable(int d, Job& job, int64_t gtid) {
  if (dryrun_ || exact_ || !coherence_ || devs_[d].capacity >= 0 || max_group_ < 2) return false;
  if (devs_[d].green && devs_[d].sms < 64) return false;  // a slice of a GPU: single tasks stay stealable
  int64_t tid = 0;
  const Product& p = job.prod_of(gtid, &tid);
  if (p.k_steps > kMaxKSteps) return false;
  // tasks for the CUDA-core kernel launch alone; k-splits are planned per group
  const int64_t nt = std::min<int64_t>(tile_, p.N - (tid % p.grid_cols) * tile_);
  return !(small_gemm_enabled() && (nt <= kSmallMaxN || p.K <= kSmallMaxK));
}

// _execute_task for several tasks at once: each task's directory sequence is the
// reference's (admit C, acquire A then B per k, release, release C); the
// arithmetic of all of them is ONE launch on stream s.
void Session::issue_group(int d, Job& job, const std::vector<int64_t>& gtids, int s) {
  NvtxRange nv("tr.task_group x%lld", static_cast<long long>(gtids.size()));
  DeviceCtx& dc = devs_[d];
  StreamCtx& sc = dc.streams[s];
  const int64_t T = tile_;
  GemmGroup grp;
  grp.n_tasks = static_cast<int32_t>(gtids.size());
  grp.k_split = 1;
  std::vector<TileKey> used;
  std::vector<int32_t> used_phys;
  std::vector<int32_t> wt_phys;  // slots the launch writes through
  const Product* p0 = nullptr;
  int64_t tid0 = 0;
  const size_t gtile = static_cast<size_t>(T * T * job.prod_of(gtids[0], &tid0).c.esize());
  for (size_t q = 0; q < gtids.size(); ++q) {
    int64_t tid = 0;
    const Product& p = job.prod_of(gtids[q], &tid);
    p0 = &p;
    const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
    const int64_t mt = std::min(T, p.M - i * T), nt = std::min(T, p.N - j * T);
    {
      DirLock g(dir_->mu);
      dir_->admit_output_locked(d, TileKey{p.c_uid, i, j});
    }
    GemmArgs& args = grp.task[q];
    std::memset(&args, 0, sizeof(args));
    args.m_valid = static_cast<int32_t>(mt);
    args.n_valid = static_cast<int32_t>(nt);
    args.n_ksteps = static_cast<int32_t>(p.k_steps);
    args.planes = planes_;
    if (p.c.location == TR_LOC_HOST) {  // the group buffer; written back after the launch
      args.c = static_cast<char*>(sc.gout) + q * gtile;
      args.ldc = nt;
    } else {
      args.c = const_cast<char*>(static_cast<const char*>(p.c.ptr)) + (i * T * p.c.ld + j * T) * p.c.esize();
      args.ldc = p.c.ld;
    }
    args.c_f64 = p.c.dtype == TR_DTYPE_F64;
    args.epilogue = p.axpy ? EPI_ACCUMULATE : EPI_STORE;
    args.scaled = p.axpy;
    args.alpha = p.alpha;
    args.seg_kb = seg_kb_for(planes_);
    args.k_split = 1;
    if (p.post != POST_NONE) {
      args.post = p.post;
      args.act = p.act;
      args.bias = p.bias ? p.bias + j * T : nullptr;
      args.aux = p.aux ? p.aux + (i * T) * p.ldaux + j * T : nullptr;
      args.ldaux = p.ldaux;
    }
    for (int64_t k = 0; k < p.k_steps; ++k) {
      const int64_t ar = p.ta ? k : i, ac = p.ta ? i : k;
      const int64_t br = p.tb ? j : k, bc = p.tb ? k : j;
      const int32_t pa = acquire(d, s, job, p.a, p.a_uid, p.ta, ar, ac, 0);
      const int32_t pb = acquire(d, s, job, p.b, p.b_uid, p.tb, br, bc, 1);
      args.a_z[k] = pa * planes_;
      args.b_z[k] = pb * planes_;
      args.k_len[k] = static_cast<int32_t>(std::min(T, p.K - k * T));
      used.push_back(TileKey{p.a_uid, ar, ac});
      used.push_back(TileKey{p.b_uid, br, bc});
      used_phys.push_back(pa);
      used_phys.push_back(pb);
    }
  }
  // split-K across the group (k-shares folded into the persistent unit walk);
  // the partials of task t go to its own region of the stream's workspace
  const int split = group_split(d, grp, group_uses_pairs(grp.task[0].m_valid));
  if (split > 1) {
    size_t total = 0;
    for (int t = 0; t < grp.n_tasks; ++t)
      total += static_cast<size_t>(split) * grp.task[t].m_valid * ((grp.task[t].n_valid + 255) / 256 * 256);
    if (float* ws = workspace(d, sc, total * sizeof(float))) {
      grp.k_split = split;
      for (int t = 0; t < grp.n_tasks; ++t) {
        GemmArgs& a = grp.task[t];
        a.k_split = split;
        a.ws = ws;
        a.ws_ld = (a.n_valid + 255) / 256 * 256;
        a.ws_zstride = static_cast<int64_t>(a.m_valid) * a.ws_ld;
        ws += split * a.ws_zstride;
      }
    }
  }
  std::vector<size_t> cs_pass;  // tasks whose column sums need a pass over the finished tile
  for (size_t q = 0; q < gtids.size(); ++q) {  // write-through: unsplit full tiles only
    int64_t tid = 0;
    const Product& p = job.prod_of(gtids[q], &tid);
    const int32_t wt = write_through(d, s, p, tid / p.grid_cols, tid % p.grid_cols, grp.task[q]);
    if (wt >= 0) wt_phys.push_back(wt);
    if (p.colsum && !fuse_colsum(p, tid / p.grid_cols, tid % p.grid_cols, grp.task[q])) cs_pass.push_back(q);
  }
  const bool host_c = p0->c.location == TR_LOC_HOST;
  if (host_c) wait_on(d, s, sc.gout_free);  // the previous group's writeback has read the buffer
  auto launch = [&] {
    TR_CUDA(launch_tile_gemm_group_maps(dc.tmap, grp, p0->ta, p0->tb, persistent_enabled() && !dc.host_fills,
                                        sc.stream, dc.sms));
    if (grp.k_split > 1)
      for (int t = 0; t < grp.n_tasks; ++t) TR_CUDA(launch_splitk_reduce(grp.task[t], sc.stream));
    for (size_t q : cs_pass) {
      int64_t tid = 0;
      const Product& p = job.prod_of(gtids[q], &tid);
      colsum_pass(p, tid / p.grid_cols, tid % p.grid_cols, sc.stream);
    }
    job.launches.fetch_add(grp.k_split > 1 ? grp.n_tasks : 0);
  };
  if (job.async) {
    launch();
  } else {
    TimedLaunch tl = timing_pair(d);
    TR_CUDA(cudaEventRecord(tl.start, sc.stream));
    launch();
    TR_CUDA(cudaEventRecord(tl.end, sc.stream));
    dc.timed.push_back(tl);
    if (tracing_) {
      for (size_t q = 0; q < gtids.size(); ++q) {
        int64_t tid = 0;
        const Product& p = job.prod_of(gtids[q], &tid);
        TraceRec rec;
        rec.ev = tr_trace_event{d, TR_TRACE_GEMM, s, gtids[q], static_cast<uint64_t>(dc.timed.size() - 1),
                                tid / p.grid_cols, tid % p.grid_cols, 0.0, 0.0};
        rec.t = TimedLaunch{nullptr, nullptr};
        dc.trace.push_back(rec);
      }
    }
  }
  job.launches.fetch_add(1);
  EvRef kernel_done;
  {
    DirLock g(dir_->mu);
    const EvRef ev = record(d, s);
    kernel_done = ev;
    for (int32_t ph : used_phys) note_use(dc.slots[ph], ev);
    for (int32_t ph : wt_phys) {  // the written-through tiles are ready when the launch is done
      dc.slots[ph].ready = ev;
      dc.slots[ph].uses.clear();
    }
    for (const TileKey& k : used) dir_->release_input_locked(d, k);
    for (int64_t gt : gtids) {
      int64_t tid = 0;
      const Product& p = job.prod_of(gt, &tid);
      const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
      const int64_t mt = std::min(T, p.M - i * T), nt = std::min(T, p.N - j * T);
      dir_->release_output_locked(d, TileKey{p.c_uid, i, j}, mt * nt * element_bytes_);  // coherence.py:263-280
    }
  }
  if (host_c) {
    // one pitched D2H per C tile on the writeback stream, so this stream (and the
    // next grouped launch, which waits for every other stream's kernel) does not
    // queue behind the copies; the job's final sync covers the writeback stream
    const int wb = dc.width + 2;
    wait_on(d, wb, kernel_done);
    for (size_t q = 0; q < gtids.size(); ++q) {
      int64_t tid = 0;
      const Product& p = job.prod_of(gtids[q], &tid);
      const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
      const int64_t mt = std::min(T, p.M - i * T), nt = std::min(T, p.N - j * T);
      const int64_t ces = p.c.esize();
      char* dst = const_cast<char*>(static_cast<const char*>(p.c.ptr)) + (i * T * p.c.ld + j * T) * ces;
      TimedLaunch tw{};
      trace_begin(d, wb, &tw);
      TR_CUDA(cudaMemcpy2DAsync(dst, p.c.ld * ces, static_cast<char*>(sc.gout) + q * gtile, nt * ces, nt * ces, mt,
                                cudaMemcpyDeviceToHost, dc.streams[wb].stream));
      trace_end(d, wb, tw, TR_TRACE_D2H, gtids[q], p.c_uid, i, j);
    }
    DirLock g(dir_->mu);
    sc.gout_free = record(d, wb);
  }
  if (job.async) {
    for (int64_t gt : gtids) {
      job.mark(gt);
      dc.stats.tasks_completed += 1;
      dc.stats.macs += job.task_macs(gt, tile_);
    }
    if (n_devices() > 1) {  // throttled: the launch occupies the stream until it completes
      TR_CUDA(cudaEventRecord(sc.done, sc.stream));
      sc.task = kTaskMarked;
    }
    return;
  }
  TR_CUDA(cudaEventRecord(sc.done, sc.stream));
  sc.task = gtids[0];
  sc.group_rest.assign(gtids.begin() + 1, gtids.end());
}

// ---------------------------------------------------------------- fused column sums
// Product::colsum (tr_product.colsum): the 32-row block column sums of task
// (i, j)'s final output.  fuse_colsum points the launch's epilogue at the
// tile's block of the partial-sum matrix when K1 stores the tile through its
// coalesced path (unsplit, fp32, 128-column multiples); false means the caller
// runs colsum_pass on the finished tile instead.
bool Session::fuse_colsum(const Product& p, int64_t i, int64_t j, GemmArgs& args, bool small) const {
  args.colsum = nullptr;
  if (!p.colsum) return true;
  if (args.k_split > 1 || args.c_f64) return false;
  if (!small && (args.n_valid % 128 != 0 || (args.ldc & 3) != 0 || (reinterpret_cast<uintptr_t>(args.c) & 15) != 0))
    return false;  // K1 sums on its coalesced store path only
  args.colsum = p.colsum + (i * tile_ / 32) * p.N + j * tile_;
  args.colsum_ld = p.N;
  return true;
}

void Session::colsum_pass(const Product& p, int64_t i, int64_t j, cudaStream_t s) {
  const int64_t T = tile_;
  const float* c = static_cast<const float*>(p.c.ptr) + i * T * p.c.ld + j * T;
  TR_CUDA(tile_colsum32(c, p.c.ld, std::min(T, p.M - i * T), std::min(T, p.N - j * T),
                        p.colsum + (i * T / 32) * p.N + j * T, p.N, s));
}

// ---------------------------------------------------------------- write-through
// A product whose output is read later as an input (Product::cache_as) has its
// output tiles admitted into the tile cache by the producing kernel itself: the
// epilogue writes the K2 planes next to the float32 result, so the consumer's
// acquire finds the tile resident (counted as the reference counts it: a host
// fetch, the pending entry being uncounted until requested) and no split/convert
// pass runs.  Full tiles on the coalesced epilogue path only.
int32_t Session::write_through(int d, int s, const Product& p, int64_t i, int64_t j, GemmArgs& args) {
  if (!p.cache_as || dryrun_ || !coherence_ || p.c.dtype != TR_DTYPE_F32 || args.k_split > 1) return -1;
  const int64_t T = tile_;
  if (T % 256 != 0 || std::min(T, p.M - i * T) != T || std::min(T, p.N - j * T) != T) return -1;
  if ((args.ldc & 3) != 0 || (reinterpret_cast<uintptr_t>(args.c) & 15) != 0) return -1;
  DirLock g(dir_->mu);
  int32_t slot = -1, source = TR_SOURCE_HOST;
  if (!dir_->prefetch_locked(d, TileKey{p.cache_as, i, j}, &slot, &source, false)) return -1;
  const int32_t phys = phys_of(d, slot);
  wait_slot_free(d, s, phys);  // earlier readers / fills of this physical slot
  args.wt = slot_ptr(d, phys);
  args.wt_ld = ld_;
  args.wt_plane = plane_elems_;
  return phys;
}

// ---------------------------------------------------------------- task issue
// _execute_task (scheduler.py:371-410), asynchronous: the host sequence of
// directory operations is identical; the arithmetic is enqueued on stream s.
void Session::issue(int d, Job& job, int64_t gtid, int s) {
  NvtxRange nv("tr.task %lld", static_cast<long long>(gtid));
  DeviceCtx& dc = devs_[d];
  int64_t tid = 0;
  const Product& p = job.prod_of(gtid, &tid);
  const int64_t T = tile_;
  const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
  const int64_t mt = std::min(T, p.M - i * T);
  const int64_t nt = std::min(T, p.N - j * T);
  const TileKey c_key{p.c_uid, i, j};
  const int64_t ks = p.k_steps;
  int64_t chunk = ks;
  if (!coherence_) chunk = 1;
  else if (dc.capacity >= 0 && dc.capacity < 2 * ks + 1) chunk = std::max<int64_t>(1, (dc.capacity - 1) / 2);
  chunk = std::min<int64_t>(chunk, kMaxKSteps);
  {
    DirLock g(dir_->mu);
    dir_->admit_output_locked(d, c_key);  // pinned for the whole task (scheduler.py:390)
  }
  StreamCtx* scp = dryrun_ ? nullptr : &dc.streams[s];
  const int64_t ces = p.c.esize();
  void* cptr = nullptr;
  int64_t ldc = 0;
  if (!dryrun_) {
    if (p.c.location == TR_LOC_HOST) {
      cptr = lazy_tile(d, &scp->outbuf, &scp->outbuf_cap);
      ldc = nt;
    } else {
      cptr = const_cast<char*>(static_cast<const char*>(p.c.ptr)) + (i * T * p.c.ld + j * T) * ces;
      ldc = p.c.ld;
    }
  }
  for (int64_t k0 = 0; k0 < ks; k0 += chunk) {
    const int64_t kc = std::min(chunk, ks - k0);
    GemmArgs args;
    std::memset(&args, 0, sizeof(args));
    args.m_valid = static_cast<int32_t>(mt);
    args.n_valid = static_cast<int32_t>(nt);
    args.n_ksteps = static_cast<int32_t>(kc);
    args.planes = planes_;
    args.c = cptr;
    args.ldc = ldc;
    args.c_f64 = p.c.dtype == TR_DTYPE_F64;
    args.epilogue = (k0 == 0 && !p.axpy) ? EPI_STORE : EPI_ACCUMULATE;
    args.scaled = p.axpy;
    args.alpha = p.alpha;
    args.seg_kb = seg_kb_for(planes_);
    if (p.post != POST_NONE && k0 + kc == ks) {  // fused post-op on the final chunk only
      args.post = p.post;
      args.act = p.act;
      args.bias = p.bias ? p.bias + j * T : nullptr;
      args.aux = p.aux ? p.aux + (i * T) * p.ldaux + j * T : nullptr;
      args.ldaux = p.ldaux;
    }
    std::vector<TileKey> used;
    std::vector<int32_t> used_phys;
    for (int64_t k = k0; k < k0 + kc; ++k) {
      // input acquire order per k-step: A then B (scheduler.py:394-396)
      const int64_t ar = p.ta ? k : i, ac = p.ta ? i : k;
      const int64_t br = p.tb ? j : k, bc = p.tb ? k : j;
      const int32_t pa = acquire(d, s, job, p.a, p.a_uid, p.ta, ar, ac, 0);
      const int32_t pb = acquire(d, s, job, p.b, p.b_uid, p.tb, br, bc, 1);
      args.a_z[k - k0] = pa * planes_;
      args.b_z[k - k0] = pb * planes_;
      args.k_len[k - k0] = static_cast<int32_t>(std::min(T, p.K - k * T));
      used.push_back(TileKey{p.a_uid, ar, ac});
      used.push_back(TileKey{p.b_uid, br, bc});
      used_phys.push_back(pa);
      used_phys.push_back(pb);
    }
    int64_t k_total = 0;
    for (int64_t k = 0; k < kc; ++k) k_total += args.k_len[k];
    // narrow C tile (the MLP's 10-wide output layer): Bᵀ·Aᵀ on the tensor cores
    GemmArgs targs;
    // (the exact mode has one kernel: KX, k ascending, never split)
    const bool narrow = !dryrun_ && !exact_ && narrow_tc_enabled() && T > kSmallMaxN && args.n_valid <= kSmallMaxN &&
                        k_total > kSmallMaxK && plan_narrow(d, *scp, args, targs);
    const bool small = !dryrun_ && !exact_ && !narrow && small_gemm_enabled() && small_gemm_eligible(args);
    if (!dryrun_ && !exact_ && !narrow) {
      if (small) plan_split_small(d, *scp, args);
      else plan_split_k(d, *scp, args);
    }
    const int32_t wt = (!dryrun_ && !exact_ && !narrow && k0 == 0 && kc == ks) ? write_through(d, s, p, i, j, args)
                                                                               : -1;
    const bool reduce = narrow || args.k_split > 1;
    // column sums of the final output: fused into K1's epilogue when it stores the tile, else a pass over it
    const bool cs_pass = !dryrun_ && p.colsum && k0 + kc == ks && (narrow || !fuse_colsum(p, i, j, args, small));
    auto launch = [&] {
      if (exact_) {
        TR_CUDA(launch_exact_gemm(dc.slab, dc.slab, ld_, plane_elems_, args, p.ta, p.tb,
                                  p.a.dtype == TR_DTYPE_F32 && p.b.dtype == TR_DTYPE_F32, scp->stream));
      } else if (narrow) {  // A' = Bᵀ, B' = Aᵀ: the layouts swap roles
        BoxKind ba, bb;
        gemm_boxes(!p.tb, !p.ta, targs.m_valid, &ba, &bb);
        TR_CUDA(launch_tile_gemm(dc.tmap[ba], dc.tmap[bb], targs, !p.tb, !p.ta, scp->stream));
        TR_CUDA(launch_splitk_reduce_t(args, scp->stream));
      } else {
        if (small) {
          TR_CUDA(launch_small_gemm(dc.slab, ld_, plane_elems_, args, p.ta, p.tb, scp->stream));
        } else {
          BoxKind ba, bb;
          gemm_boxes(p.ta, p.tb, args.m_valid, &ba, &bb);
          TR_CUDA(launch_tile_gemm(dc.tmap[ba], dc.tmap[bb], args, p.ta, p.tb, scp->stream));
        }
        if (args.k_split > 1) TR_CUDA(launch_splitk_reduce(args, scp->stream));
      }
      if (cs_pass) colsum_pass(p, i, j, scp->stream);
    };
    if (!dryrun_ && job.async) {
      launch();
      job.launches.fetch_add(reduce ? 2 : 1);
    } else if (!dryrun_) {
      TimedLaunch tl = timing_pair(d);
      TR_CUDA(cudaEventRecord(tl.start, scp->stream));
      launch();
      if (reduce) job.launches.fetch_add(1);
      TR_CUDA(cudaEventRecord(tl.end, scp->stream));
      dc.timed.push_back(tl);
      if (tracing_) {
        // the launch's own timing pair (dc.timed) provides the times; remember its index
        TraceRec rec;
        rec.ev = tr_trace_event{d, TR_TRACE_GEMM, s, gtid, static_cast<uint64_t>(dc.timed.size() - 1), i, j, 0.0, 0.0};
        rec.t = TimedLaunch{nullptr, nullptr};
        dc.trace.push_back(rec);
      }
      job.launches.fetch_add(1);
    }
    {
      DirLock g(dir_->mu);
      if (!dryrun_ && coherence_) {
        const EvRef ev = record(d, s);
        for (int32_t p : used_phys) note_use(dc.slots[p], ev);
        if (wt >= 0) {
          dc.slots[wt].ready = ev;
          dc.slots[wt].uses.clear();
        }
      }
      for (const TileKey& k : used) dir_->release_input_locked(d, k);
    }
  }
  const int64_t wb_bytes = mt * nt * element_bytes_;
  if (!dryrun_ && p.c.location == TR_LOC_HOST) {
    char* dst = const_cast<char*>(static_cast<const char*>(p.c.ptr)) + (i * T * p.c.ld + j * T) * ces;
    TimedLaunch tw{};
    trace_begin(d, s, &tw);
    TR_CUDA(cudaMemcpy2DAsync(dst, p.c.ld * ces, scp->outbuf, nt * ces, nt * ces, mt, cudaMemcpyDeviceToHost,
                              scp->stream));
    trace_end(d, s, tw, TR_TRACE_D2H, gtid, p.c_uid, i, j);
  }
  {
    DirLock g(dir_->mu);
    dir_->release_output_locked(d, c_key, wb_bytes);  // coherence.py:263-280
  }
  if (dryrun_ || job.async) {  // async: the task completes in stream order
    job.mark(gtid);
    dc.stats.tasks_completed += 1;
    dc.stats.macs += job.task_macs(gtid, tile_);
    if (!dryrun_ && n_devices() > 1) {  // throttled: see run_job
      TR_CUDA(cudaEventRecord(scp->done, scp->stream));
      scp->task = kTaskMarked;
    }
    return;
  }
  TR_CUDA(cudaEventRecord(scp->done, scp->stream));
  scp->task = gtid;
}

void Session::reap(int d, Job& job, bool block_oldest) {
  DeviceCtx& dc = devs_[d];
  int oldest = -1;
  for (int s = 0; s < dc.width; ++s) {
    StreamCtx& sc = dc.streams[s];
    if (sc.task == kTaskNone) continue;
    if (oldest < 0 || sc.seq < dc.streams[oldest].seq) oldest = s;
  }
  if (block_oldest && oldest >= 0) TR_CUDA(cudaEventSynchronize(dc.streams[oldest].done));
  for (int s = 0; s < dc.width; ++s) {
    StreamCtx& sc = dc.streams[s];
    if (sc.task == kTaskNone) continue;
    cudaError_t e = cudaEventQuery(sc.done);
    if (e == cudaErrorNotReady) continue;
    TR_CUDA(e);
    if (sc.task == kTaskMarked) {  // stream-ordered task, counted when it was enqueued
      sc.task = kTaskNone;
      continue;
    }
    job.mark(sc.task);
    dc.stats.tasks_completed += 1;
    dc.stats.macs += job.task_macs(sc.task, tile_);
    for (int64_t gt : sc.group_rest) {
      job.mark(gt);
      dc.stats.tasks_completed += 1;
      dc.stats.macs += job.task_macs(gt, tile_);
    }
    sc.group_rest.clear();
    sc.task = -1;
  }
}

// The device worker (scheduler.py:475-505): refill -> pop -> steal -> issue.
void Session::run_job(int d, Job& job) {
  NvtxRange nv("tr.device %lld", static_cast<long long>(d));
  DeviceCtx& dc = devs_[d];
  Station& st = *dc.station;
  uint64_t seq = 0;
  bool ahead = !dryrun_ && coherence_ && !(flags_ & TR_FLAG_NO_PREFETCH);
  for (auto& dv : devs_) ahead = ahead && dv.capacity < 0;  // bounded caches: keep eviction order exact
  // locality priority among a station's reserved tasks (unbounded caches only:
  // bounded ones keep the reference's FIFO pop and exact eviction order)
  bool prio = !dryrun_ && coherence_ && !job.async && getenv("TR_PRIORITY") == nullptr;
  for (auto& dv : devs_) prio = prio && dv.capacity < 0;
  if (const char* e = getenv("TR_PRIORITY")) prio = !dryrun_ && e[0] == '1';
  // While the job still has host tiles to fill on this device, its grouped
  // launches are non-persistent: a persistent grid holds every SM for the whole
  // launch, so the fill stream's split/convert blocks (top priority) only start
  // between launches and the next group's tiles arrive late (cfg4 N=131072 cold:
  // 0.75 s of idle tensor cores per 11.6 s product persistent, 0.13 s
  // non-persistent).  Re-evaluated every 16 issues: once every input tile is
  // resident (the first-touch phase is over) launches go persistent again.
  auto host_fills_pending = [&]() {
    if (dryrun_) return false;
    DirLock g(dir_->mu);
    for (const Product& p : job.prods)
      for (int which = 0; which < 2; ++which) {
        const Mat& m = which == 0 ? p.a : p.b;
        if (m.location != TR_LOC_HOST) continue;
        const uint64_t uid = which == 0 ? p.a_uid : p.b_uid;
        for (int64_t r = 0; r < (m.rows + tile_ - 1) / tile_; ++r)
          for (int64_t c = 0; c < (m.cols + tile_ - 1) / tile_; ++c)
            if (!(dir_->owners_locked(TileKey{uid, r, c}) >> d & 1)) return true;
      }
    return false;
  };
  dc.host_fills = host_fills_pending();
  int64_t issues = 0;
  std::vector<uint8_t> seen(ahead ? static_cast<size_t>(job.total) : 0, 0);
  std::vector<uint8_t> seen_global(seen.size(), 0);
  dc.pending_prefetch = 0;
  // A green-context device is a slice of a GPU.  When one task's CTAs fill it
  // twice over, a second concurrent task adds nothing but a task the others can
  // no longer steal (a running task is not stealable): one at a time, like the
  // reference's workers, so a throttled device never sits on work the faster
  // devices could finish first.
  int max_inflight = dc.max_inflight;
  if (dc.green && !job.prods.empty()) {
    const int64_t t = std::min<int64_t>(tile_, std::max(job.prods[0].M, job.prods[0].N));
    if (ceil_div(t, 128) * ceil_div(t, 256) >= 2 * static_cast<int64_t>(dc.sms)) max_inflight = 1;
  }
  while (!job.abort.load()) {
    int active = 0;
    if (!dryrun_) {
      reap(d, job, false);
      for (auto& sc : dc.streams) active += sc.task != kTaskNone;
    }
    if (active >= max_inflight) {
      reap(d, job, true);
      continue;
    }
    // a grouped launch takes a whole station's worth of tasks on ONE stream, so the
    // station refills to its full width regardless of the streams in flight
    const int room = (max_group_ > 1 && !dryrun_) ? dc.width : dc.width - active;
    job.claimed.fetch_add(static_cast<int64_t>(st.refill(job.queue, room).size()));
    if (ahead) fetch_ahead(d, job, seen, seen_global, dc.pending_prefetch);
    uint64_t tid;
    int victim = -1;
    bool popped;
    if (prio) {
      // locality priority: the reserved task with the most input tiles already in
      // this device's HBM (2 points) or a peer's (1 point) runs first
      popped = st.pop_best(&tid, [&](uint64_t t) {
        int64_t lt = 0;
        const Product& p = job.prod_of(static_cast<int64_t>(t), &lt);
        const int64_t i = lt / p.grid_cols, j = lt % p.grid_cols;
        int score = 0;
        DirLock g(dir_->mu);
        for (int64_t k = 0; k < p.k_steps; ++k) {
          const uint64_t oa = dir_->owners_locked(TileKey{p.a_uid, p.ta ? k : i, p.ta ? i : k});
          const uint64_t ob = dir_->owners_locked(TileKey{p.b_uid, p.tb ? j : k, p.tb ? k : j});
          for (uint64_t o : {oa, ob}) score += (o >> d & 1) ? 2 : (o ? 1 : 0);
        }
        return score;
      });
    } else {
      popped = st.pop_for_run(&tid);
    }
    if (!popped) {
      if (!job.queue.is_empty()) continue;  // raced with other refills
      bool got = false;
      if (steal_) got = steal_task(d, station_ptrs_.data(), static_cast<int>(station_ptrs_.size()), &tid, &victim);
      if (!got) {
        if (active == 0 || (job.async && job.all_done())) {  // stream-ordered launches may still run
          if (job.all_done()) return;
          std::this_thread::sleep_for(std::chrono::microseconds(50));
        } else {
          reap(d, job, true);
        }
        continue;
      }
    }
    if (victim >= 0) {
      std::lock_guard<std::mutex> g(job.mu);
      job.steals.push_back(tr_steal_event{d, victim, static_cast<int64_t>(tid), 0.0});
      dc.stats.steals_performed += 1;
      devs_[victim].stats.steals_suffered += 1;
    }
    // Stream-ordered products (job.async) are enqueued without waiting for the
    // GPU.  One device: round-robin over its streams, nothing to reap.  Several
    // devices: each keeps at most max_inflight launches in flight (their events
    // reaped like synchronous tasks), so a device pulls tasks from the shared
    // queue at the rate its GPU (or green context) retires them -- enqueue speed
    // would otherwise decide the shares (BASELINE cfg5's throttled devices).
    if (dc.host_fills && ++issues % 16 == 0) dc.host_fills = host_fills_pending();
    int s = 0;
    if (job.async && n_devices() == 1) {
      s = static_cast<int>(seq++ % static_cast<uint64_t>(max_inflight));
    } else if (!dryrun_) {
      while (dc.streams[s].task != kTaskNone) ++s;
      dc.streams[s].seq = ++seq;
    }
    // Group only while the queue still holds a round of groups for every device:
    // in a product's tail single tasks stay stealable, so a slow (e.g. green-
    // context) device never holds several tasks the others could have taken.
    const bool tail = job.n_tasks - job.claimed.load() < static_cast<int64_t>(max_group_) * n_devices();
    int64_t t0 = 0;
    const Product* p0 = &job.prod_of(static_cast<int64_t>(tid), &t0);
    if (victim < 0 && !(tail && n_devices() > 1) && groupable(d, job, static_cast<int64_t>(tid)) &&
        (p0->c.location != TR_LOC_HOST ||
         group_outbuf(d, s, static_cast<size_t>(std::min(max_group_, kMaxGroup)) * tile_ * tile_ * p0->c.esize()))) {
      // the station's other ready tasks of the same product join this launch
      std::vector<int64_t> grp{static_cast<int64_t>(tid)};
      const bool tall0 = group_uses_pairs(static_cast<int>(std::min<int64_t>(tile_, p0->M - (t0 / p0->grid_cols) * tile_)));
      uint64_t more;
      while (static_cast<int>(grp.size()) < std::min(max_group_, kMaxGroup) && st.peek_front(&more)) {
        int64_t t1 = 0;
        const Product* p1 = &job.prod_of(static_cast<int64_t>(more), &t1);
        const bool tall1 = group_uses_pairs(static_cast<int>(std::min<int64_t>(tile_, p1->M - (t1 / p1->grid_cols) * tile_)));
        if (p1 != p0 || tall1 != tall0 || !groupable(d, job, static_cast<int64_t>(more))) break;
        if (!st.pop_for_run(&more)) break;
        grp.push_back(static_cast<int64_t>(more));
      }
      if (grp.size() > 1) {
        if (!job.async)  // one grouped launch in flight per device: pairs lose SM pairs to a concurrent kernel
          while (true) {
            int busy = 0;
            for (int q = 0; q < dc.width; ++q) busy += dc.streams[q].task != kTaskNone && q != s;
            if (!busy) break;
            reap(d, job, true);
          }
        issue_group(d, job, grp, s);
        continue;
      }
    }
    issue(d, job, static_cast<int64_t>(tid), s);
  }
}

void Session::worker_main(int d) {
  pin_thread_to_core(d, dryrun_ ? -1 : devs_[d].gpu);
  if (!dryrun_) cudaSetDevice(devs_[d].gpu);
  uint64_t seen = 0;
  for (;;) {
    Job* job;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return shutdown_ || generation_ != seen; });
      if (shutdown_) return;
      seen = generation_;
      job = job_;
    }
    try {
      run_job(d, *job);
    } catch (const Error& e) {
      job->set_error(e.status, e.what());
    } catch (const std::exception& e) {
      job->set_error(TR_ERR_INTERNAL, e.what());
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      workers_done_ += 1;
    }
    cv_done_.notify_all();
  }
}

// ---------------------------------------------------------------- one product
namespace {
struct HostReg {
  std::vector<const void*> regs;
  void ensure(const Mat& m) {
    if (m.location != TR_LOC_HOST || !m.ptr) return;
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, m.ptr);
    if (e == cudaSuccess && attr.type == cudaMemoryTypeHost) return;
    cudaGetLastError();
    const size_t bytes = static_cast<size_t>(((m.rows - 1) * m.ld + m.cols) * m.esize());
    if (cudaHostRegister(const_cast<void*>(m.ptr), bytes, cudaHostRegisterPortable) == cudaSuccess)
      regs.push_back(m.ptr);
    else
      cudaGetLastError();  // fall back to pageable copies
  }
  ~HostReg() {
    for (const void* p : regs) cudaHostUnregister(const_cast<void*>(p));
  }
};
}  // namespace

void Session::gemm(const Mat& a, uint64_t a_uid, bool ta, const Mat& b, uint64_t b_uid, bool tb, const Mat& c,
                   uint64_t c_uid, int64_t task_offset, int64_t task_stride, tr_gemm_report* rep) {
  Product p;
  p.a = a;
  p.b = b;
  p.c = c;
  p.ta = ta;
  p.tb = tb;
  p.a_uid = a_uid;
  p.b_uid = b_uid;
  p.c_uid = c_uid;
  std::vector<Product> v{p};
  run_products(std::move(v), task_offset, task_stride, rep);
}

// Enqueue order of one product's task ids (see tr_session_set_order).
static std::vector<int64_t> product_order(const Product& p, int order, int64_t room) {
  const int64_t total = p.grid_rows * p.grid_cols;
  std::vector<int64_t> ids;
  ids.reserve(static_cast<size_t>(total));
  if (order == 1) {
    const int64_t G = 2;
    for (int64_t b = 0; b < p.grid_rows; b += G)
      for (int64_t j = 0; j < p.grid_cols; ++j)
        for (int64_t i = b; i < std::min(b + G, p.grid_rows); ++i) ids.push_back(i * p.grid_cols + j);
  } else if (order == 2 || order == 4) {
    // shells (order 4: the k-panel schedule walks its tasks in shells order too): task (i, j) in shell max(i, j); each shell adds one A row and one
    // B column of tiles, so compute starts after 2 k-panels instead of a full row
    const int64_t g = std::max(p.grid_rows, p.grid_cols);
    for (int64_t sh = 0; sh < g; ++sh) {
      for (int64_t i = 0; i < std::min(sh, p.grid_rows); ++i)
        if (sh < p.grid_cols) ids.push_back(i * p.grid_cols + sh);
      if (sh < p.grid_rows)
        for (int64_t j = 0; j <= std::min(sh, p.grid_cols - 1); ++j) ids.push_back(sh * p.grid_cols + j);
    }
  } else if (order == 3) {
    // blocked: b x b task blocks whose (b + b) k-panels fit the tile budget, so
    // each A/B tile is fetched once per block instead of once per task row
    // (each block walked in shells from its corner, so compute starts after two
    // k-panels of the block instead of its whole first task row)
    const int64_t ks = std::max<int64_t>(1, p.k_steps);
    const int64_t bsz = std::max<int64_t>(1, (room == INT64_MAX ? total : (room - 8)) / (2 * ks));
    for (int64_t bi = 0; bi < p.grid_rows; bi += bsz)
      for (int64_t bj = 0; bj < p.grid_cols; bj += bsz) {
        const int64_t br = std::min(bsz, p.grid_rows - bi), bc = std::min(bsz, p.grid_cols - bj);
        for (int64_t sh = 0; sh < std::max(br, bc); ++sh) {
          for (int64_t i = 0; i < std::min(sh, br); ++i)
            if (sh < bc) ids.push_back((bi + i) * p.grid_cols + bj + sh);
          if (sh < br)
            for (int64_t j = 0; j <= std::min(sh, bc - 1); ++j) ids.push_back((bi + sh) * p.grid_cols + bj + j);
        }
      }
  } else {
    for (int64_t t = 0; t < total; ++t) ids.push_back(t);
  }
  return ids;
}

void Session::run_products(std::vector<Product> prods, int64_t task_offset, int64_t task_stride,
                           tr_gemm_report* rep) {
  NvtxRange nv("tr.products x%lld", static_cast<long long>(prods.size()));
  if (prods.empty()) fail(TR_ERR_VALUE, "empty product batch");
  if (task_stride < 1 || task_offset < 0 || task_offset >= task_stride) fail(TR_ERR_VALUE, "bad task shard");
  const int64_t T = tile_;
  int64_t total = 0, in_tiles_all = 0;
  for (Product& p : prods) {
    const Mat &a = p.a, &b = p.b, &c = p.c;
    p.M = p.ta ? a.cols : a.rows;
    p.K = p.ta ? a.rows : a.cols;
    const int64_t Kb = p.tb ? b.cols : b.rows;
    p.N = p.tb ? b.rows : b.cols;
    if (a.rows < 1 || a.cols < 1 || b.rows < 1 || b.cols < 1) fail(TR_ERR_SHAPE, "matrix dimensions must be >= 1");
    if (p.K != Kb)
      fail(TR_ERR_SHAPE, "inner dimensions differ: (%lld, %lld) x (%lld, %lld)", (long long)p.M, (long long)p.K,
           (long long)Kb, (long long)p.N);
    if (c.rows != p.M || c.cols != p.N)
      fail(TR_ERR_SHAPE, "output is %lldx%lld, expected %lldx%lld", (long long)c.rows, (long long)c.cols,
           (long long)p.M, (long long)p.N);
    for (const Mat* m : {&a, &b, &c})
      if (m->ld < m->cols || (!dryrun_ && !m->ptr)) fail(TR_ERR_SHAPE, "bad matrix descriptor (ld < cols or null)");
    if (p.post != POST_NONE && (c.location != TR_LOC_DEVICE || c.dtype != TR_DTYPE_F32))
      fail(TR_ERR_VALUE, "fused epilogues need a float32 device output");
    if (p.post == POST_ACT_GRAD && !p.aux) fail(TR_ERR_VALUE, "POST_ACT_GRAD needs the activation (aux) matrix");
    if (exact_ && (p.post != POST_NONE || p.axpy || p.colsum || p.cache_as))
      fail(TR_ERR_VALUE, "precision 'exact' runs plain products only (no fused epilogue, axpy or write-through)");
    if (p.colsum && (c.location != TR_LOC_DEVICE || c.dtype != TR_DTYPE_F32 || T % 32 != 0))
      fail(TR_ERR_VALUE, "fused column sums need a float32 device output and a tile size that is a multiple of 32");
    if (p.axpy && (p.post != POST_NONE || c.location != TR_LOC_DEVICE || c.dtype != TR_DTYPE_F32))
      fail(TR_ERR_VALUE, "axpy products accumulate into a float32 device matrix, without a post-op");
    p.grid_rows = ceil_div(p.M, T);
    p.grid_cols = ceil_div(p.N, T);
    p.k_steps = ceil_div(p.K, T);
    p.base = total;
    total += p.grid_rows * p.grid_cols;
    in_tiles_all += ceil_div(a.rows, T) * ceil_div(a.cols, T) + ceil_div(b.rows, T) * ceil_div(b.cols, T);
  }
  Job job(total);
  job.prods = std::move(prods);
  // Stream-ordered mode (tr_session_set_async): with a caller stream and every
  // operand in device memory, the call returns once all tasks are enqueued; the
  // caller's stream waits for the product, the next product's streams wait for
  // the caller's stream, so successive products (and the caller's own kernels)
  // stay ordered without a host round trip between them.
  job.async = async_ && ext_on_ && !dryrun_ && !tracing_;
  for (const Product& p : job.prods)
    for (const Mat* m : {&p.a, &p.b, &p.c}) job.async = job.async && m->location == TR_LOC_DEVICE;
  // plan(): every task enqueued up front (scheduler.py:189-192).  Row-major as in
  // the reference, or -- when no device has a bounded capacity, so the hit/miss
  // counters cannot depend on the order -- in "shells" (all tasks with
  // max(i, j) = s before shell s + 1), which spreads first-touch host traffic
  // over the run instead of loading every B panel during the first task row.
  // Products of a batch are interleaved round-robin.
  int order = order_;
  int64_t room = INT64_MAX;  // smallest tile budget of any device
  for (auto& dc : devs_) {
    const int64_t cap = dc.capacity >= 0 ? dc.capacity : (dryrun_ ? INT64_MAX : dc.max_slots);
    room = std::min(room, cap);
  }
  if (order < 0 && sim_) order = 0;  // the reference's row-major plan: exact sim parity
  if (order < 0) {
    bool bounded = false;
    for (auto& dc : devs_) bounded = bounded || dc.capacity >= 0;
    if (bounded) order = 0;                          // reference order: exact LRU parity
    else if (in_tiles_all > room) order = 3;         // out-of-core: blocked
    else order = 2;                                  // in-core: shells
  }
  std::vector<std::vector<int64_t>> per;
  for (const Product& p : job.prods) per.push_back(product_order(p, order, room));
  std::vector<int64_t> ids;
  ids.reserve(static_cast<size_t>(total));
  if (max_group_ > 1 && !dryrun_) {
    // grouped launches take consecutive tasks of ONE product: keep products contiguous
    for (size_t q = 0; q < per.size(); ++q)
      for (int64_t t : per[q]) ids.push_back(job.prods[q].base + t);
  }
  const bool interleave = ids.empty();  // products round-robin (per-task launches)
  for (size_t r = 0; interleave; ++r) {
    bool any = false;
    for (size_t q = 0; q < per.size(); ++q)
      if (r < per[q].size()) {
        ids.push_back(job.prods[q].base + per[q][r]);
        any = true;
      }
    if (!any) break;
  }
  int64_t planned = 0;
  for (int64_t t : ids) {
    if (t % task_stride != task_offset) continue;
    job.queue.enqueue(static_cast<uint64_t>(t));
    job.order.push_back(t);
    ++planned;
  }
  job.n_tasks = planned;
  for (auto& dc : devs_) {
    dc.station->clear();
    dc.stats = tr_device_stats{};
  }
  peer_served_.assign(devs_.size(), 0);

  int prev_dev = 0;
  if (!dryrun_) cudaGetDevice(&prev_dev);
  struct RestoreDev {
    bool on;
    int dev;
    ~RestoreDev() {
      if (on) cudaSetDevice(dev);
    }
  } restore{!dryrun_, prev_dev};
  HostReg reg;
  if (!dryrun_) {
    for (const Product& p : job.prods) {
      reg.ensure(p.a);
      reg.ensure(p.b);
      reg.ensure(p.c);
    }
    // slab room for this job: the tiles already cached plus the job's input tiles
    // not yet resident on the device (a warm re-multiply needs no growth)
    for (int d = 0; d < n_devices(); ++d) {
      int64_t missing = 0;
      {
        DirLock g(dir_->mu);
        for (const Product& p : job.prods)
          for (int which = 0; which < 2; ++which) {
            const Mat& m = which == 0 ? p.a : p.b;
            const uint64_t uid = which == 0 ? p.a_uid : p.b_uid;
            for (int64_t r = 0; r < ceil_div(m.rows, T); ++r)
              for (int64_t c = 0; c < ceil_div(m.cols, T); ++c)
                missing += !(dir_->owners_locked(TileKey{uid, r, c}) >> d & 1);
          }
      }
      ensure_slab(d, dir_->used_tiles(d) + missing);
    }
  }
  // out-of-core (the inputs exceed the HBM slab, capacity unbounded): the
  // directory learns every input tile's remaining requests so that physical
  // evictions and fetch-ahead replace dead tiles first
  bool unbounded = true;
  for (auto& dc : devs_) unbounded = unbounded && dc.capacity < 0;
  job.out_of_core = !dryrun_ && coherence_ && unbounded && in_tiles_all > room;
  struct FutureGuard {
    Directory* dir;
    bool on;
    ~FutureGuard() {
      if (!on) return;
      DirLock g(dir->mu);
      dir->clear_future_locked();
    }
  } future_guard{dir_.get(), job.out_of_core};
  if (job.out_of_core) {
    std::unordered_map<TileKey, int64_t, TileKeyHash> future;
    for (int64_t gt : job.order) {
      int64_t tid = 0;
      const Product& p = job.prod_of(gt, &tid);
      const int64_t i = tid / p.grid_cols, j = tid % p.grid_cols;
      for (int64_t k = 0; k < p.k_steps; ++k) {
        future[TileKey{p.a_uid, p.ta ? k : i, p.ta ? i : k}] += 1;
        future[TileKey{p.b_uid, p.tb ? j : k, p.tb ? k : j}] += 1;
      }
    }
    DirLock g(dir_->mu);
    dir_->set_future_locked(std::move(future));
  }
  const tr_cache_stats before = dir_->stats();
  const std::vector<tr_cache_stats> before_dev = dir_->stats_per_device();
  if (!dryrun_) {
    if (ext_on_) {
      // inputs produced on the caller's stream (e.g. torch) must be complete first
      if (!ext_ready_) TR_CUDA(cudaEventCreateWithFlags(&ext_ready_, cudaEventDisableTiming));
      TR_CUDA(cudaEventRecord(ext_ready_, ext_stream_));
    }
    // device-side span of the product: every stream starts after span_start,
    // span_end is recorded after every stream's last operation
    for (auto& dc : devs_) {
      TR_CUDA(cudaSetDevice(dc.gpu));
      if (ext_on_) TR_CUDA(cudaStreamWaitEvent(dc.streams[0].stream, ext_ready_, 0));
      TR_CUDA(cudaEventRecord(dc.span_start, dc.streams[0].stream));
      for (size_t s = 1; s < dc.streams.size(); ++s)
        TR_CUDA(cudaStreamWaitEvent(dc.streams[s].stream, dc.span_start, 0));
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  const double sim_before = sim_now();
  if (sim_) {
    run_sim(job);  // one thread, the reference's event order (scheduler.py:432-464)
  } else if (panels_apply(job) && run_panels(job)) {
    // cold single-device product: done by the k-panel schedule on this thread
  } else {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      workers_done_ = 0;
      generation_ += 1;
    }
    cv_.notify_all();
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_done_.wait(lk, [&] { return workers_done_ == n_devices(); });
      job_ = nullptr;
    }
  }
  last_makespan_ = sim_ ? sim_now() - sim_before : 0.0;

  if (job.async) {
    for (auto& dc : devs_) {
      TR_CUDA(cudaSetDevice(dc.gpu));
      for (int s = 1; s < static_cast<int>(dc.streams.size()); ++s) wait_on(dc.id, 0, record(dc.id, s));
      TR_CUDA(cudaEventRecord(dc.span_end, dc.streams[0].stream));
      TR_CUDA(cudaStreamWaitEvent(ext_stream_, dc.span_end, 0));
    }
  } else if (!dryrun_) {
    for (auto& dc : devs_) {
      cudaSetDevice(dc.gpu);
      for (int s = 1; s < static_cast<int>(dc.streams.size()); ++s) wait_on(dc.id, 0, record(dc.id, s));
      cudaEventRecord(dc.span_end, dc.streams[0].stream);
      for (auto& sc : dc.streams) {
        cudaError_t e = cudaStreamSynchronize(sc.stream);
        if (e != cudaSuccess) job.set_error(TR_ERR_CUDA, std::string("stream sync: ") + cudaGetErrorString(e));
        sc.task = -1;
      }
    }
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // trace (before the timing events are recycled)
  last_trace_.clear();
  if (tracing_) {
    for (auto& dc : devs_) {
      for (auto& rec : dc.trace) {
        float a = 0, b = 0;
        if (rec.ev.kind == TR_TRACE_GEMM) {
          const TimedLaunch& tl = dc.timed[static_cast<size_t>(rec.ev.matrix)];
          rec.ev.matrix = 0;
          cudaEventElapsedTime(&a, dc.span_start, tl.start);
          cudaEventElapsedTime(&b, dc.span_start, tl.end);
        } else {
          cudaEventElapsedTime(&a, dc.span_start, rec.t.start);
          cudaEventElapsedTime(&b, dc.span_start, rec.t.end);
          dc.timed_pool.push_back(rec.t);
        }
        cudaGetLastError();
        rec.ev.start_ms = a;
        rec.ev.end_ms = b;
        last_trace_.push_back(rec.ev);
      }
      dc.trace.clear();
    }
  }
  // kernel timings
  for (auto& dc : devs_) {
    double ms = 0;
    for (auto& tl : dc.timed) {
      float x = 0;
      if (cudaEventElapsedTime(&x, tl.start, tl.end) == cudaSuccess) ms += x;
      else cudaGetLastError();
      dc.timed_pool.push_back(tl);
    }
    dc.last_launches = static_cast<int64_t>(dc.timed.size());
    dc.timed.clear();
    dc.last_kernel_ms = ms;
    float span = 0;
    if (!dryrun_ && !job.async && cudaEventElapsedTime(&span, dc.span_start, dc.span_end) != cudaSuccess)
      cudaGetLastError();
    dc.last_span_ms = span;
  }
  if (job.err_status) throw Error(job.err_status, job.err_msg);
  if (!job.all_done())
    fail(TR_ERR_RUNTIME, "run incomplete: %lld/%lld tasks", (long long)job.done_count.load(), (long long)job.n_tasks);

  if (rep) {
    rep->grid_rows = job.prods[0].grid_rows;
    rep->grid_cols = job.prods[0].grid_cols;
    rep->k_steps = job.prods[0].k_steps;
    rep->total_tasks = job.n_tasks;
    rep->wall_seconds = wall;
    rep->cache = sub_stats(dir_->stats(), before);
    rep->n_steals = static_cast<int64_t>(job.steals.size());
    rep->gpu_launches = job.launches.load();
    rep->makespan = last_makespan_;
    const auto after_dev = dir_->stats_per_device();
    for (int d = 0; d < n_devices(); ++d) {
      if (rep->cache_per_device) rep->cache_per_device[d] = sub_stats(after_dev[d], before_dev[d]);
      if (rep->devices) rep->devices[d] = devs_[d].stats;
    }
    if (rep->steals)
      for (int64_t k = 0; k < std::min<int64_t>(rep->steals_cap, rep->n_steals); ++k) rep->steals[k] = job.steals[k];
    if (rep->completion)
      for (int64_t t = 0; t < std::min<int64_t>(rep->completion_cap, job.total); ++t)
        rep->completion[t] = job.done[static_cast<size_t>(t)].load();
  }
}

void Session::span_ms(double* out) const {
  for (int d = 0; d < static_cast<int>(devs_.size()); ++d) out[d] = devs_[d].last_span_ms;
}

void Session::set_inflight(int n) {
  for (auto& dc : devs_) dc.max_inflight = std::max(1, std::min(n, dc.width));
}

void Session::kernel_ms(double* out) const {
  for (int d = 0; d < static_cast<int>(devs_.size()); ++d) out[d] = devs_[d].last_kernel_ms;
}

}  // namespace tr
