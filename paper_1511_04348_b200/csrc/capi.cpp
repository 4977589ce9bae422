// extern "C" boundary: include/tilerun_b200.h.  Every entry point catches C++
// exceptions and turns them into a tr_status plus a thread-local message.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "devpool.h"
#include "directory.h"
#include "mlp_kernels.h"
#include "msqueue.h"
#include "session.h"
#include "station.h"
#include "tile_gemm.h"

namespace tr {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
}  // namespace tr

struct tr_queue {
  tr::MSQueue q;
};
struct tr_directory {
  tr::Directory* d;
  bool owned;
};
struct tr_station {
  tr::Station s;
  tr_station(int owner, int width) : s(owner, width) {}
};
struct tr_session {
  std::unique_ptr<tr::Session> s;
  tr_directory dir;
};

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    tr::set_last_error("");
    return TR_OK;
  } catch (const tr::Error& e) {
    tr::set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    tr::set_last_error("out of host memory");
    return TR_ERR_INTERNAL;
  } catch (const std::exception& e) {
    tr::set_last_error(e.what());
    return TR_ERR_INTERNAL;
  }
}

tr::TileKey K(const tr_tile_key* k) { return tr::TileKey{k->matrix, k->row, k->col}; }
void copy_keys(const std::vector<tr::TileKey>& v, tr_tile_key* out, int64_t cap) {
  for (int64_t i = 0; i < static_cast<int64_t>(v.size()) && i < cap; ++i) {
    out[i].matrix = v[i].matrix;
    out[i].row = v[i].row;
    out[i].col = v[i].col;
  }
}

void check_dev(tr::Directory* d, int32_t dev) {
  if (dev < 0 || dev >= d->n_devices()) tr::fail(TR_ERR_CONFIG, "unknown device id %d", dev);
}

tr::Mat to_mat(const tr_matrix* m) {
  if (!m) tr::fail(TR_ERR_VALUE, "null matrix");
  tr::Mat r;
  r.ptr = m->ptr;
  r.rows = m->rows;
  r.cols = m->cols;
  r.ld = m->ld;
  r.dtype = m->dtype;
  r.location = m->location;
  if (r.dtype != TR_DTYPE_F32 && r.dtype != TR_DTYPE_F64) tr::fail(TR_ERR_VALUE, "unsupported dtype %d", r.dtype);
  if (r.location != TR_LOC_HOST && r.location != TR_LOC_DEVICE) tr::fail(TR_ERR_VALUE, "bad location %d", r.location);
  return r;
}

std::unique_ptr<tr::Directory> make_directory(const tr_machine* m, int enabled, int policy, int debug) {
  if (!m || m->n_devices < 1) tr::fail(TR_ERR_CONFIG, "machine needs at least one device");
  const int n = m->n_devices;
  std::vector<int64_t> caps(n), hops(static_cast<size_t>(n) * n);
  std::vector<bool> hw(n);
  for (int d = 0; d < n; ++d) {
    caps[d] = m->devices[d].capacity_tiles;
    hw[d] = m->devices[d].kind == TR_KIND_HOST_WORKER;
  }
  for (int64_t i = 0; i < static_cast<int64_t>(n) * n; ++i) hops[i] = m->hops ? m->hops[i] : (i % (n + 1) ? 1 : 0);
  return std::make_unique<tr::Directory>(n, caps, hw, hops, enabled != 0, policy, debug != 0);
}

}  // namespace

extern "C" {

const char* tr_last_error(void) { return tr::g_last_error.c_str(); }
int tr_abi_version(void) { return TR_ABI_VERSION; }

int tr_cuda_device_count(int32_t* out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

// ---- queue
int tr_queue_create(tr_queue** out) {
  return guarded([&] { *out = new tr_queue(); });
}
int tr_queue_destroy(tr_queue* q) {
  return guarded([&] { delete q; });
}
int tr_queue_enqueue(tr_queue* q, uint64_t v) {
  return guarded([&] { q->q.enqueue(v); });
}
int tr_queue_dequeue(tr_queue* q, uint64_t* v, int32_t* got) {
  return guarded([&] { *got = q->q.dequeue(v) ? 1 : 0; });
}
int tr_queue_is_empty(tr_queue* q, int32_t* empty) {
  return guarded([&] { *empty = q->q.is_empty() ? 1 : 0; });
}

// ---- directory
int tr_dir_create(const tr_machine* m, int32_t enabled, int32_t policy, int32_t debug, tr_directory** out) {
  return guarded([&] {
    auto d = make_directory(m, enabled, policy, debug);
    *out = new tr_directory{d.release(), true};
  });
}
int tr_dir_destroy(tr_directory* d) {
  return guarded([&] {
    if (d && d->owned) {
      delete d->d;
      delete d;
    }
  });
}
int tr_dir_lookup(tr_directory* d, int32_t requester, const tr_tile_key* key, int32_t* level, int32_t* owner) {
  return guarded([&] {
    check_dev(d->d, requester);
    *level = d->d->lookup(requester, K(key), owner);
  });
}
int tr_dir_admit(tr_directory* d, int32_t device, const tr_tile_key* key, tr_tile_key* evicted, int32_t cap,
                 int32_t* n_evicted) {
  return guarded([&] {
    check_dev(d->d, device);
    auto ev = d->d->admit(device, K(key));
    copy_keys(ev, evicted, cap);
    *n_evicted = static_cast<int32_t>(ev.size());
  });
}
int tr_dir_pin(tr_directory* d, int32_t device, const tr_tile_key* key) {
  return guarded([&] {
    check_dev(d->d, device);
    d->d->pin(device, K(key));
  });
}
int tr_dir_unpin(tr_directory* d, int32_t device, const tr_tile_key* key) {
  return guarded([&] {
    check_dev(d->d, device);
    d->d->unpin(device, K(key));
  });
}
int tr_dir_is_pinned(tr_directory* d, int32_t device, const tr_tile_key* key, int32_t* pinned) {
  return guarded([&] {
    check_dev(d->d, device);
    *pinned = d->d->is_pinned(device, K(key)) ? 1 : 0;
  });
}
int tr_dir_residents(tr_directory* d, int32_t device, tr_tile_key* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    check_dev(d->d, device);
    auto v = d->d->residents(device);
    copy_keys(v, out, cap);
    *n = static_cast<int64_t>(v.size());
  });
}
int tr_dir_used_tiles(tr_directory* d, int32_t device, int64_t* n) {
  return guarded([&] {
    check_dev(d->d, device);
    *n = d->d->used_tiles(device);
  });
}
int tr_dir_acquire_input(tr_directory* d, int32_t requester, const tr_tile_key* key, int64_t nbytes,
                         tr_acquire_result* res, tr_tile_key* evicted, int32_t cap) {
  return guarded([&] {
    check_dev(d->d, requester);
    tr::Acquired a = d->d->acquire_input(requester, K(key), nbytes);
    res->level = a.level;
    res->source = a.source;
    res->nbytes_moved = a.nbytes;
    res->n_evicted = static_cast<int32_t>(a.evicted.size());
    copy_keys(a.evicted, evicted, cap);
  });
}
int tr_dir_release_input(tr_directory* d, int32_t device, const tr_tile_key* key) {
  return guarded([&] {
    check_dev(d->d, device);
    d->d->release_input(device, K(key));
  });
}
int tr_dir_admit_output(tr_directory* d, int32_t device, const tr_tile_key* key, tr_tile_key* evicted, int32_t cap,
                        int32_t* n_evicted) {
  return guarded([&] {
    check_dev(d->d, device);
    auto ev = d->d->admit_output(device, K(key));
    copy_keys(ev, evicted, cap);
    *n_evicted = static_cast<int32_t>(ev.size());
  });
}
int tr_dir_release_output(tr_directory* d, int32_t device, const tr_tile_key* key, int64_t nbytes) {
  return guarded([&] {
    check_dev(d->d, device);
    d->d->release_output(device, K(key), nbytes);
  });
}
int tr_dir_stats(tr_directory* d, tr_cache_stats* global, tr_cache_stats* per_device) {
  return guarded([&] {
    if (global) *global = d->d->stats();
    if (per_device) {
      auto v = d->d->stats_per_device();
      for (size_t i = 0; i < v.size(); ++i) per_device[i] = v[i];
    }
  });
}
int tr_dir_check_invariants(tr_directory* d) {
  return guarded([&] { d->d->check_invariants(); });
}

// ---- stations
int tr_station_create(int32_t owner, int32_t width, tr_station** out) {
  return guarded([&] {
    if (width < 1) tr::fail(TR_ERR_CONFIG, "station width must be >= 1");
    *out = new tr_station(owner, width);
  });
}
int tr_station_destroy(tr_station* s) {
  return guarded([&] { delete s; });
}
int tr_station_refill(tr_station* s, tr_queue* q, uint64_t* pulled, int32_t cap, int32_t* n) {
  return guarded([&] {
    auto v = s->s.refill(q->q, s->s.width());
    for (int32_t i = 0; i < static_cast<int32_t>(v.size()) && i < cap; ++i) pulled[i] = v[i];
    *n = static_cast<int32_t>(v.size());
  });
}
int tr_station_pop_for_run(tr_station* s, uint64_t* tid, int32_t* got) {
  return guarded([&] { *got = s->s.pop_for_run(tid) ? 1 : 0; });
}
int tr_station_try_steal(tr_station* s, uint64_t* tid, int32_t* got) {
  return guarded([&] { *got = s->s.try_steal(tid) ? 1 : 0; });
}
int tr_station_reserved_count(tr_station* s, int32_t* n) {
  return guarded([&] { *n = s->s.reserved_count(); });
}
int tr_steal_task(int32_t thief, tr_station* const* stations, int32_t n, uint64_t* tid, int32_t* victim,
                  int32_t* got) {
  return guarded([&] {
    std::vector<tr::Station*> v;
    for (int32_t i = 0; i < n; ++i) v.push_back(&stations[i]->s);
    int vic = -1;
    *got = tr::steal_task(thief, v.data(), n, tid, &vic) ? 1 : 0;
    *victim = vic;
  });
}

// ---- session
int tr_session_create(const tr_machine* m, int32_t tile_size, int32_t precision, uint32_t flags,
                      int64_t hbm_budget_bytes, tr_session** out) {
  return guarded([&] {
    if (!m) tr::fail(TR_ERR_CONFIG, "null machine");
    int prev = -1;
    if (!(flags & TR_FLAG_DRYRUN) && cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    auto s = std::make_unique<tr_session>();
    s->s = std::make_unique<tr::Session>(*m, tile_size, precision, flags, hbm_budget_bytes);
    s->dir = tr_directory{&s->s->directory(), false};
    if (prev >= 0) cudaSetDevice(prev);
    *out = s.release();
  });
}
int tr_session_destroy(tr_session* s) {
  return guarded([&] { delete s; });
}
int tr_session_directory(tr_session* s, tr_directory** out) {
  return guarded([&] { *out = &s->dir; });
}
int tr_gemm_shard(tr_session* s, const tr_matrix* a, uint64_t a_uid, int32_t ta, const tr_matrix* b, uint64_t b_uid,
                  int32_t tb, const tr_matrix* c, uint64_t c_uid, int64_t task_offset, int64_t task_stride,
                  tr_gemm_report* report) {
  return guarded([&] {
    s->s->gemm(to_mat(a), a_uid, ta != 0, to_mat(b), b_uid, tb != 0, to_mat(c), c_uid, task_offset, task_stride,
               report);
  });
}
int tr_gemm_batch(tr_session* s, int32_t n, const tr_product* products, tr_gemm_report* report) {
  return guarded([&] {
    if (n < 1 || !products) tr::fail(TR_ERR_VALUE, "empty product batch");
    std::vector<tr::Product> v(static_cast<size_t>(n));
    for (int32_t k = 0; k < n; ++k) {
      const tr_product& q = products[k];
      tr::Product& p = v[static_cast<size_t>(k)];
      p.a = to_mat(&q.a);
      p.b = to_mat(&q.b);
      p.c = to_mat(&q.c);
      p.ta = q.transpose_a != 0;
      p.tb = q.transpose_b != 0;
      p.a_uid = q.a_uid;
      p.b_uid = q.b_uid;
      p.c_uid = q.c_uid;
      if (q.post < TR_POST_NONE || q.post > TR_POST_ACT_GRAD) tr::fail(TR_ERR_VALUE, "unknown post-op %d", q.post);
      if (q.act < TR_ACT_IDENTITY || q.act > TR_ACT_RELU) tr::fail(TR_ERR_VALUE, "unknown activation %d", q.act);
      p.post = q.post;
      p.act = q.act;
      p.bias = q.bias;
      p.aux = q.aux;
      p.ldaux = q.ldaux;
      p.cache_as = q.cache_as;
      p.axpy = q.axpy != 0;
      p.alpha = q.alpha;
      p.colsum = q.colsum;
    }
    s->s->run_products(std::move(v), 0, 1, report);
  });
}
int tr_gemm(tr_session* s, const tr_matrix* a, uint64_t a_uid, int32_t ta, const tr_matrix* b, uint64_t b_uid,
            int32_t tb, const tr_matrix* c, uint64_t c_uid, tr_gemm_report* report) {
  return tr_gemm_shard(s, a, a_uid, ta, b, b_uid, tb, c, c_uid, 0, 1, report);
}
int tr_session_lock_stats(tr_session* s, int32_t reset, int64_t* out) {
  return guarded([&] {
    if (!out) tr::fail(TR_ERR_VALUE, "null output");
    s->s->directory().mu.stats(&out[0], &out[1], &out[2], &out[3]);
    if (reset) s->s->directory().mu.reset();
  });
}
int tr_session_kernel_ms(tr_session* s, double* per_device_ms) {
  return guarded([&] { s->s->kernel_ms(per_device_ms); });
}
int tr_session_trace(tr_session* s, tr_trace_event* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    const auto& t = s->s->trace();
    for (int64_t i = 0; i < cap && i < static_cast<int64_t>(t.size()); ++i) out[i] = t[static_cast<size_t>(i)];
    *n = static_cast<int64_t>(t.size());
  });
}
int tr_session_span_ms(tr_session* s, double* per_device_ms) {
  return guarded([&] { s->s->span_ms(per_device_ms); });
}
int tr_session_sim_now(tr_session* s, double* out) {
  return guarded([&] { *out = s->s->sim_now(); });
}
int tr_session_set_inflight(tr_session* s, int32_t max_inflight) {
  return guarded([&] {
    if (max_inflight < 1) tr::fail(TR_ERR_VALUE, "max_inflight must be >= 1");
    s->s->set_inflight(max_inflight);
  });
}

// ---- dense in-core product
int tr_dense_gemm(const tr_matrix* a, int32_t ta, const tr_matrix* b, int32_t tb, const tr_matrix* c,
                  int32_t precision, int32_t accumulate, void* stream) {
  return guarded([&] {
    tr::Mat A = to_mat(a), B = to_mat(b), C = to_mat(c);
    if (A.location != TR_LOC_DEVICE || B.location != TR_LOC_DEVICE || C.location != TR_LOC_DEVICE)
      tr::fail(TR_ERR_VALUE, "tr_dense_gemm takes device matrices");
    const int64_t M = ta ? A.cols : A.rows, K = ta ? A.rows : A.cols;
    const int64_t Kb = tb ? B.cols : B.rows, N = tb ? B.rows : B.cols;
    if (K != Kb) tr::fail(TR_ERR_SHAPE, "inner dimensions differ");
    if (C.rows != M || C.cols != N) tr::fail(TR_ERR_SHAPE, "output shape mismatch");
    // as the reference's matrices (tiles.py as_matrix): every dimension >= 1
    if (M < 1 || N < 1 || K < 1)
      tr::fail(TR_ERR_SHAPE, "matrix dimensions must be >= 1, got %lld x %lld x %lld", static_cast<long long>(M),
               static_cast<long long>(K), static_cast<long long>(N));
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) tr::fail(TR_ERR_SHAPE, "dimension too large");
    if (precision != TR_PREC_BF16 && precision != TR_PREC_FP32ACC && precision != TR_PREC_EXACT &&
      precision != TR_PREC_FP32HI)
      tr::fail(TR_ERR_VALUE, "unknown precision");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (precision == TR_PREC_EXACT) {  // KX over float64 copies of A and B (one row stride for both)
      const int64_t ld = (std::max(A.cols, B.cols) + 7) / 8 * 8;
      double *xa = nullptr, *xb = nullptr;
      TR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xa), static_cast<size_t>(A.rows * ld * 8), st));
      TR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xb), static_cast<size_t>(B.rows * ld * 8), st));
      TR_CUDA(tr::launch_exact_convert(A.ptr, A.dtype == TR_DTYPE_F64, A.ld, A.rows, A.cols, xa, ld, st));
      TR_CUDA(tr::launch_exact_convert(B.ptr, B.dtype == TR_DTYPE_F64, B.ld, B.rows, B.cols, xb, ld, st));
      tr::GemmArgs x;
      std::memset(&x, 0, sizeof(x));
      x.m_valid = static_cast<int32_t>(M);
      x.n_valid = static_cast<int32_t>(N);
      x.n_ksteps = 1;
      x.k_len[0] = static_cast<int32_t>(K);
      x.c = const_cast<void*>(C.ptr);
      x.ldc = C.ld;
      x.c_f64 = C.dtype == TR_DTYPE_F64;
      x.epilogue = accumulate ? tr::EPI_ACCUMULATE : tr::EPI_STORE;
      TR_CUDA(tr::launch_exact_gemm(xa, xb, ld, 0, x, ta != 0, tb != 0,
                                    A.dtype == TR_DTYPE_F32 && B.dtype == TR_DTYPE_F32, st));
      TR_CUDA(cudaFreeAsync(xa, st));
      TR_CUDA(cudaFreeAsync(xb, st));
      return;
    }
    const int planes = precision == TR_PREC_FP32HI ? 3 : precision == TR_PREC_FP32ACC ? 2 : 1;
    auto pack = [&](const tr::Mat& m, uint16_t** buf, tr::PlaneGeom* g) {
      const int64_t ld = (m.cols + 7) / 8 * 8;
      const int64_t pe = m.rows * ld;
      TR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(buf), static_cast<size_t>(planes * pe * 2), st));
      TR_CUDA(tr::launch_split_convert(m.ptr, m.dtype == TR_DTYPE_F64, m.ld, m.rows, m.cols, *buf, ld, m.rows, pe,
                                       planes, st));
      g->base = *buf;
      g->cols = m.cols;
      g->rows = m.rows;
      g->nplanes = planes;
      g->ld = ld;
      g->plane_stride = pe;
    };
    uint16_t *pa = nullptr, *pb = nullptr;
    tr::PlaneGeom ga, gb;
    pack(A, &pa, &ga);
    pack(B, &pb, &gb);
    tr::BoxKind ba, bb;
    tr::gemm_boxes(ta != 0, tb != 0, static_cast<int>(M), &ba, &bb);
    CUtensorMap tma, tmb;
    if (tr::make_plane_tmap(&tma, ga, ba) || tr::make_plane_tmap(&tmb, gb, bb))
      tr::fail(TR_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    tr::GemmArgs args;
    std::memset(&args, 0, sizeof(args));
    args.m_valid = static_cast<int32_t>(M);
    args.n_valid = static_cast<int32_t>(N);
    args.n_ksteps = 1;
    args.planes = planes;
    args.a_z[0] = 0;
    args.b_z[0] = 0;
    args.k_len[0] = static_cast<int32_t>(K);
    args.c = const_cast<void*>(C.ptr);
    args.ldc = C.ld;
    args.c_f64 = C.dtype == TR_DTYPE_F64;
    args.epilogue = accumulate ? tr::EPI_ACCUMULATE : tr::EPI_STORE;
    args.seg_kb = tr::seg_kb_for(planes);
    TR_CUDA(tr::launch_tile_gemm(tma, tmb, args, ta != 0, tb != 0, st));
    TR_CUDA(cudaFreeAsync(pa, st));
    TR_CUDA(cudaFreeAsync(pb, st));
  });
}

int tr_session_set_order(tr_session* s, int32_t order) {
  return guarded([&] {
    if (order < -1 || order > 4)
      tr::fail(TR_ERR_VALUE,
               "order must be -1 (auto), 0 (row-major), 1 (banded), 2 (shells), 3 (blocked) or 4 (k-panels)");
    s->s->set_order(order);
  });
}
int tr_release_cached_memory(void) {
  return guarded([&] { tr::DevPool::get().trim(); });
}
int tr_mlp_bias_act(float* y, float* a, const float* bias, int64_t rows, int64_t cols, int32_t act, void* stream) {
  return guarded([&] { TR_CUDA(tr::mlp_bias_act(y, a, bias, rows, cols, act, static_cast<cudaStream_t>(stream))); });
}
int tr_mlp_act_grad(float* dy, const float* dout, const float* y, const float* a, int64_t n, int32_t act,
                    void* stream) {
  return guarded([&] { TR_CUDA(tr::mlp_act_grad(dy, dout, y, a, n, act, static_cast<cudaStream_t>(stream))); });
}
int tr_mlp_mse_grad(float* dout, const float* pred, const float* target, int64_t n, double* loss_sum,
                    void* stream) {
  return guarded(
      [&] { TR_CUDA(tr::mlp_mse_grad(dout, pred, target, n, n, loss_sum, static_cast<cudaStream_t>(stream))); });
}
int tr_mlp_mse_grad_global(float* dout, const float* pred, const float* target, int64_t n, int64_t n_global,
                           double* loss_sum, void* stream) {
  return guarded([&] {
    if (n_global < n) tr::fail(TR_ERR_VALUE, "n_global (%lld) < n (%lld)", (long long)n_global, (long long)n);
    TR_CUDA(tr::mlp_mse_grad(dout, pred, target, n, n_global, loss_sum, static_cast<cudaStream_t>(stream)));
  });
}
int tr_mlp_colsum(const float* m, int64_t rows, int64_t cols, float* out, void* stream) {
  return guarded([&] { TR_CUDA(tr::mlp_colsum(m, rows, cols, out, static_cast<cudaStream_t>(stream))); });
}
int tr_mlp_colsum_finish(const float* part, int64_t n_blocks, int64_t cols, float* out, void* stream) {
  return guarded([&] {
    TR_CUDA(tr::mlp_colsum_finish(part, n_blocks, cols, out, static_cast<cudaStream_t>(stream)));
  });
}
int tr_mlp_sgd(float* w, const float* g, int64_t n, float lr, void* stream) {
  return guarded([&] { TR_CUDA(tr::mlp_sgd(w, g, n, lr, static_cast<cudaStream_t>(stream))); });
}
int tr_session_forget(tr_session* s, uint64_t uid, int64_t* dropped) {
  return guarded([&] {
    tr::DirLock g(s->s->directory().mu);
    const int64_t n = s->s->directory().forget_locked(uid);
    if (dropped) *dropped = n;
  });
}
int tr_session_set_external_stream(tr_session* s, void* stream, int enabled) {
  return guarded([&] { s->s->set_external_stream(static_cast<cudaStream_t>(stream), enabled != 0); });
}

int tr_session_set_async(tr_session* s, int on) {
  return guarded([&] { s->s->set_async(on != 0); });
}
int tr_set_gemm_pairs(int32_t on) {
  return guarded([&] { tr::set_gemm_pairs(on != 0); });
}

int tr_set_gemm_multicast(int32_t on) {
  return guarded([&] { tr::set_gemm_multicast(on != 0); });
}
int tr_k1_die_map(int32_t gpu, int32_t* n0, int32_t* n1) {
  return guarded([&] {
    if (!n0 || !n1) tr::fail(TR_ERR_VALUE, "null output");
    *n0 = *n1 = 0;
    tr::die_map_prepare(gpu);
    int a = 0, b = 0;
    if (tr::die_map_ready(gpu, &a, &b)) {
      *n0 = a;
      *n1 = b;
    }
  });
}
int tr_set_task_group(int32_t max_tasks) {
  return guarded([&] {
    if (max_tasks < 1 || max_tasks > tr::kMaxGroup) tr::fail(TR_ERR_VALUE, "task group must be in 1..%d", tr::kMaxGroup);
    tr::set_task_group_max(max_tasks);
  });
}

int tr_set_splitk(int32_t max_splits) {
  return guarded([&] {
    if (max_splits < 1 || max_splits > 8) tr::fail(TR_ERR_VALUE, "split-K factor must be in 1..8");
    tr::set_splitk_max(max_splits);
  });
}

int tr_set_small_gemm(int32_t on) {
  return guarded([&] { tr::set_small_gemm(on != 0); });
}

int tr_set_narrow_tc(int32_t on) {
  return guarded([&] { tr::set_narrow_tc(on != 0); });
}

}  // extern "C"
