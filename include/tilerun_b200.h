/*
 * tilerun_b200 — C ABI of the B200-native out-of-core tiled GEMM runtime.
 *
 * This is the drop-in boundary for the reference package `tilerun`
 * (/root/reference/pkg/src/tilerun).  The reference is pure Python; its
 * "FFI" for this path is its public Python API, so every entry point below
 * names the reference symbol it replaces (file:line under pkg/src/tilerun/).
 * The Python mirror (paper_1511_04348_b200/) binds these with ctypes; the
 * binding a maintainer of the reference would add is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Every function returns int status (tr_status).  On failure the
 *     thread-local message is available from tr_last_error().
 *   - Plain pointers and sizes only; no torch / numpy types.
 *   - Matrices are row-major, described by tr_matrix.  Host matrices should be
 *     pinned (cudaHostAlloc / cudaHostRegister) for full H2D/D2H bandwidth; the
 *     runtime registers unpinned host ranges for the duration of a call.
 *   - Tile identity is (matrix uid, tile row, tile col) in STORED coordinates,
 *     as in scheduler.py:99-138 (Operand).  A uid must name immutable content
 *     for the lifetime of the session (ann.py:138-140,247).
 */
#ifndef TILERUN_B200_H
#define TILERUN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TR_ABI_VERSION 1

/* ---------------------------------------------------------------- status */
typedef enum {
  TR_OK = 0,
  TR_ERR_CONFIG = 1,     /* devices.py:26-27  ConfigError(ValueError)            */
  TR_ERR_SHAPE = 2,      /* ValueError: shape / tile / mode (tiles.py:57-58,165-168; scheduler.py:173-180) */
  TR_ERR_CAPACITY = 3,   /* coherence.py:33-34 CapacityError(RuntimeError)       */
  TR_ERR_RUNTIME = 4,    /* RuntimeError: incomplete run / double execution (scheduler.py:80-81,587-590) */
  TR_ERR_CUDA = 5,       /* CUDA runtime / driver failure (RuntimeError)        */
  TR_ERR_VALUE = 6,      /* other ValueError (pin/unpin misuse, duplicate admit, bad enum) */
  TR_ERR_INTERNAL = 7,   /* invariant violation (AssertionError in coherence.py:300-313) */
  TR_ERR_NODEVICE = 8    /* no CUDA device / driver: the product path cannot run */
} tr_status;

typedef enum { TR_DTYPE_F32 = 0, TR_DTYPE_F64 = 1 } tr_dtype;
typedef enum { TR_LOC_HOST = 0, TR_LOC_DEVICE = 1 } tr_location;

/* Arithmetic of the tile kernel.  FP32ACC: each fp32/f64 tile is split once at
 * admission into bf16 hi + lo planes and every k-block issues hi*lo + lo*hi +
 * hi*hi tcgen05 MMAs into an fp32 TMEM accumulator.  BF16: one plane, one MMA. */
/* TR_PREC_EXACT: the reference's own arithmetic (a rounded multiply then a
 * rounded add per rank-1 update, k ascending, in the output dtype) on CUDA
 * cores: results bit for bit the reference's; tiles cached as float64.
 * TR_PREC_FP32HI: three bf16 planes (hi, mid, lo: all 24 bits of an fp32
 * value) and the six MMAs of weight >= 2^-16 per k-block -- about 10x more
 * accurate than FP32ACC at twice its tensor work. */
typedef enum { TR_PREC_BF16 = 0, TR_PREC_FP32ACC = 1, TR_PREC_EXACT = 2, TR_PREC_FP32HI = 3 } tr_precision;

typedef enum { TR_POLICY_LRU = 0, TR_POLICY_FIFO = 1 } tr_policy; /* coherence.py:95-99 */
typedef enum { TR_HIT_L1 = 0, TR_HIT_L2 = 1, TR_HIT_MISS = 2 } tr_hit_level; /* coherence.py:37-40 */
#define TR_SOURCE_HOST (-1)                                              /* devices.py:20 HOST */
typedef enum { TR_KIND_ACCELERATOR = 0, TR_KIND_HOST_WORKER = 1 } tr_device_kind; /* devices.py:17-18 */

/* -------------------------------------------------------------- library */
const char* tr_last_error(void);
int tr_abi_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int tr_cuda_device_count(int32_t* out);

/* ------------------------------------------------ task queue (msqueue.py:28-67)
 * Lock-free Michael–Scott MPMC FIFO of uint64 values (counted-pointer CAS).
 * Replaces MichaelScottQueue.{enqueue,dequeue,is_empty} (msqueue.py:36-58). */
typedef struct tr_queue tr_queue;
int tr_queue_create(tr_queue** out);
int tr_queue_destroy(tr_queue* q);
int tr_queue_enqueue(tr_queue* q, uint64_t value);
/* *got = 1 and *value set when an element was dequeued, *got = 0 when empty. */
int tr_queue_dequeue(tr_queue* q, uint64_t* value, int32_t* got);
int tr_queue_is_empty(tr_queue* q, int32_t* empty);

/* ------------------------------------- machine description (devices.py:30-216) */
typedef struct {
  int32_t device_id;      /* DeviceSpec.device_id (devices.py:43)                       */
  int32_t kind;           /* tr_device_kind; host workers only in TR_FLAG_SIM sessions    */
  int64_t capacity_tiles; /* DeviceSpec.capacity_tiles; -1 = unbounded (HBM-budget bound)  */
  int32_t slots;          /* reservation-station width (devices.py:49), = CUDA streams   */
  int32_t gpu;            /* physical CUDA ordinal; -1 = device_id % visible GPUs        */
  double flops_per_unit;  /* simulated engine: flops per time unit (devices.py:255-261)   */
  double host_bandwidth;  /* simulated engine: bytes per time unit to/from host (264-283) */
  int32_t sm_count;       /* > 0: the logical device runs on a green context of this many
                             SMs of its GPU (disjoint from the GPU's other such devices);
                             0 = the whole GPU.  Inhomogeneous devices on one GPU.       */
} tr_device_spec;

typedef struct {
  int32_t n_devices;
  const tr_device_spec* devices;
  const int64_t* hops;    /* n x n ProximityMatrix.hops (devices.py:78-118)             */
  int32_t element_bytes;  /* Machine.element_bytes (devices.py:145-154): byte accounting */
  const double* peer_bandwidth; /* n x n ProximityMatrix.peer_bandwidth (simulated engine; may be NULL) */
  double transfer_latency;      /* Machine.transfer_latency (simulated engine)                  */
} tr_machine;

/* ----------------------------------- cache directory (coherence.py:86-313) */
typedef struct {
  uint64_t matrix; /* interned uid */
  int64_t row;
  int64_t col;
} tr_tile_key; /* tiles.py:29-34 TileKey */

typedef struct {
  int64_t l1_hits, l2_hits, host_fetches, bytes_host, bytes_peer, evictions, writebacks, bytes_writeback;
} tr_cache_stats; /* coherence.py:59-83 CacheStats, field for field */

typedef struct {
  int32_t level;  /* tr_hit_level */
  int32_t source; /* device id or TR_SOURCE_HOST */
  int64_t nbytes_moved;
  int32_t n_evicted;
} tr_acquire_result; /* coherence.py:49-56 AcquireResult */

typedef struct tr_directory tr_directory;
/* CacheDirectory(machine, enabled, policy, debug)  coherence.py:95-114 */
int tr_dir_create(const tr_machine* m, int32_t enabled, int32_t policy, int32_t debug, tr_directory** out);
int tr_dir_destroy(tr_directory* d);
/* lookup  coherence.py:118-134 (owner = -1 unless L2) */
int tr_dir_lookup(tr_directory* d, int32_t requester, const tr_tile_key* key, int32_t* level, int32_t* owner);
/* admit  coherence.py:136-174; evicted keys copied to `evicted` (capacity `cap`) */
int tr_dir_admit(tr_directory* d, int32_t device, const tr_tile_key* key, tr_tile_key* evicted, int32_t cap,
                 int32_t* n_evicted);
int tr_dir_pin(tr_directory* d, int32_t device, const tr_tile_key* key);   /* 176-180 */
int tr_dir_unpin(tr_directory* d, int32_t device, const tr_tile_key* key); /* 182-192 */
int tr_dir_is_pinned(tr_directory* d, int32_t device, const tr_tile_key* key, int32_t* pinned);
int tr_dir_residents(tr_directory* d, int32_t device, tr_tile_key* out, int64_t cap, int64_t* n);
int tr_dir_used_tiles(tr_directory* d, int32_t device, int64_t* n);
/* acquire_input  coherence.py:210-246 */
int tr_dir_acquire_input(tr_directory* d, int32_t requester, const tr_tile_key* key, int64_t nbytes,
                         tr_acquire_result* res, tr_tile_key* evicted, int32_t cap);
int tr_dir_release_input(tr_directory* d, int32_t device, const tr_tile_key* key);           /* 248-252 */
int tr_dir_admit_output(tr_directory* d, int32_t device, const tr_tile_key* key, tr_tile_key* evicted,
                        int32_t cap, int32_t* n_evicted);                                        /* 254-261 */
int tr_dir_release_output(tr_directory* d, int32_t device, const tr_tile_key* key, int64_t nbytes); /* 263-280 */
int tr_dir_stats(tr_directory* d, tr_cache_stats* global, tr_cache_stats* per_device /* n_devices */);
int tr_dir_check_invariants(tr_directory* d); /* 296-313 */

/* ------------------- reservation stations + stealing (scheduler.py:200-249) */
typedef struct tr_station tr_station;
int tr_station_create(int32_t owner, int32_t width, tr_station** out);
int tr_station_destroy(tr_station* s);
/* refill from `q` until full; pulled ids copied out (scheduler.py:214-224) */
int tr_station_refill(tr_station* s, tr_queue* q, uint64_t* pulled, int32_t cap, int32_t* n);
int tr_station_pop_for_run(tr_station* s, uint64_t* tid, int32_t* got); /* front, 226-228 */
int tr_station_try_steal(tr_station* s, uint64_t* tid, int32_t* got);   /* back, 230-232 */
int tr_station_reserved_count(tr_station* s, int32_t* n);
/* steal_task  scheduler.py:239-249: victim = most reserved, ties to lowest id. */
int tr_steal_task(int32_t thief, tr_station* const* stations, int32_t n, uint64_t* tid, int32_t* victim,
                  int32_t* got);

/* ------------------------------------------ session (scheduler.py:522-621) */
typedef struct tr_session tr_session;

enum {
  TR_FLAG_STEAL = 1u << 0,     /* Runtime(steal=True)                                  */
  TR_FLAG_COHERENCE = 1u << 1, /* Runtime(coherence=True); off = bypass (2g^3 host)     */
  TR_FLAG_DEBUG = 1u << 2,     /* Runtime(directory_debug=True): invariants per mutation */
  TR_FLAG_DRYRUN = 1u << 3,    /* schedule-only test mode: no CUDA, no arithmetic, C untouched */
  TR_FLAG_FIFO = 1u << 4,      /* FIFO eviction instead of LRU                          */
  TR_FLAG_NO_PREFETCH = 1u << 5, /* disable fetch-ahead of reserved tasks' input tiles  */
  TR_FLAG_TRACE = 1u << 6,      /* record a device timeline of every copy/kernel (tr_session_trace) */
  TR_FLAG_SIM = 1u << 7         /* simulated engine (scheduler.py:432-464): the reference's deterministic
                                   event order and cost model, per-device clocks persisting across calls,
                                   host workers allowed; no CUDA, no arithmetic (implies DRYRUN) */
};

typedef struct {
  const void* ptr; /* host or device base pointer                          */
  int64_t rows, cols;
  int64_t ld;      /* elements between rows (>= cols)                         */
  int32_t dtype;   /* tr_dtype                                                */
  int32_t location;/* tr_location                                             */
} tr_matrix;

typedef struct {
  int64_t tasks_completed, steals_performed, steals_suffered; /* scheduler.py:261-267 */
  int64_t peer_copies_served; /* B200 addition: L2 fills this device sourced over NVLink / D2D */
  int64_t macs;               /* B200 addition: sum over completed tasks of rows x cols x K (work share) */
} tr_device_stats;

typedef struct {
  int32_t thief, victim;
  int64_t task_id;
  double time;    /* simulated time of the steal (TR_FLAG_SIM sessions), else 0 */
} tr_steal_event; /* scheduler.py:252-258 (queue_empty_observed is always true) */

typedef struct {
  /* outputs filled by tr_gemm */
  int64_t grid_rows, grid_cols, k_steps, total_tasks;
  double wall_seconds;
  tr_cache_stats cache;            /* per-call delta (scheduler.py:576-607) */
  int64_t n_steals;                /* total steal events (may exceed steals_cap) */
  int64_t gpu_launches;            /* kernels launched by this call                 */
  /* caller-provided arrays (may be NULL) */
  tr_cache_stats* cache_per_device; /* n_devices */
  tr_device_stats* devices;         /* n_devices */
  tr_steal_event* steals;           /* steals_cap entries */
  int64_t steals_cap;
  uint8_t* completion;              /* total_tasks bytes: exactly-once bitmap snapshot */
  int64_t completion_cap;
  double makespan;                  /* TR_FLAG_SIM: simulated time of this call (scheduler.py:602), else 0 */
} tr_gemm_report;

/* Runtime(machine, tile_size, mode, steal, coherence, seed, directory_debug)
 * (scheduler.py:531-546).  hbm_budget_bytes: per-GPU bytes the tile cache may
 * occupy (0 = 80% of free memory at creation). */
int tr_session_create(const tr_machine* m, int32_t tile_size, int32_t precision, uint32_t flags,
                      int64_t hbm_budget_bytes, tr_session** out);
int tr_session_destroy(tr_session* s);
/* Borrowed pointer to the session's directory (Runtime.directory). */
int tr_session_directory(tr_session* s, tr_directory** out);
/* Runtime.multiply(a, b, transpose_a, transpose_b, a_uid, b_uid, c_uid)  scheduler.py:559-612:
 * plans one task per C tile (row-major ids, plan() scheduler.py:165-197), runs one
 * pinned worker thread per device (_run_threaded scheduler.py:467-516) whose
 * reservation-station slots are CUDA streams, and blocks until every task executed
 * exactly once.  `c` must be zero-initialised storage of a.rows x b.cols (after
 * transposition) of c->dtype; it is fully overwritten. */
int tr_gemm(tr_session* s, const tr_matrix* a, uint64_t a_uid, int32_t transpose_a, const tr_matrix* b,
            uint64_t b_uid, int32_t transpose_b, const tr_matrix* c, uint64_t c_uid, tr_gemm_report* report);
/* Partial product for static multi-process sharding: only tasks t with
 * t % task_stride == task_offset are planned (all others are left untouched). */
int tr_gemm_shard(tr_session* s, const tr_matrix* a, uint64_t a_uid, int32_t transpose_a, const tr_matrix* b,
                  uint64_t b_uid, int32_t transpose_b, const tr_matrix* c, uint64_t c_uid, int64_t task_offset,
                  int64_t task_stride, tr_gemm_report* report);
/* A batch of INDEPENDENT products scheduled as one round (their tasks interleave
 * on the devices' streams; no product may read another's output).  Each may
 * carry a fused epilogue post-op for float32 DEVICE outputs (MLP training):
 *   TR_POST_BIAS_ACT  C = act(A.B + bias[col])        forward layer, ann.py:155-158
 *   TR_POST_ACT_GRAD  C = (A.B) * act'(aux[row, col])  dX of layer l+1 times the
 *                     activation derivative of layer l = dY of layer l, ann.py:171,222
 * act' is taken from the activation OUTPUT (sigmoid: a(1-a), relu: a > 0). */
typedef enum { TR_POST_NONE = 0, TR_POST_BIAS_ACT = 1, TR_POST_ACT_GRAD = 2 } tr_post_op;
typedef struct {
  tr_matrix a;
  uint64_t a_uid;
  int32_t transpose_a;
  tr_matrix b;
  uint64_t b_uid;
  int32_t transpose_b;
  tr_matrix c;
  uint64_t c_uid;
  int32_t post;        /* tr_post_op */
  int32_t act;         /* tr_activation of the post-op */
  const float* bias;   /* TR_POST_BIAS_ACT: c.cols floats (device), may be NULL */
  const float* aux;    /* TR_POST_ACT_GRAD: c.rows x c.cols activation output (device) */
  int64_t ldaux;
  uint64_t cache_as;   /* != 0: the result will be read as an INPUT under this uid (e.g. the next
                          layer's activations); the producing kernel also writes its converted
                          tiles straight into the tile cache (float32 device outputs, full tiles;
                          uncounted until requested, like a fetch-ahead), saving the later
                          split/convert pass.  0 = off. */
  int32_t axpy;        /* != 0: C += alpha * A.B (float32 device C, post-op NONE) -- e.g. the fused SGD
                          update W += (-lr) X^T dY of ann.py:247 without a gradient buffer */
  float alpha;
  float* colsum;       /* != NULL: column sums of the FINAL output (after the post-op) per 32-row
                          block, colsum[(r / 32) * c.cols + col] = sum of C[r..r+31][col] (rows in
                          order); finish with tr_mlp_colsum_finish -- the bias gradient
                          db = colsum(dY) of ann.py:173 without a pass over dY.  ceil(c.rows/32)
                          x c.cols floats (device); float32 device C; tile size a multiple of 32. */
} tr_product;
int tr_gemm_batch(tr_session* s, int32_t n, const tr_product* products, tr_gemm_report* report);
/* Device-side duration (ms) of the last tr_gemm's GEMM kernels on each device,
 * measured with CUDA events on the launching streams (sum over launches). */
int tr_session_kernel_ms(tr_session* s, double* per_device_ms /* n_devices */);
/* The directory lock's accounting since the last reset: out[0] ns held, out[1] ns
 * callers waited to acquire it, out[2] acquisitions, out[3] longest hold (ns).
 * reset != 0 zeroes it after reading.  B200 addition (coherence.py:202-209 makes
 * every directory operation one critical section; this measures its cost). */
int tr_session_lock_stats(tr_session* s, int32_t reset, int64_t* out /* 4 */);
/* Timeline of the last tr_gemm (sessions created with TR_FLAG_TRACE): one entry
 * per H2D tile copy, split/convert, peer copy, GEMM launch and D2H writeback,
 * with CUDA-event times in ms relative to the product's start on that device. */
typedef enum { TR_TRACE_H2D = 0, TR_TRACE_CONVERT = 1, TR_TRACE_PEER = 2, TR_TRACE_GEMM = 3, TR_TRACE_D2H = 4 } tr_trace_kind;
typedef struct {
  int32_t device, kind, stream;
  int64_t task;           /* task id (GEMM, D2H) or -1 */
  uint64_t matrix;        /* tile uid (copies, converts) or 0 */
  int64_t row, col;
  double start_ms, end_ms;
} tr_trace_event;
int tr_session_trace(tr_session* s, tr_trace_event* out, int64_t cap, int64_t* n);
/* Device-side span (ms) of the last tr_gemm on each device: CUDA events recorded
 * before the first and after the last operation of every worker stream. */
int tr_session_span_ms(tr_session* s, double* per_device_ms /* n_devices */);
/* TR_FLAG_SIM sessions: max over devices of their compute / transfer clocks
 * (Runtime.sim_now, scheduler.py:552-553); 0 for other sessions. */
int tr_session_sim_now(tr_session* s, double* out);
/* Tasks a device keeps executing concurrently (default min(2, slots)); the rest
 * of its reservation-station entries stay reserved (stealable).  1 serialises
 * a device's tasks, which the roofline measurement uses. */
int tr_session_set_inflight(tr_session* s, int32_t max_inflight);
/* Order in which tr_gemm enqueues task ids: 0 = row-major (the reference's,
 * scheduler.py:189-192), 1 = banded (pairs of task rows walked column by
 * column), 2 = shells (tasks with max(i,j) = s before shell s+1: first-touch
 * host traffic spread over the run), 3 = blocked (b x b task blocks whose
 * 2b k-panels fit the smallest device tile budget: out-of-core reuse),
 * -1 = auto (default): row-major if some device has a bounded capacity (LRU
 * eviction sequences -- and so the counters -- then match the reference),
 * blocked if A+B exceed the HBM tile budget, shells otherwise. */
int tr_session_set_order(tr_session* s, int32_t order);
/* Sessions return HBM slabs/staging buffers to a process-wide cache reused by
 * later sessions; this frees every cached block. */
int tr_release_cached_memory(void);

/* ------------------------------- dense in-core product (ann.py:62-75 DenseBackend)
 * One K1 launch over whole matrices on the current CUDA device, no scheduler and
 * no tile cache: a, b, c are DEVICE matrices.  accumulate: c += a@b.  `stream`
 * is a cudaStream_t (NULL = legacy default stream). */
int tr_dense_gemm(const tr_matrix* a, int32_t transpose_a, const tr_matrix* b, int32_t transpose_b,
                  const tr_matrix* c, int32_t precision, int32_t accumulate, void* stream);

/* ------------------------------ MLP elementwise kernels (ann.py:30-56,151-248)
 * Device float32 arrays, launched on `stream` (cudaStream_t).  These replace the
 * reference's host float64 numpy steps around the products. */
typedef enum { TR_ACT_IDENTITY = 0, TR_ACT_SIGMOID = 1, TR_ACT_RELU = 2 } tr_activation; /* ann.py:27 */
/* y += bias (per column; bias may be NULL); a = act(y)      ann.py:155-158 */
int tr_mlp_bias_act(float* y, float* a, const float* bias, int64_t rows, int64_t cols, int32_t act, void* stream);
/* dy = dout * act'(a) from the activation output a (y unused, may be NULL)  ann.py:222, 40-48 */
int tr_mlp_act_grad(float* dy, const float* dout, const float* y, const float* a, int64_t n, int32_t act,
                    void* stream);
/* dout = 2 (pred - target) / n; *loss_sum (device double) = sum (pred - target)^2, summed in a
 * fixed order (bitwise reproducible)                          ann.py:51-56 */
int tr_mlp_mse_grad(float* dout, const float* pred, const float* target, int64_t n, double* loss_sum,
                    void* stream);
/* Data-parallel form: this rank holds n of the batch's n_global elements;
 * dout = 2 (pred - target) / n_global, so summing dout-derived gradients over
 * the ranks gives the full-batch gradient; *loss_sum = this shard's sum. */
int tr_mlp_mse_grad_global(float* dout, const float* pred, const float* target, int64_t n, int64_t n_global,
                           double* loss_sum, void* stream);
/* out[c] = sum_r m[r, c], fixed summation order (reproducible)   ann.py:173 */
int tr_mlp_colsum(const float* m, int64_t rows, int64_t cols, float* out, void* stream);
/* out[c] = sum over b < n_blocks of part[b * cols + c], blocks in order (tr_product.colsum). */
int tr_mlp_colsum_finish(const float* part, int64_t n_blocks, int64_t cols, float* out, void* stream);
/* w -= lr * g                                                ann.py:243-247 */
int tr_mlp_sgd(float* w, const float* g, int64_t n, float lr, void* stream);

/* Drop every resident tile of matrix `uid` from the session's tile cache on all
 * devices (the uid's content is dead, e.g. a retired weight version, ann.py:247).
 * Not counted as an eviction.  The reference has no equivalent: its unbounded
 * caches keep stale versions forever. */
int tr_session_forget(tr_session* s, uint64_t uid, int64_t* dropped);

/* enabled != 0: order every product of the session after the work already queued
 * on `stream` (a cudaStream_t, e.g. the caller's framework stream; NULL is the
 * legacy default stream).  enabled == 0 clears it. */
int tr_session_set_external_stream(tr_session* s, void* stream, int enabled);

/* Stream-ordered products (1) or blocking products (0, default; the reference's
 * semantics, scheduler.py:587-590).  When on, a product whose operands are ALL
 * in device memory, run with an external stream set and tracing off, returns
 * once every task is enqueued: the external stream waits for the product, and
 * the next product starts after the external stream's queued work.  The report's
 * counters and completion bitmap are final on return; per-launch kernel times
 * and the device span are not measured (0).  Any other product blocks as usual. */
int tr_session_set_async(tr_session* s, int on);

/* Kernel variant switch (process-wide): 1 = CTA pairs (tcgen05 cta_group::2,
 * 256 x 256 per pair) for tiles taller than 128 rows, 0 = single CTAs
 * (128 x 256, default).  Also settable with TR_GEMM_PAIRS=1 in the environment. */
int tr_set_gemm_pairs(int32_t on);
/* Grouped launches as TMA-multicast clusters of two CTA pairs sharing their A
 * tile (0 = off, the default; TR_GEMM_MC=1).  Measured slower on B200: only 33
 * such clusters (132 SMs) are co-resident against 74 pairs (148 SMs). */
int tr_set_gemm_multicast(int32_t on);
/* K1's die map of GPU `gpu` (measured once per process, at the first session on
 * that GPU, or here): *n0 / *n1 = CTA-pair clusters expected on each die of a
 * persistent launch; both 0 when not measured or not usable (TR_K1_DIE=0
 * disables it).  Grouped persistent launches then give each die a compact block
 * of output units. */
int tr_k1_die_map(int32_t gpu, int32_t* n0, int32_t* n1);

/* Split-K policy (process-wide): at most `max_splits` (1..8) K-splits per tile
 * GEMM launch whose output has fewer 128 x 256 blocks than the GPU has SMs
 * (partials reduced in a fixed order: deterministic).  1 disables.  Default 8,
 * or TR_SPLITK=<n> in the environment. */
int tr_set_splitk(int32_t max_splits);

/* CUDA-core tile GEMM (process-wide): tasks whose output tile is at most 32
 * columns wide, or whose total contraction is at most 32, run on a CUDA-core
 * kernel instead of a mostly padded 128 x 256 tensor-core tile (the MLP's
 * 10-wide output layer).  Default on; 0 sends every task to the tensor cores;
 * TR_SMALL_GEMM=0 in the environment sets the default. */
int tr_set_small_gemm(int32_t on);

/* Narrow outputs on the tensor cores (process-wide): a task whose output tile
 * is at most 32 columns wide (contraction longer than 32) runs as the
 * transposed product Bᵀ·Aᵀ -- its long side on the MMA's N dimension -- split
 * along k, and a reduction writes C.  Default on; 0 leaves such tasks to the
 * CUDA-core kernel; TR_NARROW_TC=0 in the environment sets the default. */
int tr_set_narrow_tc(int32_t on);

/* Grouped launches (process-wide, sessions created afterwards): up to
 * `max_tasks` (1..8) ready tasks of one product from a device's reservation
 * station run as ONE tile-GEMM launch (device outputs, unchunked tasks).  Each
 * task keeps its own directory sequence; 1 disables.  Default 4, or TR_GROUP=<n>. */
int tr_set_task_group(int32_t max_tasks);

#ifdef __cplusplus
}
#endif

#endif /* TILERUN_B200_H */
