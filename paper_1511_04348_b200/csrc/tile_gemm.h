// K1: the per-task tile GEMM  C[i,j] (+)= sum_k A[i,k] . B[k,j]  on sm_100a.
//
// Replaces the reference's per-k-step numpy kernel
//   tiles.py:154-179  accumulate_product  (called per k-step, scheduler.py:393-404)
// with ONE launch per task (or per chunk of k-steps when the tile cache is too
// small to pin all of a task's inputs).  The k-loop runs inside the kernel and the
// accumulator stays in TMEM across every k-step, so C is written exactly once.
//
// Operands are read by TMA out of tile-cache slots ("planes" of bf16).  In the
// FP32-accurate mode every fp32/f64 tile was split once at admission (K2,
// convert.cu) into hi = bf16(x) and lo = bf16(x - hi); each 64-wide k-block then
// issues three MMAs  hi*lo + lo*hi + hi*hi  into the same fp32 accumulator.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tr {

constexpr int kMaxKSteps = 64;  // k-steps per launch; longer tasks are chunked (accumulate=1)

enum Epilogue : int32_t {
  EPI_STORE = 0,        // C = acc
  EPI_ACCUMULATE = 1,   // C += acc
};

// Fused post-op applied to the final value v (after STORE/ACCUMULATE), float32
// outputs only (MLP training, ann.py:151-174):
enum PostOp : int32_t {
  POST_NONE = 0,
  POST_BIAS_ACT = 1,  // C = act(v + bias[col])                 forward layer (K3 fused)
  POST_ACT_GRAD = 2,  // C = v * act'(aux[row, col])            dX of layer l+1 -> dY of layer l (K4 fused)
};

struct GemmArgs {
  int32_t m_valid;               // output rows actually stored
  int32_t n_valid;               // output cols actually stored
  int32_t n_ksteps;              // number of k-steps in this launch
  int32_t planes;                // 1 = bf16, 2 = hi/lo split (fp32acc), 3 = hi/mid/lo (fp32hi)
  int32_t a_z[kMaxKSteps];       // TMA dim-2 index of A's hi plane per k-step (lo = +1)
  int32_t b_z[kMaxKSteps];       // same for B
  int32_t k_len[kMaxKSteps];     // contraction extent of each k-step
  void* c;                       // output (row-major, ldc elements)
  int64_t ldc;
  int32_t c_f64;                 // 0: float32 output, 1: float64 output
  int32_t epilogue;              // Epilogue
  int32_t seg_kb;                // k-blocks (of 64) per TMEM partial sum; see below
  int32_t post;                  // PostOp
  int32_t scaled;                // non-zero: the product is alpha * A.B (before STORE / ACCUMULATE)
  float alpha;
  int32_t act;                   // Activation of the post-op
  const float* bias;             // POST_BIAS_ACT: bias of this tile's first column
  const float* aux;              // POST_ACT_GRAD: activation output at this tile's origin
  int64_t ldaux;
  // Split-K (k_split > 1): CTA z of the grid's z dimension accumulates only the
  // k-blocks [z*kb/k_split, (z+1)*kb/k_split) and stores its raw fp32 partial
  // at ws + z*ws_zstride (row-major, ws_ld); launch_splitk_reduce then sums
  // the partials in z order (deterministic) and applies epilogue + post-op.
  int32_t k_split;
  float* ws;
  int64_t ws_ld;
  int64_t ws_zstride;
  // Write-through (non-null wt): the final values are also split into `planes`
  // bf16 planes at wt (row stride wt_ld, plane stride wt_plane) -- a tile-cache
  // slot, exactly as K2 would convert them.  Full tiles, coalesced path only.
  uint16_t* wt;
  int64_t wt_ld;
  int64_t wt_plane;
  // Fused column sums (non-null colsum): each epilogue warp also sums its 32
  // rows of final values per column and stores colsum[(row / 32) * colsum_ld +
  // col] (tile-relative row / col; the caller offsets the pointer to the tile).
  // Coalesced unsplit path only; the session runs tile_colsum32 otherwise.
  float* colsum;
  int64_t colsum_ld;
};

// Several tasks in ONE launch (a station's worth of ready tasks): CTAs
// [cta_begin[t], cta_begin[t+1]) of the flattened grid compute task t, M-blocks
// fastest (m_blocks[t] CTAs along M, a multiple of the CTA-pair size).  One
// launch instead of one per task removes the per-launch prologue/tail and the
// wave-quantisation loss of a 512-CTA task grid (3.46 waves of 148 SMs), and
// keeps CTA pairs from competing with a concurrent kernel for SM pairs.
constexpr int kMaxGroup = 8;
constexpr int kMaxDieClusters = 80;
struct GemmGroup {
  int32_t n_tasks;
  int32_t k_split;  // > 1: every task split into k_split k-shares (units z * tiles + tile; partials to task.ws)
  int32_t cta_begin[kMaxGroup + 1];
  int32_t m_blocks[kMaxGroup];
  // Die-aware unit order (persistent CTA-pair launches over a whole B200; see
  // die_map_prepare): cluster c is expected on die die_rank[c] >> 8 as that
  // die's (die_rank[c] & 0xFF)-th cluster.  A performance hint only -- the
  // cluster -> unit assignment stays a bijection whatever the real placement.
  int32_t die_mode;
  int32_t die_n[2];
  uint16_t die_rank[kMaxDieClusters];
  GemmArgs task[kMaxGroup];
};

// Measures, once per GPU, which SMs share a die (L2 latency signatures) and
// where a persistent CTA-pair launch places each cluster; afterwards grouped
// K1 launches on that GPU give each die a compact block of output units (a
// row half of the tasks' tiles) so the two dies' L2 halves stop caching the
// same panels.  Synchronous (runs small kernels on the current device); call
// before any stream work, e.g. at session creation.  TR_K1_DIE=0 disables.
void die_map_prepare(int gpu);
bool die_map_ready(int gpu, int* n0, int* n1);

// Accumulation-precision note (measured on B200, tools/probe_accum.py): the
// tcgen05 fp32 accumulator rounds toward zero, so a long K accumulated in TMEM
// drifts linearly in K (-1e-4 relative at K=32768).  The kernel therefore
// accumulates at most `seg_kb` k-blocks in TMEM, then the epilogue warps add
// the partial sum into fp32 registers with round-to-nearest (double-buffered
// TMEM, so the tensor pipe never waits).  FP32-accurate mode uses seg_kb = 4.
constexpr int kSegKbFp32Acc = 4;
// fp32hi (3 planes, 6 MMA passes per k-block): the same TMEM additions per
// partial sum as fp32acc, so half the k-blocks
constexpr int kSegKbFp32Hi = 2;
inline int seg_kb_for(int planes) { return planes == 3 ? kSegKbFp32Hi : planes == 2 ? kSegKbFp32Acc : 0; }

// Geometry of a 3-D bf16 tensor map: dim0 = columns (contiguous), dim1 = rows,
// dim2 = plane index.  Used for both tile-cache slabs and dense matrices.
struct PlaneGeom {
  void* base;
  int64_t cols, rows, nplanes;
  int64_t ld;            // elements between rows
  int64_t plane_stride;  // elements between planes
};

// Box shapes the kernel family needs; one tensor map per (geometry, box).
enum BoxKind : int32_t { BOX_K128 = 0, BOX_MN64 = 1, BOX_K256 = 2, BOX_K64 = 3 };

// Encodes a tensor map for `g` with the given box; returns 0 on success.
int make_plane_tmap(CUtensorMap* out, const PlaneGeom& g, BoxKind box);

// Launches the tile GEMM.  a_mn: A stored K x M (transposed operand, MN-major);
// b_kmajor: B stored N x K (transposed operand, K-major).
// tmA/tmB must have been made with the boxes reported by gemm_boxes(a_mn, b_kmajor, m_valid).
cudaError_t launch_tile_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, bool a_mn,
                             bool b_kmajor, cudaStream_t stream);
// All tasks of `g` must share the operand layouts (a_mn, b_kmajor), planes and
// pair choice (m_valid > 128 for every task, or for none); no split-K.
cudaError_t launch_tile_gemm_group(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, bool a_mn,
                                   bool b_kmajor, cudaStream_t stream);
// Same, with the persistence choice explicit (launches that run concurrently
// with others -- the k-panel schedule's -- do better non-persistent) and the
// SMs a persistent grid may fill (0: the whole GPU; a green-context device
// passes its own SM count).
cudaError_t launch_tile_gemm_group(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, bool a_mn,
                                   bool b_kmajor, bool persistent, cudaStream_t stream, int sm_budget = 0);
void gemm_boxes(bool a_mn, bool b_kmajor, int m_valid, BoxKind* box_a, BoxKind* box_b, bool grouped = false);
// A grouped launch given the slab's tensor maps of every box kind (maps[BoxKind]):
// picks the boxes, and TMA-multicast clusters of two CTA pairs (256 x 512 units,
// A loaded once per cluster) when gemm_multicast_enabled() and the group allows.
cudaError_t launch_tile_gemm_group_maps(const CUtensorMap* maps, GemmGroup& g, bool a_mn, bool b_kmajor,
                                        bool persistent, cudaStream_t stream, int sm_budget = 0);
// TMA multicast for grouped launches (default off; TR_GEMM_MC=1 enables).
bool gemm_multicast_enabled();
void set_gemm_multicast(bool on);
// Sums the k_split partials of a split-K launch in z order into C, then applies
// args.epilogue (STORE / ACCUMULATE) and args.post, exactly like the kernel's own
// epilogue would have (same argument block).
cudaError_t launch_splitk_reduce(const GemmArgs& args, cudaStream_t stream);
// Narrow outputs on the tensor cores: a task whose C tile is at most
// kSmallMaxN columns wide (and whose contraction is longer than kSmallMaxK) is
// computed as P = Bᵀ·Aᵀ -- the long side on the MMA's N, the narrow side on its
// 128 rows -- with the k-loop split over the grid; P's partials go to args.ws
// (rows = C's columns, ws_ld) and launch_splitk_reduce_t sums them in z order
// into C[r, c] with the task's epilogue / post-op.  Process-wide switch,
// default on (TR_NARROW_TC=0 or set_narrow_tc(false): such tasks run on the
// CUDA-core kernel instead).
cudaError_t launch_splitk_reduce_t(const GemmArgs& args, cudaStream_t stream);
bool narrow_tc_enabled();
void set_narrow_tc(bool on);
// Split-K policy switch (process-wide): max splits per launch, 1 disables.
// Default 8; TR_SPLITK=<n> in the environment overrides.
int splitk_max();
void set_splitk_max(int n);
// CTA-pair (cta_group::2, 256 x 256) variant for tiles taller than 128 rows.
// Off by default; TR_GEMM_PAIRS=1 or set_gemm_pairs(true) selects it.
bool gemm_pairs_enabled();
void set_gemm_pairs(bool on);
// Grouped launches (launch_tile_gemm_group) use CTA pairs by default
// (TR_GROUP_PAIRS=0 or set_group_pairs(false) selects single CTAs).
bool group_pairs_enabled();
void set_group_pairs(bool on);
// Whether a grouped launch of tiles with m_valid rows runs CTA pairs: enabled,
// taller than 128 rows, and no more row padding than single CTAs (784 rows:
// 7 x 128 singles, not 4 x 256 pairs).  Every task of a group must agree.
bool group_uses_pairs(int m_valid);
// Grouped launches are persistent by default (one CTA / pair per SM walking
// several output units, the store of one tile overlapping the next tile's
// k-loop); TR_PERSISTENT=0 or set_persistent(false) launches one CTA per unit.
bool persistent_enabled();
void set_persistent(bool on);

// K1s (small_gemm.cu): the task GEMM on CUDA cores for tiles a 128 x 256
// tensor-core tile would mostly pad -- outputs at most kSmallMaxN columns wide
// (the MLP's 10-wide output layer) or a total contraction of at most kSmallMaxK
// (its dX = dY W^T).  Same operands (tile-cache planes at slab + z * plane_stride,
// row stride ld; hi + lo re-assembled in fp32), same GemmArgs contract
// (epilogue, post-op, write-through, split-K partials into args.ws for
// launch_splitk_reduce), fp32 FMA in ascending k.
constexpr int kSmallMaxN = 32;
constexpr int kSmallMaxK = 32;
bool small_gemm_eligible(const GemmArgs& args);
// split-K factor for a narrow task on `sms` SMs (1: no split)
int small_gemm_split(const GemmArgs& args, int sms);
cudaError_t launch_small_gemm(const uint16_t* slab, int64_t ld, int64_t plane_stride, const GemmArgs& args,
                              bool a_mn, bool b_kmajor, cudaStream_t stream);
// Process-wide switch (default on; TR_SMALL_GEMM=0 or set_small_gemm(false)
// sends every task to the tensor-core kernel).
bool small_gemm_enabled();
void set_small_gemm(bool on);

// KX: precision "exact" (exact_gemm.cu) -- the reference's arithmetic bit for
// bit: per output element a rounded multiply then a rounded add (float32 when
// both operands and C are float32, else float64 with C's dtype rounding), k ascending, from 0 (EPI_STORE) or from C's current value
// (EPI_ACCUMULATE).  Tiles are float64, row-major with `ld` doubles per row; k-step
// ks of A starts at a_base + (a_z[ks] / 4) * slot_doubles (likewise B).  No
// post-op, scaling, split-K, write-through or column sums.
cudaError_t launch_exact_gemm(const void* a_base, const void* b_base, int64_t ld, int64_t slot_doubles,
                              const GemmArgs& args, bool a_mn, bool b_kmajor, bool f32_operands,
                              cudaStream_t stream);
// Tile admission for the exact mode: the rows x cols region as float64 (ld_dst per row).
cudaError_t launch_exact_convert(const void* src, int src_f64, int64_t ld_src, int64_t rows, int64_t cols, void* dst,
                                 int64_t ld_dst, cudaStream_t stream);

// K2: tile admission.  Converts a row-major fp32/f64 region (rows x cols, ld_src)
// into `planes` bf16 planes of a rows_cap x ld_dst slot, zero-filling everything
// outside the valid region so ragged tiles contribute nothing in K.
cudaError_t launch_split_convert(const void* src, int src_f64, int64_t ld_src, int64_t rows, int64_t cols,
                                 uint16_t* dst, int64_t ld_dst, int64_t rows_cap, int64_t plane_stride,
                                 int planes, cudaStream_t stream);

}  // namespace tr
