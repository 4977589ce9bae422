// K1 tile GEMM and K2 split/convert for sm_100a.  See tile_gemm.h for the contract.
//
// Kernel anatomy (one CTA per 128 x 256 output block, 384 threads = 3 warpgroups):
//   warp 0       TMA producer  (one elected lane; STAGES-deep smem ring, mbarrier full/empty)
//   warp 1       MMA issuer    (one lane issues tcgen05.mma; commits free smem stages)
//   warp 2       TMEM allocator (512 columns = two 128 x 256 fp32 partial-sum buffers)
//   warp 3       idle (completes warpgroup 0, which hands registers to the epilogue)
//   warps 4..11  epilogue      (every seg_kb k-blocks: tcgen05.ld TMEM -> fp32 registers,
//                               round-to-nearest add; at the end: registers -> global)
// setmaxnreg moves registers from warpgroup 0 (64 each) to the epilogue
// warpgroups (216 each): 128 accumulators per thread plus room to keep several
// rows of global reads (C, activations) in flight in the store phase.
// All k-steps of a task (each a separate tile-cache slot, i.e. a different TMA
// dim-2 coordinate) stream through the same ring; C is written exactly once.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include <atomic>
#include <cstdlib>
#include <mutex>

#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "act.cuh"
#include "sm100_ptx.cuh"
#include "tile_gemm.h"

namespace tr {

namespace {

constexpr int BM = 128;                   // output rows per CTA (TMEM lanes)
constexpr int BN = 256;                   // output cols per CTA / per CTA pair
constexpr int BK = 64;                    // bf16 elements = 128 B = one SW128 row
constexpr int A_BYTES = BM * BK * 2;      // 16 KiB per plane
constexpr int MN_GROUP_BYTES = 64 * BK * 2;  // one 64-wide MN-major TMA box (8 KiB)
constexpr int EPI_WARP0 = 4;                 // warps 4..11: epilogue (2 per TMEM lane quadrant)
constexpr int EPI_WARPS = 8;
constexpr int NUM_THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int TMEM_COLS = 2 * BN;             // double-buffered 128 x 256 fp32 partial sums
constexpr int SMEM_BUDGET = 227 * 1024;

// CG = 1: one CTA computes 128 x 256 with tcgen05 cta_group::1.
// CG = 2: a CTA pair (cluster of 2, one per SM of a TPC) computes 256 x 256 with
//         cta_group::2: each CTA stages its 128 rows of A and 128 of the 256
//         columns of B, the leader issues M=256 MMAs over both CTAs' smem, and
//         each CTA's TMEM holds its 128 x 256 accumulator.  Per SM this halves
//         the B bytes fetched and the smem bytes the tensor core reads.
// hi = bf16(v), lo = bf16(v - hi) for 4 consecutive values (the K2 split of a
// float32 input, bit for bit), stored as 8-byte vectors into 1 or 2 planes; 3
// planes (fp32hi): hi, mid = bf16(v - hi), lo = bf16(v - hi - mid) -- every
// difference is exact in float32, so the three planes carry all 24 bits.
__device__ __forceinline__ void split4(uint16_t* dst, int64_t plane, int planes, float4 v) {
  // packed conversions (one cvt.rn.bf16x2.f32 per pair): the epilogue's store
  // phase is instruction-bound when it also writes the planes
  const __nv_bfloat162 h01 = __floats2bfloat162_rn(v.x, v.y);
  const __nv_bfloat162 h23 = __floats2bfloat162_rn(v.z, v.w);
  uint2 hi;
  hi.x = *reinterpret_cast<const uint32_t*>(&h01);
  hi.y = *reinterpret_cast<const uint32_t*>(&h23);
  *reinterpret_cast<uint2*>(dst) = hi;
  if (planes >= 2) {
    const float2 f01 = __bfloat1622float2(h01);
    const float2 f23 = __bfloat1622float2(h23);
    // an infinite hi carries the value alone (lo = 0, not inf - inf = NaN)
    const float2 r01 = make_float2(isinf(f01.x) ? 0.f : v.x - f01.x, isinf(f01.y) ? 0.f : v.y - f01.y);
    const float2 r23 = make_float2(isinf(f23.x) ? 0.f : v.z - f23.x, isinf(f23.y) ? 0.f : v.w - f23.y);
    const __nv_bfloat162 l01 = __floats2bfloat162_rn(r01.x, r01.y);
    const __nv_bfloat162 l23 = __floats2bfloat162_rn(r23.x, r23.y);
    uint2 lo;
    lo.x = *reinterpret_cast<const uint32_t*>(&l01);
    lo.y = *reinterpret_cast<const uint32_t*>(&l23);
    *reinterpret_cast<uint2*>(dst + plane) = lo;
    if (planes == 3) {
      const float2 m01 = __bfloat1622float2(l01);
      const float2 m23 = __bfloat1622float2(l23);
      const __nv_bfloat162 t01 = __floats2bfloat162_rn(r01.x - m01.x, r01.y - m01.y);
      const __nv_bfloat162 t23 = __floats2bfloat162_rn(r23.x - m23.x, r23.y - m23.y);
      uint2 t;
      t.x = *reinterpret_cast<const uint32_t*>(&t01);
      t.y = *reinterpret_cast<const uint32_t*>(&t23);
      *reinterpret_cast<uint2*>(dst + 2 * plane) = t;
    }
  }
}

// The MMA passes of one k-block: plane pairs (a, b), smallest terms first and
// hi*hi last.  fp32acc (2 planes): the products of (hi+lo)(hi+lo) but lo*lo;
// fp32hi (3 planes): the six products of (hi+mid+lo)(hi+mid+lo) of weight >= 2^-16.
__host__ __device__ constexpr int n_passes(int planes) { return planes == 1 ? 1 : (planes == 2 ? 3 : 6); }
__host__ __device__ constexpr int pass_a(int planes, int pass) {
  return planes == 2 ? (pass == 1 ? 1 : 0) : planes == 3 ? (pass == 1 ? 2 : pass == 2 || pass == 4 ? 1 : 0) : 0;
}
__host__ __device__ constexpr int pass_b(int planes, int pass) {
  return planes == 2 ? (pass == 0 ? 1 : 0) : planes == 3 ? (pass == 0 ? 2 : pass == 2 || pass == 3 ? 1 : 0) : 0;
}
static_assert(pass_a(3, 0) == 0 && pass_b(3, 0) == 2 && pass_a(3, 1) == 2 && pass_b(3, 1) == 0 &&
                  pass_a(3, 2) == 1 && pass_b(3, 2) == 1 && pass_a(3, 3) == 0 && pass_b(3, 3) == 1 &&
                  pass_a(3, 4) == 1 && pass_b(3, 4) == 0 && pass_a(3, 5) == 0 && pass_b(3, 5) == 0,
              "fp32hi pass table");

template <int PLANES, int CG>
struct Cfg {
  static constexpr int BN_LOCAL = BN / CG;                // B columns staged per CTA
  static constexpr int B_BYTES = BN_LOCAL * BK * 2;       // per plane
  static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES);
  static constexpr int STAGE_ROWS = 8;                    // epilogue staging: rows per warp per round
  static constexpr int STAGE_LD = 132;                    // padded row (floats): conflict-free both ways
  static constexpr int EPI_STAGE_BYTES = EPI_WARPS * STAGE_ROWS * STAGE_LD * 4;
  static constexpr int STAGES = std::min(6, (SMEM_BUDGET - 2048 - EPI_STAGE_BYTES) / STAGE_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE_BYTES;
  static_assert(STAGES >= 1, "operand stage does not fit in shared memory");
};

// Output unit u of a group launch -> (task, row/column origin, split-K share).
// A unit is one 128 x 256 CTA tile (CG = 1) or one 256 x 256 pair tile (CG = 2)
// over the k-blocks of share z of nz.  Grouped launches fold split-K into the
// unit index (grp.k_split shares of every tile: u = z * tiles + tile), so a
// persistent grid balances them like any other units; single-task launches
// split along the grid's z dimension.
struct Unit {
  int t, m0, n0, z, nz;
};
// MC = 2 (TMA multicast, clusters of two CTA pairs): a unit is 256 x 512 --
// pair p of the cluster computes columns [n0 + 256 p, n0 + 256 p + 256) of the
// same 256 rows; rank = the CTA's rank in the cluster.
template <int CG, int MC = 1>
__device__ __forceinline__ Unit unit_of(const GemmGroup& grp, int u, uint32_t rank) {
  Unit r;
  const int tiles = grp.cta_begin[grp.n_tasks] / (CG * MC);
  if (grp.k_split > 1) {
    r.z = u / tiles;
    r.nz = grp.k_split;
    u -= r.z * tiles;
  } else {
    r.z = static_cast<int>(blockIdx.z);
    r.nz = static_cast<int>(gridDim.z);
  }
  const int cta = u * CG * MC;  // the unit's first CTA index in the flattened (non-persistent) grid
  int t = 0;
  while (t + 1 < grp.n_tasks && cta >= grp.cta_begin[t + 1]) ++t;
  const int local_unit = (cta - grp.cta_begin[t]) / (CG * MC);
  const int mb = grp.m_blocks[t] / CG;  // row blocks of BM * CG rows, fastest
  const int in_pair = static_cast<int>(rank) % CG, pair = static_cast<int>(rank) / CG;
  r.t = t;
  r.m0 = (local_unit % mb) * (BM * CG) + in_pair * BM;
  r.n0 = ((local_unit / mb) * MC + pair) * BN;
  return r;
}

// The it-th output unit of cluster `cl` (of n_cl), or -1 when it has no more.
// Default: units cl, cl + n_cl, ... (row blocks fastest inside a task).  Die
// mode (grp.die_mode): the units are listed task by task, the upper half of
// the row blocks column by column, then the lower half; die 0's clusters take
// the first n0 / (n0 + n1) of the list and die 1's the rest, each die striding
// through its share by its clusters' ranks -- so at any time a die works on
// ~half the row blocks of a few columns (its own A and B panels) instead of
// both dies reading every panel of the wave.
template <int CG, int MC>
__device__ __forceinline__ int unit_for(const GemmGroup& grp, int cl, int n_cl, int it, int n_units) {
  if (MC != 1 || CG != 2 || !grp.die_mode) {
    const int u = cl + it * n_cl;
    return u < n_units ? u : -1;
  }
  const int dr = grp.die_rank[cl];
  const int d = dr >> 8, r = dr & 0xFF;
  const int q0 = static_cast<int>(static_cast<int64_t>(n_units) * grp.die_n[0] / (grp.die_n[0] + grp.die_n[1]));
  const int q = (d ? q0 : 0) + r + it * grp.die_n[d];
  if (q >= (d ? n_units : q0)) return -1;
  int t = 0, base = 0;
  while (t + 1 < grp.n_tasks) {
    const int nt = (grp.cta_begin[t + 1] - grp.cta_begin[t]) / CG;
    if (q < base + nt) break;
    base += nt;
    ++t;
  }
  const int mb = grp.m_blocks[t] / CG;                                    // row blocks (256 rows)
  const int nb = (grp.cta_begin[t + 1] - grp.cta_begin[t]) / grp.m_blocks[t];  // column blocks
  const int ql = q - base;
  const int h0 = (mb + 1) / 2;
  int row, col;
  if (ql < h0 * nb) {
    col = ql / h0;
    row = ql % h0;
  } else {
    const int q2 = ql - h0 * nb, h1 = mb - h0;
    col = q2 / h1;
    row = h0 + q2 % h1;
  }
  return grp.cta_begin[t] / CG + col * mb + row;  // that tile's index in the default order (unit_of)
}

// k-blocks of a task and share z of nz of them
struct KRange {
  int total, lo, hi;
};
__device__ __forceinline__ KRange krange(const GemmArgs& args, int z, int nz) {
  int total_kb = 0;
  for (int ks = 0; ks < args.n_ksteps; ++ks) total_kb += (args.k_len[ks] + BK - 1) / BK;
  KRange r;
  r.total = total_kb;
  r.lo = static_cast<int>((static_cast<int64_t>(z) * total_kb) / nz);
  r.hi = static_cast<int>((static_cast<int64_t>(z + 1) * total_kb) / nz);
  return r;
}

// The CTA (pair) walks output units u = cluster, cluster + n_clusters, ... of the
// group -- one unit per CTA when the grid covers every unit, several when the
// launch is persistent (grouped launches: one CTA per SM).  The producer and
// the MMA issuer run straight across units; the epilogue warps drain unit i's
// TMEM partial sums while the tensor core already computes unit i+1 into the
// other TMEM buffer, so the store of one tile overlaps the next tile's k-loop.
template <bool A_MN, bool B_K, int PLANES, int CG, int MC = 1>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tile_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmGroup grp) {
  static_assert(MC == 1 || CG == 2, "multicast clusters are made of CTA pairs");
  using C = Cfg<PLANES, CG>;
  constexpr int STAGES = C::STAGES;
  constexpr int STAGE_BYTES = C::STAGE_BYTES;
  constexpr int B_BYTES = C::B_BYTES;
  constexpr int BN_LOCAL = C::BN_LOCAL;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2] MMA -> epilogue: partial sum ready in TMEM buffer b
  uint64_t* acc_empty = acc_full + 2;   // [2] epilogue -> MMA: TMEM buffer b drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // rank in the cluster; the CTA pair = ranks {2p, 2p + 1}, its leader 2p
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0u;
  const uint32_t lead_rank = rank & ~1u;
  const bool leader = rank == lead_rank;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << lead_rank);
  const int n_units = (grp.cta_begin[grp.n_tasks] / (CG * MC)) * (grp.k_split > 1 ? grp.k_split : 1);
  const int first_unit = static_cast<int>(blockIdx.x) / (CG * MC);
  const int unit_stride = static_cast<int>(gridDim.x) / (CG * MC);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], MC);  // MC = 2: a stage is free once BOTH pairs' MMAs read it
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], EPI_WARPS * CG);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 2) {
    if (CG == 2) ptx::tmem_alloc_cg2(tmem_slot, TMEM_COLS);
    else ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // barrier inits + TMEM address visible pair-wide
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < EPI_WARP0) {
  ptx::setmaxnreg_dec<64>();
  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs of a pair load their halves)
      const uint32_t full0 = ptx::smem_u32(&full[0]);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0, u; (u = unit_for<CG, MC>(grp, first_unit, unit_stride, it, n_units)) >= 0; ++it) {
        const Unit un = unit_of<CG, MC>(grp, u, rank);
        const GemmArgs& args = grp.task[un.t];
        const int nb0 = un.n0 + static_cast<int>(rank - lead_rank) * BN_LOCAL;  // B columns this CTA stages
        const KRange kr = krange(args, un.z, un.nz);
        int g = 0;  // global k-block index
        for (int ks = 0; ks < args.n_ksteps; ++ks) {
          const int nkb = (args.k_len[ks] + BK - 1) / BK;
          const int az = args.a_z[ks];
          const int bz = args.b_z[ks];
          for (int kb = 0; kb < nkb; ++kb, ++g) {
            if (g < kr.lo || g >= kr.hi) continue;
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            uint8_t* sb = sa + PLANES * A_BYTES;
            const int k0 = kb * BK;
            // completion bytes of both CTAs go to the pair leader's full barrier
            const uint32_t bar = (CG == 2) ? ptx::mapa_shared(full0 + stage * 8, lead_rank) : 0u;
            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], CG * STAGE_BYTES);
            auto load = [&](void* dst, const CUtensorMap* tm, int c0, int c1, int c2) {
              if (CG == 2) ptx::tma_load_3d_cg2(dst, tm, bar, c0, c1, c2);
              else ptx::tma_load_3d(dst, tm, &full[stage], c0, c1, c2);
            };
#pragma unroll
            for (int p = 0; p < PLANES; ++p) {
              if (MC == 2) {
                // the two pairs need the same A rows: each CTA loads half of its
                // 128-row A tile (64 rows) and multicasts it to itself and to the
                // same-position CTA of the other pair (64-row boxes either layout)
                const int h = static_cast<int>(rank >> 1);  // which half this CTA loads
                const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 2u)));
                if (!A_MN)
                  ptx::tma_load_3d_cg2_mc(sa + p * A_BYTES + h * (A_BYTES / 2), &tmA, bar, mask, k0, un.m0 + 64 * h,
                                          az + p);
                else
                  ptx::tma_load_3d_cg2_mc(sa + p * A_BYTES + h * MN_GROUP_BYTES, &tmA, bar, mask, un.m0 + 64 * h, k0,
                                          az + p);
              } else if (!A_MN) {
                load(sa + p * A_BYTES, &tmA, k0, un.m0, az + p);
              } else {
#pragma unroll
                for (int gg = 0; gg < BM / 64; ++gg)
                  load(sa + p * A_BYTES + gg * MN_GROUP_BYTES, &tmA, un.m0 + 64 * gg, k0, az + p);
              }
              if (B_K) {
                load(sb + p * B_BYTES, &tmB, k0, nb0, bz + p);
              } else {
#pragma unroll
                for (int gg = 0; gg < BN_LOCAL / 64; ++gg)
                  load(sb + p * B_BYTES + gg * MN_GROUP_BYTES, &tmB, nb0 + 64 * gg, k0, bz + p);
              }
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (the pair's leader issues for both CTAs).  The
      // whole warp walks the k-loop -- converged, so barrier phases, stage
      // addresses and descriptors are warp-uniform (uniform registers) -- and one
      // elected lane issues each k-block's MMAs and their commits.
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM * CG, BN, A_MN, !B_K);
      int stage = 0;
      uint32_t phase = 0;
      int seg = 0;  // TMEM partial sums issued so far (all units)
      for (int it = 0, u; (u = unit_for<CG, MC>(grp, first_unit, unit_stride, it, n_units)) >= 0; ++it) {
        const Unit un = unit_of<CG, MC>(grp, u, rank);
        const GemmArgs& args = grp.task[un.t];
        const KRange kr = krange(args, un.z, un.nz);
        const int seg_kb = args.seg_kb > 0 ? args.seg_kb : max(kr.hi - kr.lo, 1);
        int kb_in_seg = 0;
        uint32_t tmem_d = tmem_base;
        uint32_t accumulate = 0;
        int g = 0;
        for (int ks = 0; ks < args.n_ksteps; ++ks) {
          const int nkb = (args.k_len[ks] + BK - 1) / BK;
          for (int kb = 0; kb < nkb; ++kb, ++g) {
            if (g < kr.lo || g >= kr.hi) continue;
            if (kb_in_seg == 0) {
              // new partial sum: wait until the epilogue(s) drained this TMEM buffer
              const int buf = seg & 1;
              ptx::mbar_wait(&acc_empty[buf], ((seg >> 1) & 1) ^ 1);
              ptx::tc_fence_after();
              tmem_d = tmem_base + static_cast<uint32_t>(buf * BN);
              accumulate = 0;
            }
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a_base = ptx::smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t b_base = a_base + PLANES * A_BYTES;
            const bool seg_done = kb_in_seg + 1 == seg_kb;
            if (ptx::elect_one()) {
              uint32_t acc = accumulate;
              // small cross terms first, then hi*hi (n_passes / pass_a / pass_b)
#pragma unroll
              for (int pass = 0; pass < n_passes(PLANES); ++pass) {
                const int pa = pass_a(PLANES, pass);
                const int pb = pass_b(PLANES, pass);
                // k16 advances the start address field (bits [0,14), 16-byte units)
                const uint64_t a0 = A_MN ? ptx::sdesc_sw128(a_base + pa * A_BYTES, MN_GROUP_BYTES, 1024)
                                         : ptx::sdesc_sw128(a_base + pa * A_BYTES, 16, 1024);
                const uint64_t b0 = B_K ? ptx::sdesc_sw128(b_base + pb * B_BYTES, 16, 1024)
                                        : ptx::sdesc_sw128(b_base + pb * B_BYTES, MN_GROUP_BYTES, 1024);
#pragma unroll
                for (int k16 = 0; k16 < BK / 16; ++k16) {
                  const uint64_t adesc = a0 + static_cast<uint64_t>((A_MN ? 2048 : 32) * k16 >> 4);
                  const uint64_t bdesc = b0 + static_cast<uint64_t>((B_K ? 32 : 2048) * k16 >> 4);
                  if (CG == 2) ptx::mma_bf16_cg2(tmem_d, adesc, bdesc, idesc, acc);
                  else ptx::mma_bf16(tmem_d, adesc, bdesc, idesc, acc);
                  acc = 1;
                }
              }
              // the stage's smem is released in every CTA that received its data
              if (CG == 2) ptx::mma_commit_cg2_mc(&empty[stage], MC == 2 ? 0xF : pair_mask);
              else ptx::mma_commit(&empty[stage]);
              if (seg_done) {
                if (CG == 2) ptx::mma_commit_cg2_mc(&acc_full[seg & 1], pair_mask);
                else ptx::mma_commit(&acc_full[seg & 1]);
              }
            }
            __syncwarp();
            accumulate = 1;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            if (++kb_in_seg == seg_kb) {
              kb_in_seg = 0;
              ++seg;
            }
          }
        }
        if (kb_in_seg != 0) {  // the unit's last, partial segment
          if (ptx::elect_one()) {
            if (CG == 2) ptx::mma_commit_cg2_mc(&acc_full[seg & 1], pair_mask);
            else ptx::mma_commit(&acc_full[seg & 1]);
          }
          __syncwarp();
          ++seg;
        }
      }
    }
  }
  } else {
    ptx::setmaxnreg_inc<216>();
    // ---------------- epilogue: TMEM partial sums -> fp32 registers (RNE) -> global
    const int q = warp & 3;                      // TMEM lane quadrant this warp may access
    const int half = (warp - EPI_WARP0) >> 2;    // column half of the 256-wide tile
    const int row = q * 32 + lane;
    const uint32_t tlane = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(half * 128);
    const uint32_t empty_leader = (CG == 2) ? ptx::mapa_shared(ptx::smem_u32(&acc_empty[0]), lead_rank) : 0u;
    float* stage = epi_stage + (warp - EPI_WARP0) * (C::STAGE_ROWS * C::STAGE_LD);
    int seg = 0;
    for (int it = 0, u; (u = unit_for<CG, MC>(grp, first_unit, unit_stride, it, n_units)) >= 0; ++it) {
      const Unit un = unit_of<CG, MC>(grp, u, rank);
      const GemmArgs& args = grp.task[un.t];
      const KRange kr = krange(args, un.z, un.nz);
      const int my_kb = kr.hi - kr.lo;
      const int seg_kb = args.seg_kb > 0 ? args.seg_kb : max(my_kb, 1);
      const int n_seg = (my_kb + seg_kb - 1) / seg_kb;
      float acc[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) acc[j] = 0.f;
      for (int s = 0; s < n_seg; ++s, ++seg) {
        const int buf = seg & 1;
        ptx::mbar_wait(&acc_full[buf], (seg >> 1) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < 8; c0 += 4) {  // four loads in flight per wait
          uint32_t r[4][16];
#pragma unroll
          for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x16(tlane + static_cast<uint32_t>(buf * BN + (c0 + c) * 16), r[c]);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[(c0 + c) * 16 + j] += __uint_as_float(r[c][j]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) ptx::mbar_arrive_cluster(empty_leader + buf * 8);
          else ptx::mbar_arrive(&acc_empty[buf]);
        }
      }
      const int grow = un.m0 + row;
      const int gcol0 = un.n0 + half * 128;
      const bool part = un.nz > 1;  // split-K: raw fp32 partials into the workspace
      float* obase = part ? args.ws + un.z * args.ws_zstride : static_cast<float*>(args.c);
      const int64_t ldo = part ? args.ws_ld : args.ldc;
      if ((part || !args.c_f64) && gcol0 + 128 <= args.n_valid && (ldo & 3) == 0 &&
          (reinterpret_cast<uintptr_t>(obase) & 15) == 0) {
        // Coalesced store: the warp's 32 x 128 block goes out through its own
        // small staging area (8 rows per round; rows padded to 132 floats keep
        // the row-per-thread writes and row-per-warp reads conflict-free), so
        // every global access is 512 contiguous bytes.
        const bool acc_mode = !part && args.epilogue == EPI_ACCUMULATE;
        const int post = part ? static_cast<int>(POST_NONE) : args.post;
        const int c = 4 * lane;
        float bias4[4] = {0.f, 0.f, 0.f, 0.f};
        if (post == POST_BIAS_ACT && args.bias)
          for (int x = 0; x < 4; ++x) bias4[x] = args.bias[gcol0 + c + x];
        const int row0 = un.m0 + q * 32;
        // fused column sums of the final values over this warp's 32 rows (in row order)
        const bool do_cs = !part && args.colsum != nullptr;
        float4 csum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int rb = 0; rb < 32; rb += C::STAGE_ROWS) {
          if (lane >= rb && lane < rb + C::STAGE_ROWS) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              *reinterpret_cast<float4*>(stage + (lane - rb) * C::STAGE_LD + 4 * j) =
                  make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
          }
          __syncwarp();
          // Rows go out in batches of PRE: the batch's global reads (C when
          // accumulating, the activation for act_grad) are all issued before the
          // first use, so a warp waits one memory latency per batch, not per row.
          constexpr int PRE = 8;
#pragma unroll 1
          for (int r0 = 0; r0 < C::STAGE_ROWS; r0 += PRE) {
            // pre[]: the activation rows for act_grad, else the C rows when accumulating
            // (both at once -- an accumulating act_grad product -- reads C inline)
            const bool pre_aux = post == POST_ACT_GRAD;
            const bool aux_vec = (args.ldaux & 3) == 0 && (reinterpret_cast<uintptr_t>(args.aux) & 15) == 0;
            float4 pre[PRE];
#pragma unroll
            for (int i = 0; i < PRE; ++i) {
              const int64_t grow_i = row0 + rb + r0 + i;
              pre[i] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (grow_i < args.m_valid) {
                if (pre_aux) {
                  const float* ax = args.aux + grow_i * args.ldaux + gcol0 + c;
                  pre[i] = aux_vec ? __ldg(reinterpret_cast<const float4*>(ax))
                                   : make_float4(__ldg(ax), __ldg(ax + 1), __ldg(ax + 2), __ldg(ax + 3));
                }
                else if (acc_mode) pre[i] = *reinterpret_cast<const float4*>(obase + grow_i * ldo + gcol0 + c);
              }
            }
#pragma unroll
            for (int i = 0; i < PRE; ++i) {
              const int64_t grow_i = row0 + rb + r0 + i;
              if (grow_i >= args.m_valid) break;
              float4* d4 = reinterpret_cast<float4*>(obase + grow_i * ldo + gcol0 + c);
              float4 v = *reinterpret_cast<const float4*>(stage + (r0 + i) * C::STAGE_LD + c);
              if (args.scaled && !part) v = make_float4(args.alpha * v.x, args.alpha * v.y, args.alpha * v.z, args.alpha * v.w);
              if (acc_mode) {
                const float4 o = pre_aux ? *d4 : pre[i];
                v.x += o.x;
                v.y += o.y;
                v.z += o.z;
                v.w += o.w;
              }
              if (post == POST_BIAS_ACT) {
                v.x = act_fwd(args.act, v.x + bias4[0]);
                v.y = act_fwd(args.act, v.y + bias4[1]);
                v.z = act_fwd(args.act, v.z + bias4[2]);
                v.w = act_fwd(args.act, v.w + bias4[3]);
              } else if (post == POST_ACT_GRAD) {
                v.x *= act_grad_from_out(args.act, pre[i].x);
                v.y *= act_grad_from_out(args.act, pre[i].y);
                v.z *= act_grad_from_out(args.act, pre[i].z);
                v.w *= act_grad_from_out(args.act, pre[i].w);
              }
              *d4 = v;
              if (do_cs) {
                csum.x += v.x;
                csum.y += v.y;
                csum.z += v.z;
                csum.w += v.w;
              }
              if (args.wt)  // write-through: the converted planes of this row segment (as K2)
                split4(args.wt + grow_i * args.wt_ld + gcol0 + c, args.wt_plane, PLANES, v);
            }
          }
          __syncwarp();
        }
        if (do_cs && row0 < args.m_valid) {
          float* cs = args.colsum + static_cast<int64_t>(row0 / 32) * args.colsum_ld + gcol0 + c;
          cs[0] = csum.x;
          cs[1] = csum.y;
          cs[2] = csum.z;
          cs[3] = csum.w;
        }
      } else if (grow < args.m_valid && gcol0 < args.n_valid) {
        const int ncols = min(128, args.n_valid - gcol0);
        const int64_t off = static_cast<int64_t>(grow) * args.ldc + gcol0;
        const bool acc_mode = !part && args.epilogue == EPI_ACCUMULATE;
        if (args.scaled && !part)
#pragma unroll
          for (int j = 0; j < 128; ++j) acc[j] *= args.alpha;
        if (args.c_f64 && !part) {
          double* dst = static_cast<double*>(args.c) + off;
#pragma unroll
          for (int j = 0; j < 128; ++j)
            if (j < ncols) dst[j] = acc_mode ? dst[j] + static_cast<double>(acc[j]) : static_cast<double>(acc[j]);
        } else {
          float* dst = part ? obase + static_cast<int64_t>(grow) * ldo + gcol0 : static_cast<float*>(args.c) + off;
          const int post = part ? static_cast<int>(POST_NONE) : args.post;
          const float* bias = args.bias ? args.bias + gcol0 : nullptr;
          const float* aux = args.aux ? args.aux + static_cast<int64_t>(grow) * args.ldaux + gcol0 : nullptr;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            if (j >= ncols) continue;
            float v = acc_mode ? dst[j] + acc[j] : acc[j];
            if (post == POST_BIAS_ACT) v = act_fwd(args.act, v + (bias ? bias[j] : 0.f));
            else if (post == POST_ACT_GRAD) v = v * act_grad_from_out(args.act, aux[j]);
            dst[j] = v;
          }
        }
      }
    }
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // the peer's TMEM/barriers stay alive until the leader is done
  else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if (CG == 2) ptx::tmem_dealloc_cg2(tmem_base, TMEM_COLS);
    else ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- die map
// Which die each SM sits on (B200: two dies, each with half the L2; addresses
// are homed on one die at fine grain and an L2 hit costs more from the far
// die): every SM times dependent L2-only loads of kDieLines lines 2 KB apart;
// its near/far pattern over the lines is its die's signature.
constexpr int kDieLines = 256, kDieReps = 32, kDieStride = 2048 / 8;

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void die_probe_kernel(const uint64_t* buf, float* lat, int nsm_cap) {
  if (threadIdx.x != 0) return;
  const uint32_t sm = sm_id();
  if (static_cast<int>(sm) >= nsm_cap) return;
  for (int j = 0; j < kDieLines; ++j) {
    uint64_t a = reinterpret_cast<uint64_t>(buf + j * kDieStride);
    asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));  // into L2 (the line holds its own address)
    a = reinterpret_cast<uint64_t>(buf + j * kDieStride);
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < kDieReps; ++r) asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));
    const long long t1 = clock64();
    lat[sm * kDieLines + j] = a == 0 ? -1.f : static_cast<float>(t1 - t0) / kDieReps;
  }
}

__global__ void die_where_kernel(int* sm_of_block) {
  if (threadIdx.x == 0) sm_of_block[blockIdx.x] = static_cast<int>(sm_id());
}

struct DieMap {
  int n_clusters = 0;
  int n[2] = {0, 0};
  uint16_t rank[kMaxDieClusters] = {};
};
std::mutex g_die_mu;
DieMap* g_die[64] = {};     // per device: null = not measured / not usable
bool g_die_tried[64] = {};

const DieMap* die_lookup(int gpu) {
  if (gpu < 0 || gpu >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_die_mu);
  return g_die[gpu];
}

DieMap* die_measure() {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) !=
                                                 cudaSuccess)
    return nullptr;
  if (nsm < 8 || nsm / 2 > kMaxDieClusters || nsm > 256) return nullptr;
  const size_t words = static_cast<size_t>(kDieLines) * kDieStride;
  std::vector<uint64_t> h(words, 0);
  uint64_t* buf = nullptr;
  float* lat = nullptr;
  int* where = nullptr;
  if (cudaMalloc(&buf, words * 8) != cudaSuccess) return nullptr;
  bool ok = cudaMalloc(&lat, sizeof(float) * 256 * kDieLines) == cudaSuccess &&
            cudaMalloc(&where, sizeof(int) * 512) == cudaSuccess;
  std::vector<float> L(static_cast<size_t>(256) * kDieLines, 0.f);
  std::vector<int> so(nsm, -1);
  const int smem = 200 * 1024;  // one CTA per SM
  if (ok) {
    for (int j = 0; j < kDieLines; ++j) h[static_cast<size_t>(j) * kDieStride] = reinterpret_cast<uint64_t>(buf + j * kDieStride);
    ok = cudaMemcpy(buf, h.data(), words * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemset(lat, 0, sizeof(float) * 256 * kDieLines) == cudaSuccess &&
         cudaFuncSetAttribute(die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
         cudaFuncSetAttribute(die_where_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  }
  if (ok) {
    die_probe_kernel<<<nsm, 32, smem>>>(buf, lat, 256);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nsm / 2 * 2));
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    ok = cudaLaunchKernelEx(&cfg, die_where_kernel, where) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
         cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(so.data(), where, sizeof(int) * nsm / 2 * 2, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaGetLastError();
  if (buf) cudaFree(buf);
  if (lat) cudaFree(lat);
  if (where) cudaFree(where);
  if (!ok) return nullptr;
  // two-means over the SMs' latency vectors: start from agreement with SM 0's
  // near/far pattern (per-line midpoint threshold), then re-assign each SM by
  // its projection on the per-line contrast between the two groups' means
  // (noisy lines carry little weight); every SM must sit clearly on one side
  const auto at = [&](int s, int j) { return L[static_cast<size_t>(s) * kDieLines + j]; };
  std::vector<int> die(nsm, 0);
  std::vector<double> mu0(kDieLines), mu1(kDieLines);
  for (int j = 0; j < kDieLines; ++j) {
    float lo = 1e30f, hi = 0.f;
    for (int s = 0; s < nsm; ++s) {
      if (at(s, j) <= 0.f) return nullptr;
      lo = std::min(lo, at(s, j));
      hi = std::max(hi, at(s, j));
    }
    mu0[j] = 0.5 * (lo + hi);  // threshold, reused below
  }
  for (int s = 0; s < nsm; ++s) {
    int agree = 0;
    for (int j = 0; j < kDieLines; ++j) agree += (at(s, j) > mu0[j]) == (at(0, j) > mu0[j]);
    die[s] = agree * 2 > kDieLines ? 0 : 1;
  }
  double min_margin = 0.0, gap = 0.0;
  for (int iter = 0; iter < 4; ++iter) {
    int c0 = 0, c1 = 0;
    std::fill(mu0.begin(), mu0.end(), 0.0);
    std::fill(mu1.begin(), mu1.end(), 0.0);
    for (int s = 0; s < nsm; ++s) {
      (die[s] ? c1 : c0) += 1;
      for (int j = 0; j < kDieLines; ++j) (die[s] ? mu1 : mu0)[j] += at(s, j);
    }
    if (c0 == 0 || c1 == 0) return nullptr;
    double wsum = 0.0;
    for (int j = 0; j < kDieLines; ++j) {
      mu0[j] /= c0;
      mu1[j] /= c1;
      wsum += std::fabs(mu1[j] - mu0[j]);
    }
    gap = wsum / kDieLines;  // mean |latency difference| between the groups per line
    min_margin = 1e30;
    for (int s = 0; s < nsm; ++s) {
      double score = 0.0;
      for (int j = 0; j < kDieLines; ++j) score += (at(s, j) - 0.5 * (mu0[j] + mu1[j])) * (mu1[j] - mu0[j]);
      // +-1 when the SM's vector equals its group's mean
      double half = 0.0;
      for (int j = 0; j < kDieLines; ++j) half += 0.5 * (mu1[j] - mu0[j]) * (mu1[j] - mu0[j]);
      const double z = half > 0 ? score / half : 0.0;
      die[s] = z > 0 ? 1 : 0;
      min_margin = std::min(min_margin, std::fabs(z));
    }
  }
  if (getenv("TR_K1_DIE_DEBUG")) fprintf(stderr, "die map: mean gap %.1f cycles, min margin %.2f\n", gap, min_margin);
  if (gap < 8.0 || min_margin < 0.3) return nullptr;  // no clean two-way split
  auto* m = new DieMap;
  m->n_clusters = nsm / 2;
  for (int c = 0; c < m->n_clusters; ++c) {
    const int s0 = so[2 * c], s1 = so[2 * c + 1];
    if (s0 < 0 || s0 >= nsm || s1 < 0 || s1 >= nsm || die[s0] != die[s1]) {
      if (getenv("TR_K1_DIE_DEBUG")) fprintf(stderr, "die map: cluster %d on sms %d / %d\n", c, s0, s1);
      delete m;
      return nullptr;
    }
    const int d = die[s0];
    m->rank[c] = static_cast<uint16_t>((d << 8) | m->n[d]);
    m->n[d] += 1;
  }
  if (m->n[0] < m->n_clusters / 4 || m->n[1] < m->n_clusters / 4) {
    delete m;
    return nullptr;
  }
  return m;
}

template <bool A_MN, bool B_K, int PLANES, int CG, int MC = 1>
cudaError_t launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, int k_split,
                           bool persistent, int sm_budget, cudaStream_t stream) {
  using C = Cfg<PLANES, CG>;
  auto kern = tile_gemm_kernel<A_MN, B_K, PLANES, CG, MC>;
  constexpr int CL = CG * MC;  // CTAs per cluster
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int max_clusters = 0;  // co-resident clusters of CL CTAs (MC = 2: GPC granularity)
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr_err == cudaSuccess && MC > 1) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(CL * 64);
      q.blockDim = dim3(NUM_THREADS);
      q.dynamicSmemBytes = C::SMEM;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = CL;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      attr_err = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &q);
    }
  });
  if (attr_err != cudaSuccess) return attr_err;
  // flattened grid: task t owns CTAs [cta_begin[t], cta_begin[t+1]), M-blocks fastest
  g.cta_begin[0] = 0;
  for (int t = 0; t < g.n_tasks; ++t) {
    const GemmArgs& a = g.task[t];
    g.m_blocks[t] = ((a.m_valid + BM * CG - 1) / (BM * CG)) * CG;
    g.cta_begin[t + 1] = g.cta_begin[t] + g.m_blocks[t] * ((a.n_valid + BN - 1) / BN);
  }
  // persistent: one CTA (pair) per SM walks several output units; otherwise one unit per CTA
  int ctas = g.cta_begin[g.n_tasks] * (g.k_split > 1 ? g.k_split : 1);
  if (persistent) {
    int dev = 0, sms = sm_budget;
    if (sms <= 0 && cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ctas = std::min(ctas, MC > 1 ? std::max(CL, max_clusters * CL) : std::max(CG, (sms / CG) * CG));
  }
  dim3 grid(static_cast<unsigned>(ctas), 1, (k_split > 1 && g.k_split <= 1) ? k_split : 1);
  // die-aware unit order: a persistent pair grid over the whole GPU, >= 2 waves of units
  g.die_mode = 0;
  if (CG == 2 && MC == 1 && persistent && g.k_split <= 1 && grid.z == 1) {
    int dev = 0;
    const DieMap* dm = cudaGetDevice(&dev) == cudaSuccess ? die_lookup(dev) : nullptr;
    if (dm && ctas == 2 * dm->n_clusters && g.cta_begin[g.n_tasks] / 2 >= 2 * dm->n_clusters) {
      g.die_mode = 1;
      g.die_n[0] = dm->n[0];
      g.die_n[1] = dm->n[1];
      std::memcpy(g.die_rank, dm->rank, sizeof(g.die_rank));
    }
  }
  if (CG == 1) {
    kern<<<grid, NUM_THREADS, C::SMEM, stream>>>(tmA, tmB, g);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, g);
}

// ---------------------------------------------------------------- K2 split/convert
template <typename T>
__global__ void split_convert_kernel(const T* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                                     uint16_t* __restrict__ dst, int64_t ld_dst, int64_t rows_cap, int64_t cols_cap,
                                     int64_t plane_stride, int planes) {
  const int64_t chunks_per_row = cols_cap / 8;
  const int64_t total = rows_cap * chunks_per_row;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / chunks_per_row;
    const int64_t c = (idx - r * chunks_per_row) * 8;
    uint16_t hi[8], lo[8], lo2[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t cc = c + j;
      const double v = (r < rows && cc < cols) ? static_cast<double>(src[r * ld_src + cc]) : 0.0;
      const __nv_bfloat16 h = __float2bfloat16_rn(static_cast<float>(v));
      const float hf = __bfloat162float(h);
      const double rest = isinf(hf) ? 0.0 : v - static_cast<double>(hf);  // inf carried by hi alone
      const __nv_bfloat16 l = __float2bfloat16_rn(static_cast<float>(rest));
      const __nv_bfloat16 l2 = __float2bfloat16_rn(static_cast<float>(rest - static_cast<double>(__bfloat162float(l))));
      hi[j] = __bfloat16_as_ushort(h);
      lo[j] = __bfloat16_as_ushort(l);
      lo2[j] = __bfloat16_as_ushort(l2);
    }
    uint16_t* d = dst + r * ld_dst + c;
    *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(hi);
    if (planes >= 2) *reinterpret_cast<uint4*>(d + plane_stride) = *reinterpret_cast<const uint4*>(lo);
    if (planes == 3) *reinterpret_cast<uint4*>(d + 2 * plane_stride) = *reinterpret_cast<const uint4*>(lo2);
  }
}

// Split-K reduction: C (+)= sum_z ws[z] in z order, then the fused post-op.
__global__ void splitk_reduce_kernel(const __grid_constant__ GemmArgs args) {
  const int64_t n = args.n_valid;
  const int64_t total = static_cast<int64_t>(args.m_valid) * n;
  const bool acc_mode = args.epilogue == EPI_ACCUMULATE;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / n, c = idx - r * n;
    const float* w = args.ws + r * args.ws_ld + c;
    float v = w[0];
    for (int z = 1; z < args.k_split; ++z) v += w[z * args.ws_zstride];
    if (args.scaled) v *= args.alpha;
    const int64_t off = r * args.ldc + c;
    if (args.c_f64) {
      double* dst = static_cast<double*>(args.c) + off;
      *dst = acc_mode ? *dst + static_cast<double>(v) : static_cast<double>(v);
      continue;
    }
    float* dst = static_cast<float*>(args.c) + off;
    if (acc_mode) v += *dst;
    if (args.post == POST_BIAS_ACT) v = act_fwd(args.act, v + (args.bias ? args.bias[c] : 0.f));
    else if (args.post == POST_ACT_GRAD) v = v * act_grad_from_out(args.act, args.aux[r * args.ldaux + c]);
    *dst = v;
  }
}

// The transposed-product reduction: the partials of P = Bᵀ·Aᵀ (narrow C
// computed with its long side on the MMA's N) sit at ws + z*ws_zstride as
// rows = C's columns; C[r, c] (+)= alpha * sum_z P_z[c, r] in z order, then the
// post-op -- the same epilogue contract as splitk_reduce_kernel.
__global__ void splitk_reduce_t_kernel(const __grid_constant__ GemmArgs args) {
  const int64_t m = args.m_valid;
  const int64_t total = m * args.n_valid;
  const bool acc_mode = args.epilogue == EPI_ACCUMULATE;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx % m, c = idx / m;  // r fastest: the partials are read along their rows
    const float* w = args.ws + c * args.ws_ld + r;
    float v = w[0];
    for (int z = 1; z < args.k_split; ++z) v += w[z * args.ws_zstride];
    if (args.scaled) v *= args.alpha;
    const int64_t off = r * args.ldc + c;
    if (args.c_f64) {
      double* dst = static_cast<double*>(args.c) + off;
      *dst = acc_mode ? *dst + static_cast<double>(v) : static_cast<double>(v);
      continue;
    }
    float* dst = static_cast<float*>(args.c) + off;
    if (acc_mode) v += *dst;
    if (args.post == POST_BIAS_ACT) v = act_fwd(args.act, v + (args.bias ? args.bias[c] : 0.f));
    else if (args.post == POST_ACT_GRAD) v = v * act_grad_from_out(args.act, args.aux[r * args.ldaux + c]);
    *dst = v;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

int make_plane_tmap(CUtensorMap* out, const PlaneGeom& g, BoxKind box) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.cols), static_cast<cuuint64_t>(g.rows),
                        static_cast<cuuint64_t>(g.nplanes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.ld * 2), static_cast<cuuint64_t>(g.plane_stride * 2)};
  cuuint32_t boxd[3] = {64, 128, 1};
  if (box == BOX_MN64) boxd[1] = 64;
  if (box == BOX_K256) boxd[1] = 256;
  if (box == BOX_K64) boxd[1] = 64;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g.base, dims, strides, boxd, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : static_cast<int>(r);
}

bool group_uses_pairs(int m_valid) {
  // pairs (256-row units) unless they pad more rows than 128-row CTAs would
  const int r = m_valid % (2 * BM);
  return m_valid > BM && group_pairs_enabled() && (r == 0 || r > BM);
}

void gemm_boxes(bool a_mn, bool b_kmajor, int m_valid, BoxKind* box_a, BoxKind* box_b, bool grouped) {
  const bool pair = grouped ? group_uses_pairs(m_valid) : (m_valid > BM && gemm_pairs_enabled());
  *box_a = a_mn ? BOX_MN64 : BOX_K128;
  *box_b = b_kmajor ? (pair ? BOX_K128 : BOX_K256) : BOX_MN64;
}

template <int P>
static cudaError_t dispatch_planes(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, int k_split,
                                   bool a_mn, bool b_kmajor, bool pair, bool persistent, cudaStream_t stream,
                                   int sm_budget) {
  switch ((a_mn ? 4 : 0) | (b_kmajor ? 2 : 0) | (pair ? 1 : 0)) {
    case 0: return launch_variant<false, false, P, 1>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 1: return launch_variant<false, false, P, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 2: return launch_variant<false, true, P, 1>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 3: return launch_variant<false, true, P, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 4: return launch_variant<true, false, P, 1>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 5: return launch_variant<true, false, P, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    case 6: return launch_variant<true, true, P, 1>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
    default: return launch_variant<true, true, P, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
  }
}

static cudaError_t dispatch(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, int k_split, bool a_mn,
                            bool b_kmajor, bool pair, int planes, bool persistent, cudaStream_t stream,
                            int sm_budget = 0, bool mc = false) {
  if (mc && pair && !a_mn && !b_kmajor && planes <= 2)  // TMA-multicast clusters of two CTA pairs (opt-in)
    return planes == 2 ? launch_variant<false, false, 2, 2, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream)
                       : launch_variant<false, false, 1, 2, 2>(tmA, tmB, g, k_split, persistent, sm_budget, stream);
  switch (planes) {
    case 1: return dispatch_planes<1>(tmA, tmB, g, k_split, a_mn, b_kmajor, pair, persistent, stream, sm_budget);
    case 2: return dispatch_planes<2>(tmA, tmB, g, k_split, a_mn, b_kmajor, pair, persistent, stream, sm_budget);
    case 3: return dispatch_planes<3>(tmA, tmB, g, k_split, a_mn, b_kmajor, pair, persistent, stream, sm_budget);
    default: return cudaErrorInvalidValue;
  }
}

static bool args_ok(const GemmArgs& a) {
  return a.m_valid > 0 && a.n_valid > 0 && a.n_ksteps > 0 && a.n_ksteps <= kMaxKSteps;
}

cudaError_t launch_tile_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, bool a_mn,
                             bool b_kmajor, cudaStream_t stream) {
  if (!args_ok(args)) return cudaErrorInvalidValue;
  // CTA pairs once a tile has more than one 128-row block; single CTAs otherwise.
  const bool pair = args.m_valid > BM && gemm_pairs_enabled();
  GemmGroup g;
  g.n_tasks = 1;
  g.k_split = 1;  // split along the grid's z dimension instead
  g.task[0] = args;
  return dispatch(tmA, tmB, g, args.k_split, a_mn, b_kmajor, pair, args.planes, /*persistent=*/false, stream);
}

cudaError_t launch_tile_gemm_group(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, bool a_mn,
                                   bool b_kmajor, cudaStream_t stream) {
  return launch_tile_gemm_group(tmA, tmB, g, a_mn, b_kmajor, persistent_enabled(), stream);
}

cudaError_t launch_tile_gemm_group(const CUtensorMap& tmA, const CUtensorMap& tmB, GemmGroup& g, bool a_mn,
                                   bool b_kmajor, bool persistent, cudaStream_t stream, int sm_budget) {
  if (g.n_tasks < 1 || g.n_tasks > kMaxGroup) return cudaErrorInvalidValue;
  const bool pair = group_uses_pairs(g.task[0].m_valid);
  const int split = g.k_split > 1 ? g.k_split : 1;
  for (int t = 0; t < g.n_tasks; ++t) {
    const GemmArgs& a = g.task[t];
    if (!args_ok(a) || (a.k_split > 1 ? a.k_split : 1) != split || (split > 1 && !a.ws) ||
        a.planes != g.task[0].planes || group_uses_pairs(a.m_valid) != pair)
      return cudaErrorInvalidValue;
  }
  return dispatch(tmA, tmB, g, 1, a_mn, b_kmajor, pair, g.task[0].planes, persistent, stream, sm_budget);
}

// Whether a grouped launch runs as TMA-multicast clusters (two CTA pairs sharing
// A: 256 x 512 units, the A tile loaded once per cluster and multicast).  Opt-in
// (TR_GEMM_MC=1 / set_gemm_multicast): a B200 co-schedules only 33 clusters of
// four one-CTA-per-SM CTAs (132 SMs) against 74 pairs (148 SMs).
static std::atomic<int> g_mc{-1};

bool gemm_multicast_enabled() {
  int v = g_mc.load();
  if (v < 0) {
    const char* e = getenv("TR_GEMM_MC");
    v = (e && e[0] == '1') ? 1 : 0;
    g_mc.store(v);
  }
  return v != 0;
}

void set_gemm_multicast(bool on) { g_mc.store(on ? 1 : 0); }

static bool group_multicast(const GemmGroup& g, bool a_mn, bool b_kmajor, int sm_budget) {
  if (!gemm_multicast_enabled() || a_mn || b_kmajor || g.k_split > 1 || !group_uses_pairs(g.task[0].m_valid) ||
      g.task[0].planes > 2)
    return false;
  if (sm_budget > 0) {  // a green-context device: its SM count, not the whole GPU's
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess || sm_budget < sms)
      return false;
  }
  for (int t = 0; t < g.n_tasks; ++t)
    if (g.task[t].n_valid % (2 * BN) != 0 || g.task[t].k_split > 1) return false;
  return true;
}

cudaError_t launch_tile_gemm_group_maps(const CUtensorMap* maps, GemmGroup& g, bool a_mn, bool b_kmajor,
                                        bool persistent, cudaStream_t stream, int sm_budget) {
  if (g.n_tasks < 1 || g.n_tasks > kMaxGroup) return cudaErrorInvalidValue;
  BoxKind ba, bb;
  gemm_boxes(a_mn, b_kmajor, g.task[0].m_valid, &ba, &bb, /*grouped=*/true);
  if (!group_multicast(g, a_mn, b_kmajor, sm_budget))
    return launch_tile_gemm_group(maps[ba], maps[bb], g, a_mn, b_kmajor, persistent, stream, sm_budget);
  for (int t = 0; t < g.n_tasks; ++t)
    if (!args_ok(g.task[t]) || g.task[t].planes != g.task[0].planes || !group_uses_pairs(g.task[t].m_valid))
      return cudaErrorInvalidValue;
  // each CTA loads (and multicasts) a 64-row half of its A tile
  return dispatch(maps[BOX_K64], maps[bb], g, 1, a_mn, b_kmajor, /*pair=*/true, g.task[0].planes, persistent, stream,
                  sm_budget, /*mc=*/true);
}

cudaError_t launch_splitk_reduce(const GemmArgs& args, cudaStream_t stream) {
  if (args.k_split < 2 || !args.ws) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(args.m_valid) * args.n_valid;
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + threads - 1) / threads, 148 * 8));
  splitk_reduce_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

cudaError_t launch_splitk_reduce_t(const GemmArgs& args, cudaStream_t stream) {
  if (args.k_split < 1 || !args.ws || args.wt) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(args.m_valid) * args.n_valid;
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + threads - 1) / threads, 148 * 8));
  splitk_reduce_t_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

static std::atomic<int> g_narrow_tc{-1};

bool narrow_tc_enabled() {
  int v = g_narrow_tc.load();
  if (v < 0) {
    const char* e = getenv("TR_NARROW_TC");
    v = (e && e[0] == '0') ? 0 : 1;
    g_narrow_tc.store(v);
  }
  return v == 1;
}

void set_narrow_tc(bool on) { g_narrow_tc.store(on ? 1 : 0); }

static std::atomic<int> g_splitk{-1};

int splitk_max() {
  int v = g_splitk.load();
  if (v < 0) {
    const char* e = getenv("TR_SPLITK");
    v = e ? std::max(1, std::min(8, atoi(e))) : 8;
    g_splitk.store(v);
  }
  return v;
}

void set_splitk_max(int n) { g_splitk.store(std::max(1, std::min(8, n))); }

static std::atomic<int> g_pairs{-1};

bool gemm_pairs_enabled() {
  int v = g_pairs.load();
  if (v < 0) {
    // Default: single CTAs.  Measured on B200 (tools/probe_variants.py): pairs are
    // ~2% faster for one kernel alone but ~10% slower when two tasks' kernels
    // share the GPU (cluster placement is less flexible), which is the runtime's
    // normal state.  TR_GEMM_PAIRS=1 opts in.
    const char* e = getenv("TR_GEMM_PAIRS");
    v = (e && e[0] == '1') ? 1 : 0;
    g_pairs.store(v);
  }
  return v != 0;
}

void set_gemm_pairs(bool on) { g_pairs.store(on ? 1 : 0); }

static std::atomic<int> g_persistent{-1};

bool persistent_enabled() {
  int v = g_persistent.load();
  if (v < 0) {
    const char* e = getenv("TR_PERSISTENT");
    v = (e && e[0] == '0') ? 0 : 1;
    g_persistent.store(v);
  }
  return v != 0;
}

void set_persistent(bool on) { g_persistent.store(on ? 1 : 0); }

static std::atomic<int> g_group_pairs{-1};

bool group_pairs_enabled() {
  int v = g_group_pairs.load();
  if (v < 0) {
    // Grouped launches run one at a time per device, where CTA pairs win
    // (tools/probe_pairs.py: fp32acc +3%, bf16 +5% over single CTAs).
    const char* e = getenv("TR_GROUP_PAIRS");
    v = (e && e[0] == '0') ? 0 : 1;
    g_group_pairs.store(v);
  }
  return v != 0;
}

void set_group_pairs(bool on) { g_group_pairs.store(on ? 1 : 0); }

cudaError_t launch_split_convert(const void* src, int src_f64, int64_t ld_src, int64_t rows, int64_t cols,
                                 uint16_t* dst, int64_t ld_dst, int64_t rows_cap, int64_t plane_stride,
                                 int planes, cudaStream_t stream) {
  if (planes == 4) return launch_exact_convert(src, src_f64, ld_src, rows, cols, dst, ld_dst, stream);  // exact mode
  if (ld_dst % 8 != 0 || plane_stride % 8 != 0) return cudaErrorInvalidValue;
  // The kernel's TMA boxes never read past the valid extent rounded up to 256
  // (rows or columns), so only that part of the slot is written (zero padded);
  // a ragged 4096 x 10 tile converts 4096 x 256 elements, not 4096 x 4096.
  const int64_t rows_fill = std::min(rows_cap, (rows + 255) / 256 * 256);
  const int64_t cols_fill = std::min(ld_dst, (cols + 255) / 256 * 256);
  rows_cap = rows_fill;
  const int64_t total = rows_cap * (cols_fill / 8);
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
  if (src_f64)
    split_convert_kernel<double><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        static_cast<const double*>(src), ld_src, rows, cols, dst, ld_dst, rows_cap, cols_fill, plane_stride, planes);
  else
    split_convert_kernel<float><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        static_cast<const float*>(src), ld_src, rows, cols, dst, ld_dst, rows_cap, cols_fill, plane_stride, planes);
  return cudaGetLastError();
}

void die_map_prepare(int gpu) {
  if (gpu < 0 || gpu >= 64) return;
  if (const char* e = getenv("TR_K1_DIE"); e && e[0] == '0') return;
  {
    std::lock_guard<std::mutex> lk(g_die_mu);
    if (g_die_tried[gpu]) return;
    g_die_tried[gpu] = true;
  }
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(gpu) != cudaSuccess) return;
  DieMap* m = die_measure();
  if (prev >= 0) cudaSetDevice(prev);
  std::lock_guard<std::mutex> lk(g_die_mu);
  g_die[gpu] = m;
}

bool die_map_ready(int gpu, int* n0, int* n1) {
  const DieMap* m = die_lookup(gpu);
  if (!m) return false;
  if (n0) *n0 = m->n[0];
  if (n1) *n1 = m->n[1];
  return true;
}

}  // namespace tr
