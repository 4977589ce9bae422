// K1s: the per-task tile GEMM on CUDA cores, for tiles a tensor-core launch
// would mostly pad.  See tile_gemm.h (small_gemm_eligible / launch_small_gemm).
//
// Two shapes reach it in the reference's MLP (ann.py:151-174, 784-...-10):
//   * narrow outputs (n <= 32): the 10-wide output layer's forward product and
//     its dW.  A 128 x 256 MMA tile would be 96% padding; here a CTA owns a
//     256 x 16 block, k split across CTAs (partials reduced in z order by
//     launch_splitk_reduce), and the product streams the A tile once.
//   * tiny contractions (k <= 32): the output layer's dX = dY W^T, a 4096 x
//     4096 tile per task over k = 10 -- a store-bound product (C, the fused
//     act_grad read and the write-through planes).
// Operands are the tile-cache planes the tensor-core kernel reads (hi, lo bf16),
// re-assembled as hi + lo in fp32 -- the same 16 significant bits the three
// MMAs use -- and accumulated with fp32 FMA in ascending k: deterministic, and
// within the FP32-accurate tolerance.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include <cuda_bf16.h>

#include "act.cuh"
#include "tile_gemm.h"

namespace tr {

namespace {

constexpr int KC = 32;    // k per shared-memory chunk
constexpr int NTH = 256;  // threads per CTA; each owns a 4 x 4 output block

__device__ __forceinline__ float bf16f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

// 8 consecutive bf16 at p (hi plane) and p + ps (lo plane), `n` of them valid
// (the rest 0): vector loads when all 8 are, else element by element.  Issued
// for a whole chunk before any is used, so a thread has all its loads in flight.
__device__ __forceinline__ void fetch8(const uint16_t* __restrict__ p, int64_t ps, int planes, int n, uint4& h,
                                       uint4& l) {
  if (n >= 8) {
    h = __ldg(reinterpret_cast<const uint4*>(p));
    l = planes == 2 ? __ldg(reinterpret_cast<const uint4*>(p + ps)) : make_uint4(0, 0, 0, 0);
    return;
  }
  uint16_t hs[8], ls[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    hs[j] = j < n ? p[j] : uint16_t(0);
    ls[j] = (j < n && planes == 2) ? p[ps + j] : uint16_t(0);
  }
  h = *reinterpret_cast<const uint4*>(hs);
  l = *reinterpret_cast<const uint4*>(ls);
}

// hi + lo of 8 packed pairs as fp32 (an all-zero lo plane adds nothing)
__device__ __forceinline__ void unpack8(const uint4& h, const uint4& l, float (&v)[8]) {
  const uint16_t* hs = reinterpret_cast<const uint16_t*>(&h);
  const uint16_t* ls = reinterpret_cast<const uint16_t*>(&l);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = bf16f(hs[j]) + bf16f(ls[j]);
}

__device__ __forceinline__ void split_store(uint16_t* dst, int64_t plane, int planes, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  dst[0] = __bfloat16_as_ushort(h);
  // an infinite hi carries the value alone (lo = 0, not inf - inf = NaN)
  const float hf = __bfloat162float(h);
  if (planes == 2) dst[plane] = __bfloat16_as_ushort(__float2bfloat16_rn(isinf(hf) ? 0.f : v - hf));
}

// 4 consecutive values into the planes (8-byte stores; dst 4-element aligned)
__device__ __forceinline__ void split_store4(uint16_t* dst, int64_t plane, int planes, float4 v) {
  const float x[4] = {v.x, v.y, v.z, v.w};
  uint16_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat16 b = __float2bfloat16_rn(x[i]);
    h[i] = __bfloat16_as_ushort(b);
    const float bf = __bfloat162float(b);
    l[i] = __bfloat16_as_ushort(__float2bfloat16_rn(isinf(bf) ? 0.f : x[i] - bf));
  }
  *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(h);
  if (planes == 2) *reinterpret_cast<uint2*>(dst + plane) = *reinterpret_cast<const uint2*>(l);
}

// One CTA: a BM x BN output block (BM = 16 * 256 / BN rows), k-chunks
// [lo, hi) of the task's chunk list (split-K share z = blockIdx.z).
template <bool A_MN, bool B_K, int BN>
__global__ void __launch_bounds__(NTH) small_gemm_kernel(const uint16_t* __restrict__ slab, int64_t ld, int64_t ps,
                                                         const __grid_constant__ GemmArgs args) {
  constexpr int TX = BN / 4;        // threads across the block's columns
  constexpr int BM = (NTH / TX) * 4;
  constexpr int LDA = BM + 4;       // float4-aligned rows
  __shared__ __align__(16) float As[KC][LDA];
  __shared__ __align__(16) float Bs[KC][BN + 4];

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int planes = args.planes;

  int total = 0;
  for (int s = 0; s < args.n_ksteps; ++s) total += (args.k_len[s] + KC - 1) / KC;
  const int nz = static_cast<int>(gridDim.z);
  const int lo = static_cast<int>((static_cast<int64_t>(blockIdx.z) * total) / nz);
  const int hi = static_cast<int>((static_cast<int64_t>(blockIdx.z + 1) * total) / nz);

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  int ks = 0, kk = 0, g = 0;  // walk the chunk list to this CTA's first chunk
  while (g < lo) {
    kk += KC;
    if (kk >= args.k_len[ks]) {
      ++ks;
      kk = 0;
    }
    ++g;
  }
  // Software pipeline: chunk g+1's global loads are in flight (registers)
  // while chunk g is multiplied out of shared memory.
  constexpr int AIT = (BM * KC / 8 + NTH - 1) / NTH;
  constexpr int BIT = (KC * BN / 8 + NTH - 1) / NTH;
  uint4 ah[AIT], al[AIT], bh[BIT], bl[BIT];
  auto fetch = [&](int fks, int fkk) {  // A (BM x KC) and B (KC x BN) of chunk (fks, fkk)
    const int klen = args.k_len[fks];
    const uint16_t* pa = slab + static_cast<int64_t>(args.a_z[fks]) * ps;
    const uint16_t* pb = slab + static_cast<int64_t>(args.b_z[fks]) * ps;
#pragma unroll
    for (int it = 0; it < AIT; ++it) {
      const int idx = it * NTH + tid;
      if (idx >= BM * KC / 8) break;
      if (!A_MN) {  // stored M x K: 8 consecutive k of one row
        const int r = idx / (KC / 8), kq = (idx % (KC / 8)) * 8;
        const int n = (m0 + r < args.m_valid) ? klen - (fkk + kq) : 0;
        fetch8(pa + static_cast<int64_t>(m0 + r) * ld + fkk + kq, ps, planes, n, ah[it], al[it]);
      } else {      // stored K x M: 8 consecutive m of one k
        const int k = idx / (BM / 8), mq = (idx % (BM / 8)) * 8;
        const int n = (fkk + k < klen) ? args.m_valid - (m0 + mq) : 0;
        fetch8(pa + static_cast<int64_t>(fkk + k) * ld + m0 + mq, ps, planes, n, ah[it], al[it]);
      }
    }
#pragma unroll
    for (int it = 0; it < BIT; ++it) {
      const int idx = it * NTH + tid;
      if (idx >= KC * BN / 8) break;
      if (B_K) {    // stored N x K: 8 consecutive k of one column
        const int c = idx / (KC / 8), kq = (idx % (KC / 8)) * 8;
        const int n = (n0 + c < args.n_valid) ? klen - (fkk + kq) : 0;
        fetch8(pb + static_cast<int64_t>(n0 + c) * ld + fkk + kq, ps, planes, n, bh[it], bl[it]);
      } else {      // stored K x N: 8 consecutive n of one k
        const int k = idx / (BN / 8), nq = (idx % (BN / 8)) * 8;
        const int n = (fkk + k < klen) ? args.n_valid - (n0 + nq) : 0;
        fetch8(pb + static_cast<int64_t>(fkk + k) * ld + n0 + nq, ps, planes, n, bh[it], bl[it]);
      }
    }
  };
  auto stash = [&] {  // the fetched chunk, fp32, into As[k][m] and Bs[k][n]
#pragma unroll
    for (int it = 0; it < AIT; ++it) {
      const int idx = it * NTH + tid;
      if (idx >= BM * KC / 8) break;
      float v[8];
      unpack8(ah[it], al[it], v);
      if (!A_MN) {
        const int r = idx / (KC / 8), kq = (idx % (KC / 8)) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) As[kq + j][r] = v[j];
      } else {
        const int k = idx / (BM / 8), mq = (idx % (BM / 8)) * 8;
        *reinterpret_cast<float4*>(&As[k][mq]) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(&As[k][mq + 4]) = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
#pragma unroll
    for (int it = 0; it < BIT; ++it) {
      const int idx = it * NTH + tid;
      if (idx >= KC * BN / 8) break;
      float v[8];
      unpack8(bh[it], bl[it], v);
      if (B_K) {
        const int c = idx / (KC / 8), kq = (idx % (KC / 8)) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) Bs[kq + j][c] = v[j];
      } else {
        const int k = idx / (BN / 8), nq = (idx % (BN / 8)) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) Bs[k][nq + j] = v[j];
      }
    }
  };
  if (g < hi) fetch(ks, kk);
  for (; g < hi; ++g) {
    stash();
    __syncthreads();
    const int kn = min(KC, args.k_len[ks] - kk);  // this chunk's extent
    kk += KC;
    if (kk >= args.k_len[ks]) {
      ++ks;
      kk = 0;
    }
    if (g + 1 < hi) fetch(ks, kk);  // the next chunk, while this one is multiplied
#pragma unroll 8
    for (int k = 0; k < kn; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

  // ---- epilogue: the same contract as the tensor-core kernel's.  A thread's 4
  // columns of a row are contiguous: one 16-byte access per row when aligned.
  const bool part = nz > 1;
  const bool acc_mode = !part && args.epilogue == EPI_ACCUMULATE;
  const int post = part ? static_cast<int>(POST_NONE) : args.post;
  float* const base = part ? args.ws + blockIdx.z * args.ws_zstride : static_cast<float*>(args.c);
  const int64_t ldo = part ? args.ws_ld : args.ldc;
  const int64_t c0 = n0 + tx * 4;
  if (args.scaled && !part)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] *= args.alpha;
  const bool vec = (part || !args.c_f64) && c0 + 4 <= args.n_valid && (ldo & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(base) & 15) == 0 &&
                   (!args.aux || ((args.ldaux & 3) == 0 && (reinterpret_cast<uintptr_t>(args.aux) & 15) == 0)) &&
                   (!args.wt || (args.wt_ld & 3) == 0);
  // fused column sums (args.colsum): this thread's 4 columns over its 4 rows,
  // then the 8 threads of each 32-row block are summed in row order below
  const bool do_cs = !part && !args.c_f64 && args.colsum != nullptr;
  float csum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty * 4 + i;
    if (r >= args.m_valid) break;
    if (vec) {
      float4* d4 = reinterpret_cast<float4*>(base + r * ldo + c0);
      float4 v = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      if (!part) {
        if (acc_mode) {
          const float4 o = *d4;
          v.x += o.x, v.y += o.y, v.z += o.z, v.w += o.w;
        }
        if (post == POST_BIAS_ACT) {
          const float* bb = args.bias ? args.bias + c0 : nullptr;
          v.x = act_fwd(args.act, v.x + (bb ? bb[0] : 0.f));
          v.y = act_fwd(args.act, v.y + (bb ? bb[1] : 0.f));
          v.z = act_fwd(args.act, v.z + (bb ? bb[2] : 0.f));
          v.w = act_fwd(args.act, v.w + (bb ? bb[3] : 0.f));
        } else if (post == POST_ACT_GRAD) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(args.aux + r * args.ldaux + c0));
          v.x *= act_grad_from_out(args.act, a.x);
          v.y *= act_grad_from_out(args.act, a.y);
          v.z *= act_grad_from_out(args.act, a.z);
          v.w *= act_grad_from_out(args.act, a.w);
        }
      }
      *d4 = v;
      if (do_cs) {
        csum[0] += v.x;
        csum[1] += v.y;
        csum[2] += v.z;
        csum[3] += v.w;
      }
      if (!part && args.wt) split_store4(args.wt + r * args.wt_ld + c0, args.wt_plane, planes, v);
      continue;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = c0 + j;
      if (c >= args.n_valid) break;
      float v = acc[i][j];
      if (part) {
        base[r * ldo + c] = v;
        continue;
      }
      if (args.c_f64) {
        double* dst = static_cast<double*>(args.c) + r * args.ldc + c;
        *dst = acc_mode ? *dst + static_cast<double>(v) : static_cast<double>(v);
        continue;
      }
      float* dst = static_cast<float*>(args.c) + r * args.ldc + c;
      if (acc_mode) v += *dst;
      if (post == POST_BIAS_ACT) v = act_fwd(args.act, v + (args.bias ? args.bias[c] : 0.f));
      else if (post == POST_ACT_GRAD) v *= act_grad_from_out(args.act, args.aux[r * args.ldaux + c]);
      *dst = v;
      if (do_cs) csum[j] += v;
      if (args.wt) split_store(args.wt + r * args.wt_ld + c, args.wt_plane, planes, v);
    }
  }
  if (do_cs) {  // (block-uniform branch) 32-row blocks = 8 consecutive ty; sum them in order
    float(*red)[BN] = reinterpret_cast<float(*)[BN]>(&As[0][0]);  // (NTH / TX) x BN floats
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) red[ty][tx * 4 + j] = csum[j];
    __syncthreads();
    if (ty % 8 == 0 && m0 + ty * 4 < args.m_valid) {
      for (int j = 0; j < 4; ++j) {
        const int64_t c = c0 + j;
        if (c >= args.n_valid) break;
        float s = 0.f;
        for (int y = ty; y < ty + 8; ++y) s += red[y][tx * 4 + j];
        args.colsum[((m0 + ty * 4) / 32) * args.colsum_ld + c] = s;
      }
    }
  }
}

template <bool A_MN, bool B_K, int BN>
cudaError_t launch_small(const uint16_t* slab, int64_t ld, int64_t ps, const GemmArgs& args, cudaStream_t stream) {
  constexpr int BM = (NTH / (BN / 4)) * 4;
  dim3 grid((args.m_valid + BM - 1) / BM, (args.n_valid + BN - 1) / BN, args.k_split > 1 ? args.k_split : 1);
  small_gemm_kernel<A_MN, B_K, BN><<<grid, NTH, 0, stream>>>(slab, ld, ps, args);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_small_bn(const uint16_t* slab, int64_t ld, int64_t ps, const GemmArgs& args, bool a_mn, bool b_k,
                            cudaStream_t stream) {
  if (a_mn) return b_k ? launch_small<true, true, BN>(slab, ld, ps, args, stream)
                       : launch_small<true, false, BN>(slab, ld, ps, args, stream);
  return b_k ? launch_small<false, true, BN>(slab, ld, ps, args, stream)
             : launch_small<false, false, BN>(slab, ld, ps, args, stream);
}

int total_k(const GemmArgs& args) {
  int k = 0;
  for (int s = 0; s < args.n_ksteps; ++s) k += args.k_len[s];
  return k;
}

std::atomic<int> g_small{-1};

}  // namespace

bool small_gemm_enabled() {
  int v = g_small.load();
  if (v < 0) {
    const char* e = std::getenv("TR_SMALL_GEMM");
    v = (e && e[0] == '0') ? 0 : 1;
    g_small.store(v);
  }
  return v == 1;
}

void set_small_gemm(bool on) { g_small.store(on ? 1 : 0); }

bool small_gemm_eligible(const GemmArgs& args) {
  // hi + lo planes only: fp32hi's third plane stays on the tensor cores
  return args.planes <= 2 && (args.n_valid <= kSmallMaxN || total_k(args) <= kSmallMaxK);
}

int small_gemm_split(const GemmArgs& args, int sms) {
  if (args.n_valid > kSmallMaxN || splitk_max() < 2) return 1;  // tiny contraction: nothing to split
  const int64_t ctas = ((args.m_valid + 255) / 256) * static_cast<int64_t>((args.n_valid + 15) / 16);
  int chunks = 0;
  for (int s = 0; s < args.n_ksteps; ++s) chunks += (args.k_len[s] + KC - 1) / KC;
  const int64_t want = (4LL * sms + ctas - 1) / ctas;  // ~4 CTAs per SM
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({want, 32, chunks / 8})));
}

cudaError_t launch_small_gemm(const uint16_t* slab, int64_t ld, int64_t plane_stride, const GemmArgs& args,
                              bool a_mn, bool b_kmajor, cudaStream_t stream) {
  // narrow outputs: 256 x 16 blocks; tiny contractions: 64 x 64 blocks (wider stores)
  if (args.n_valid <= kSmallMaxN) return launch_small_bn<16>(slab, ld, plane_stride, args, a_mn, b_kmajor, stream);
  return launch_small_bn<64>(slab, ld, plane_stride, args, a_mn, b_kmajor, stream);
}

}  // namespace tr
