// KX: the reference's own arithmetic on the GPU (precision "exact").
//
// The reference accumulates C in place, one rank-1 update per contraction
// index in ascending k, each element as a rounded multiply then a rounded add
// in the output's dtype (tiles.py:170-171 / 197-212: numpy `out += a[:, k] *
// b[k, :]`, no fused multiply-add).  This kernel does exactly that per output
// element -- acc = acc + a * b with __dmul_rn / __dadd_rn (or the fp32
// intrinsics when both operands and the output are float32; their values are
// exact in the float64 tiles), k ascending across all of a task's k-steps,
// starting from 0 or, for an accumulating launch, from the element's current
// value -- so results are bit for bit the reference's, whatever the tile size,
// device count or schedule.  A float32 output with a float64 operand (the
// scheduled product keeps A's dtype, scheduler.py:182) follows numpy's in-place
// `out += outer(a, b)`: a float64 product and sum, rounded to float32 every k.
//
// Tiles sit in the tile cache as float64 (8 bytes per element: the slot's four
// bf16 "planes" hold one row-major tile of `ld` doubles per row).  CUDA cores:
// 128 x 128 outputs per CTA, 8 x 8 per thread, double-buffered shared-memory
// chunks of 8 values of k; the bound is the FP64 (FP32) pipe issuing separate
// multiplies and adds -- the mode is for bit-exact parity, not speed.
#include <algorithm>
#include <cstdint>

#include "tile_gemm.h"

namespace tr {

namespace {

constexpr int XB = 128;   // output block: 128 x 128 per CTA
constexpr int XKC = 8;    // k per shared-memory chunk (double-buffered)
constexpr int XNTH = 256; // 16 x 16 threads, 8 x 8 outputs each (rows ty + 16 i, columns tx + 16 j)

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

// One k-chunk of the A and B tiles into shared memory as [k][row] / [k][col].
// Element (m, k) of A / (k, n) of B of k-step ks: stored tiles are row-major
// `ld` doubles per row; a transposed operand reads its stored tile (k, m) /
// (n, k).  The thread -> element map keeps each warp's global reads contiguous:
// k fastest where k is the stored tile's column, else the row/column index.
template <typename T, bool A_MN, bool B_K>
__device__ __forceinline__ void load_chunk(T (*As)[XB], T (*Bs)[XB], const double* ta, const double* tb, int64_t ld,
                                           int m0, int n0, int k0, int kn, const GemmArgs& args) {
#pragma unroll
  for (int r = 0; r < XKC * XB / XNTH; ++r) {
    const int e = threadIdx.x + r * XNTH;
    {
      const int kk = A_MN ? e / XB : e % XKC;
      const int mm = A_MN ? e % XB : e / XKC;
      const int m = m0 + mm, k = k0 + kk;
      double v = 0.0;
      if (kk < kn && m < args.m_valid) v = A_MN ? ta[static_cast<int64_t>(k) * ld + m] : ta[static_cast<int64_t>(m) * ld + k];
      As[kk][mm] = static_cast<T>(v);
    }
    {
      const int kk = B_K ? e % XKC : e / XB;
      const int nn = B_K ? e / XKC : e % XB;
      const int n = n0 + nn, k = k0 + kk;
      double w = 0.0;
      if (kk < kn && n < args.n_valid) w = B_K ? tb[static_cast<int64_t>(n) * ld + k] : tb[static_cast<int64_t>(k) * ld + n];
      Bs[kk][nn] = static_cast<T>(w);
    }
  }
}

// T: the arithmetic type; R32: round the running sum to float32 after every
// update (float32 output, float64 arithmetic)
template <typename T, bool A_MN, bool B_K, bool R32 = false>
__global__ void __launch_bounds__(XNTH) exact_gemm_kernel(const double* __restrict__ a_base,
                                                          const double* __restrict__ b_base, int64_t ld,
                                                          int64_t slot_doubles, const __grid_constant__ GemmArgs args) {
  __shared__ T As[2][XKC][XB];
  __shared__ T Bs[2][XKC][XB];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.x * XB, n0 = blockIdx.y * XB;
  T acc[8][8];
  const bool acc_mode = args.epilogue == EPI_ACCUMULATE;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t r = m0 + ty + 16 * i, c = n0 + tx + 16 * j;
      T v = T(0);
      if (acc_mode && r < args.m_valid && c < args.n_valid)
        v = args.c_f64 ? static_cast<T>(static_cast<const double*>(args.c)[r * args.ldc + c])
                       : static_cast<T>(static_cast<const float*>(args.c)[r * args.ldc + c]);
      acc[i][j] = v;
    }
  // the chunks of all k-steps in ascending k, double-buffered: chunk c + 1 is
  // loaded while chunk c is consumed
  int ks = 0, k0 = 0, buf = 0;
  auto step_ptrs = [&](int s, const double*& ta, const double*& tb) {
    ta = a_base + static_cast<int64_t>(args.a_z[s] / 4) * slot_doubles;
    tb = b_base + static_cast<int64_t>(args.b_z[s] / 4) * slot_doubles;
  };
  const double *ta, *tb;
  step_ptrs(0, ta, tb);
  int kn = min(XKC, args.k_len[0]);
  load_chunk<T, A_MN, B_K>(As[0], Bs[0], ta, tb, ld, m0, n0, 0, kn, args);
  __syncthreads();
  while (true) {
    // next chunk's coordinates
    int nks = ks, nk0 = k0 + XKC;
    if (nk0 >= args.k_len[ks]) {
      nks = ks + 1;
      nk0 = 0;
    }
    const bool more = nks < args.n_ksteps;
    int nkn = 0;
    if (more) {
      const double *na, *nb;
      step_ptrs(nks, na, nb);
      nkn = min(XKC, args.k_len[nks] - nk0);
      load_chunk<T, A_MN, B_K>(As[buf ^ 1], Bs[buf ^ 1], na, nb, ld, m0, n0, nk0, nkn, args);
    }
    for (int kk = 0; kk < kn; ++kk) {  // ascending k, one rounded multiply and add each
      T av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j] = add_rn(acc[i][j], mul_rn(av[i], bv[j]));
          if constexpr (R32) acc[i][j] = static_cast<T>(__double2float_rn(acc[i][j]));
        }
    }
    __syncthreads();
    if (!more) break;
    ks = nks;
    k0 = nk0;
    kn = nkn;
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t r = m0 + ty + 16 * i, c = n0 + tx + 16 * j;
      if (r >= args.m_valid || c >= args.n_valid) continue;
      if (args.c_f64) static_cast<double*>(args.c)[r * args.ldc + c] = static_cast<double>(acc[i][j]);
      else static_cast<float*>(args.c)[r * args.ldc + c] = static_cast<float>(acc[i][j]);
    }
}

template <typename T>
__global__ void exact_convert_kernel(const T* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                                     double* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    dst[r * ld_dst + c] = static_cast<double>(src[r * ld_src + c]);
  }
}

template <typename T, bool A_MN, bool B_K, bool R32 = false>
cudaError_t launch_x(const double* a_base, const double* b_base, int64_t ld, int64_t slot_doubles,
                     const GemmArgs& args, cudaStream_t s) {
  dim3 grid((args.m_valid + XB - 1) / XB, (args.n_valid + XB - 1) / XB);
  exact_gemm_kernel<T, A_MN, B_K, R32><<<grid, XNTH, 0, s>>>(a_base, b_base, ld, slot_doubles, args);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_exact_gemm(const void* a_base, const void* b_base, int64_t ld, int64_t slot_doubles,
                              const GemmArgs& args, bool a_mn, bool b_kmajor, bool f32_operands,
                              cudaStream_t stream) {
  if (args.m_valid < 1 || args.n_valid < 1 || args.n_ksteps < 1 || args.k_split > 1 || args.post != POST_NONE ||
      args.scaled || args.wt || args.colsum)
    return cudaErrorInvalidValue;
  const double* a = static_cast<const double*>(a_base);
  const double* b = static_cast<const double*>(b_base);
  if (!args.c_f64 && !f32_operands) {  // float32 output, a float64 operand
    switch ((a_mn ? 2 : 0) | (b_kmajor ? 1 : 0)) {
      case 0: return launch_x<double, false, false, true>(a, b, ld, slot_doubles, args, stream);
      case 1: return launch_x<double, false, true, true>(a, b, ld, slot_doubles, args, stream);
      case 2: return launch_x<double, true, false, true>(a, b, ld, slot_doubles, args, stream);
      default: return launch_x<double, true, true, true>(a, b, ld, slot_doubles, args, stream);
    }
  }
  const int v = (args.c_f64 ? 4 : 0) | (a_mn ? 2 : 0) | (b_kmajor ? 1 : 0);
  switch (v) {
    case 0: return launch_x<float, false, false>(a, b, ld, slot_doubles, args, stream);
    case 1: return launch_x<float, false, true>(a, b, ld, slot_doubles, args, stream);
    case 2: return launch_x<float, true, false>(a, b, ld, slot_doubles, args, stream);
    case 3: return launch_x<float, true, true>(a, b, ld, slot_doubles, args, stream);
    case 4: return launch_x<double, false, false>(a, b, ld, slot_doubles, args, stream);
    case 5: return launch_x<double, false, true>(a, b, ld, slot_doubles, args, stream);
    case 6: return launch_x<double, true, false>(a, b, ld, slot_doubles, args, stream);
    default: return launch_x<double, true, true>(a, b, ld, slot_doubles, args, stream);
  }
}

cudaError_t launch_exact_convert(const void* src, int src_f64, int64_t ld_src, int64_t rows, int64_t cols, void* dst,
                                 int64_t ld_dst, cudaStream_t stream) {
  const int64_t total = rows * cols;
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + threads - 1) / threads, 148 * 16));
  if (src_f64)
    exact_convert_kernel<double><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        static_cast<const double*>(src), ld_src, rows, cols, static_cast<double*>(dst), ld_dst);
  else
    exact_convert_kernel<float><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        static_cast<const float*>(src), ld_src, rows, cols, static_cast<double*>(dst), ld_dst);
  return cudaGetLastError();
}

}  // namespace tr
