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
// bf16 "planes" hold one row-major tile of `ld` doubles per row).  CUDA cores,
// shared-memory chunks of KC values of k; throughput is the float64 / fp32
// vector rate without FMA -- the mode is for bit-exact parity, not speed.
#include <algorithm>
#include <cstdint>

#include "tile_gemm.h"

namespace tr {

namespace {

constexpr int XB = 64;    // output block: 64 x 64 per CTA
constexpr int XKC = 16;   // k per shared-memory chunk
constexpr int XNTH = 256; // 16 x 16 threads, 4 x 4 outputs each

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

// A tile element (m, k) / B tile element (k, n) of k-step ks: stored tiles are
// row-major `ld` doubles per row; a transposed operand reads its stored tile
// (k, m) / (n, k).
// T: the arithmetic type; R32: round the running sum to float32 after every
// update (float32 output, float64 arithmetic)
template <typename T, bool A_MN, bool B_K, bool R32 = false>
__global__ void __launch_bounds__(XNTH) exact_gemm_kernel(const double* __restrict__ a_base,
                                                          const double* __restrict__ b_base, int64_t ld,
                                                          int64_t slot_doubles, const __grid_constant__ GemmArgs args) {
  __shared__ T As[XKC][XB + 1];
  __shared__ T Bs[XKC][XB + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.x * XB, n0 = blockIdx.y * XB;
  T acc[4][4];
  const bool acc_mode = args.epilogue == EPI_ACCUMULATE;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      T v = T(0);
      if (acc_mode && r < args.m_valid && c < args.n_valid)
        v = args.c_f64 ? static_cast<T>(static_cast<const double*>(args.c)[r * args.ldc + c])
                       : static_cast<T>(static_cast<const float*>(args.c)[r * args.ldc + c]);
      acc[i][j] = v;
    }
  for (int ks = 0; ks < args.n_ksteps; ++ks) {
    const double* ta = a_base + static_cast<int64_t>(args.a_z[ks] / 4) * slot_doubles;
    const double* tb = b_base + static_cast<int64_t>(args.b_z[ks] / 4) * slot_doubles;
    const int klen = args.k_len[ks];
    for (int k0 = 0; k0 < klen; k0 += XKC) {
      const int kn = min(XKC, klen - k0);
      for (int e = threadIdx.x; e < XKC * XB; e += XNTH) {
        const int kk = e / XB, mm = e % XB;  // mm fastest: coalesced along the stored rows when A is MN-major
        const int m = m0 + mm, k = k0 + kk;
        double v = 0.0;
        if (kk < kn && m < args.m_valid) v = A_MN ? ta[static_cast<int64_t>(k) * ld + m] : ta[static_cast<int64_t>(m) * ld + k];
        As[kk][mm] = static_cast<T>(v);
        const int n = n0 + mm;
        double w = 0.0;
        if (kk < kn && n < args.n_valid) w = B_K ? tb[static_cast<int64_t>(n) * ld + k] : tb[static_cast<int64_t>(k) * ld + n];
        Bs[kk][mm] = static_cast<T>(w);
      }
      __syncthreads();
      for (int kk = 0; kk < kn; ++kk) {  // ascending k, one rounded multiply and add each
        T av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j] = add_rn(acc[i][j], mul_rn(av[i], bv[j]));
            if constexpr (R32) acc[i][j] = static_cast<T>(__double2float_rn(acc[i][j]));
          }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
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
