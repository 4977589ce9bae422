// K3..K7: the elementwise / reduction steps of MLP training (ann.py) for
// device-resident float32 activations.  Each replaces a host-numpy float64 step
// of the reference:
//   K3 bias_act      Y = C + b ; A = act(Y)                       ann.py:155-158
//   K4 act_grad      dY = dOut * act'(Y, A)                       ann.py:222, 40-48
//   K4b mse_grad     dOut = 2 (pred - target) / size  (+ loss)    ann.py:51-56
//   K5 colsum        db = sum_rows dY                             ann.py:173
//   K6 sgd           W -= lr * dW                                 ann.py:243-247
// All are HBM-bound: grid-stride, 16-byte vector accesses where aligned.
#include <algorithm>
#include <cstdint>

#include <cuda_runtime.h>

#include "common.h"
#include "act.cuh"
#include "mlp_kernels.h"

namespace tr {
namespace {

constexpr int kThreads = 256;

int grid_for(int64_t n) {
  int64_t b = (n + kThreads * 4 - 1) / (kThreads * 4);
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<int>(b);
}

__global__ void bias_act_kernel(float* __restrict__ y, float* __restrict__ a, const float* __restrict__ bias,
                                int64_t rows, int64_t cols, int act) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v = y[i];
    if (bias) v += bias[i % cols];
    y[i] = v;
    a[i] = act_fwd(act, v);
  }
}

__global__ void act_grad_kernel(float* __restrict__ dy, const float* __restrict__ dout, const float* __restrict__ y,
                                const float* __restrict__ a, int64_t n, int act) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dy[i] = dout[i] * act_grad_from_out(act, a[i]);  // needs only the activation output (act.cuh)
}

// dout = 2 (pred - t) / n; loss partial sums of (pred - t)^2 in double, one atomic per block.
__global__ void mse_grad_kernel(float* __restrict__ dout, const float* __restrict__ pred,
                                const float* __restrict__ target, int64_t n, double* __restrict__ loss_sum) {
  __shared__ double part[kThreads / 32];
  double acc = 0.0;
  const float scale = 2.0f / static_cast<float>(n);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float d = pred[i] - target[i];
    dout[i] = scale * d;
    acc += static_cast<double>(d) * static_cast<double>(d);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += part[w];
    atomicAdd(loss_sum, s);
  }
}

// Column sums of a rows x cols matrix: each block owns 32 columns and loops over a
// slice of the rows; partial sums are combined with one atomic per column per block.
__global__ void colsum_kernel(const float* __restrict__ m, int64_t rows, int64_t cols, float* __restrict__ out) {
  const int64_t c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ty = threadIdx.x >> 5;  // 8 row lanes
  const int64_t r_per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * r_per, r1 = min(rows, r0 + r_per);
  __shared__ float part[8][33];
  float acc = 0.f;
  if (c < cols)
    for (int64_t r = r0 + ty; r < r1; r += 8) acc += m[r * cols + c];
  part[ty][threadIdx.x & 31] = acc;
  __syncthreads();
  if (ty == 0 && c < cols) {
    float s = 0.f;
    for (int k = 0; k < 8; ++k) s += part[k][threadIdx.x & 31];
    atomicAdd(&out[c], s);
  }
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] -= lr * g[i];
}

}  // namespace

cudaError_t mlp_bias_act(float* y, float* a, const float* bias, int64_t rows, int64_t cols, int act,
                         cudaStream_t s) {
  bias_act_kernel<<<grid_for(rows * cols), kThreads, 0, s>>>(y, a, bias, rows, cols, act);
  return cudaGetLastError();
}

cudaError_t mlp_act_grad(float* dy, const float* dout, const float* y, const float* a, int64_t n, int act,
                         cudaStream_t s) {
  act_grad_kernel<<<grid_for(n), kThreads, 0, s>>>(dy, dout, y, a, n, act);
  return cudaGetLastError();
}

cudaError_t mlp_mse_grad(float* dout, const float* pred, const float* target, int64_t n, double* loss_sum,
                         cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(loss_sum, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  mse_grad_kernel<<<grid_for(n), kThreads, 0, s>>>(dout, pred, target, n, loss_sum);
  return cudaGetLastError();
}

cudaError_t mlp_colsum(const float* m, int64_t rows, int64_t cols, float* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, static_cast<size_t>(cols) * sizeof(float), s);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>(std::min<int64_t>(64, (rows + 255) / 256)));
  colsum_kernel<<<grid, 256, 0, s>>>(m, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t mlp_sgd(float* w, const float* g, int64_t n, float lr, cudaStream_t s) {
  sgd_kernel<<<grid_for(n), kThreads, 0, s>>>(w, g, n, lr);
  return cudaGetLastError();
}

}  // namespace tr
