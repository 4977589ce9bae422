// K3..K7: the elementwise / reduction steps of MLP training (ann.py) for
// device-resident float32 activations.  Each replaces a host-numpy float64 step
// of the reference:
//   K3 bias_act      Y = C + b ; A = act(Y)                       ann.py:155-158
//   K4 act_grad      dY = dOut * act'(Y, A)                       ann.py:222, 40-48
//   K4b mse_grad     dOut = 2 (pred - target) / size  (+ loss)    ann.py:51-56
//   K5 colsum        db = sum_rows dY  (two passes, fixed order)   ann.py:173
//   K6 sgd           W -= lr * dW                                 ann.py:243-247
// All are HBM-bound: grid-stride, 16-byte vector accesses where aligned.
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

#include "common.h"
#include "act.cuh"
#include "devpool.h"
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
                                const float* __restrict__ target, int64_t n, int64_t n_mean,
                                double* __restrict__ block_sums) {
  __shared__ double part[kThreads / 32];
  double acc = 0.0;
  const float scale = 2.0f / static_cast<float>(n_mean);  // n_mean: elements of the (global) batch
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
    block_sums[blockIdx.x] = s;
  }
}

// One block: sum of n partials in a fixed order (deterministic loss).
__global__ void sum_partials_kernel(const double* __restrict__ parts, int n, double* __restrict__ out) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) acc += parts[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Column sums of a rows x cols matrix, pass 1: block (x, y) sums 32 columns over
// row slice y into part[y][c]; pass 2 adds the slices in order (deterministic).
__global__ void colsum_kernel(const float* __restrict__ m, int64_t rows, int64_t cols, float* __restrict__ part) {
  const int64_t c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ty = threadIdx.x >> 5;  // 8 row lanes
  const int64_t r_per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * r_per, r1 = min(rows, r0 + r_per);
  __shared__ float sh[8][33];
  float acc = 0.f;
  if (c < cols)
    for (int64_t r = r0 + ty; r < r1; r += 8) acc += m[r * cols + c];
  sh[ty][threadIdx.x & 31] = acc;
  __syncthreads();
  if (ty == 0 && c < cols) {
    float s = 0.f;
    for (int k = 0; k < 8; ++k) s += sh[k][threadIdx.x & 31];
    part[blockIdx.y * cols + c] = s;
  }
}

__global__ void colsum_finish_kernel(const float* __restrict__ part, int ny, int64_t cols, float* __restrict__ out) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int y = 0; y < ny; ++y) s += part[y * cols + c];
    out[c] = s;
  }
}

// The same sum for many blocks: 32 columns x 8 row lanes per CTA; lane y sums
// blocks y, y + 8, ... in order, then the 8 lane sums are added in order
// (a fixed order: bitwise reproducible).
__global__ void colsum_finish8_kernel(const float* __restrict__ part, int ny, int64_t cols, float* __restrict__ out) {
  const int64_t c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y0 = threadIdx.x >> 5;
  __shared__ float sh[8][33];
  float s = 0.f;
  if (c < cols)
    for (int y = y0; y < ny; y += 8) s += part[y * cols + c];
  sh[y0][threadIdx.x & 31] = s;
  __syncthreads();
  if (y0 == 0 && c < cols) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
    out[c] = t;
  }
}

__global__ void tile_colsum32_kernel(const float* __restrict__ m, int64_t ldm, int64_t rows, int64_t cols,
                                     float* __restrict__ part, int64_t ld_part) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
  if (c >= cols) return;
  const int n = static_cast<int>(min(rows - r0, static_cast<int64_t>(32)));
  const float* p = m + r0 * ldm + c;
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = r < n ? __ldg(p + r * ldm) : 0.f;  // all 32 loads in flight
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < 32; ++r) s += v[r];
  part[blockIdx.y * ld_part + c] = s;
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

// Grow-only scratch per (device, stream) for the two-pass reductions.  Reuse on
// the same stream is stream-ordered, so no synchronisation is needed (a
// stream-ordered allocator here would return memory at every sync point).
static cudaError_t stream_scratch(cudaStream_t s, size_t bytes, void** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> bufs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  auto& b = bufs[{dev, s}];
  if (b.second < bytes) {
    if (b.first) {
      e = cudaStreamSynchronize(s);  // the old buffer may still be in use on s
      if (e != cudaSuccess) return e;
      DevPool::get().release(dev, b.first, b.second);
      b = {nullptr, 0};
    }
    size_t cap = 0;
    e = DevPool::get().alloc(dev, std::max<size_t>(bytes, 1 << 20), &b.first, &cap);
    if (e != cudaSuccess) return e;
    b.second = cap;
  }
  *out = b.first;
  return cudaSuccess;
}

cudaError_t mlp_mse_grad(float* dout, const float* pred, const float* target, int64_t n, int64_t n_mean,
                         double* loss_sum, cudaStream_t s) {
  const int blocks = grid_for(n);
  double* parts = nullptr;
  cudaError_t e = stream_scratch(s, sizeof(double) * blocks, reinterpret_cast<void**>(&parts));
  if (e != cudaSuccess) return e;
  mse_grad_kernel<<<blocks, kThreads, 0, s>>>(dout, pred, target, n, n_mean, parts);
  sum_partials_kernel<<<1, kThreads, 0, s>>>(parts, blocks, loss_sum);
  return cudaGetLastError();
}

cudaError_t mlp_colsum_finish(const float* part, int64_t n_blocks, int64_t cols, float* out, cudaStream_t s) {
  colsum_finish8_kernel<<<static_cast<unsigned>((cols + 31) / 32), 256, 0, s>>>(part, static_cast<int>(n_blocks),
                                                                                cols, out);
  return cudaGetLastError();
}

cudaError_t tile_colsum32(const float* m, int64_t ldm, int64_t rows, int64_t cols, float* part, int64_t ld_part,
                          cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((cols + 255) / 256), static_cast<unsigned>((rows + 31) / 32));
  tile_colsum32_kernel<<<grid, 256, 0, s>>>(m, ldm, rows, cols, part, ld_part);
  return cudaGetLastError();
}

cudaError_t mlp_colsum(const float* m, int64_t rows, int64_t cols, float* out, cudaStream_t s) {
  const int ny = static_cast<int>(std::min<int64_t>(64, (rows + 255) / 256));
  float* part = nullptr;
  cudaError_t e = stream_scratch(s, sizeof(float) * ny * cols, reinterpret_cast<void**>(&part));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>(ny));
  colsum_kernel<<<grid, 256, 0, s>>>(m, rows, cols, part);
  colsum_finish_kernel<<<static_cast<unsigned>(std::min<int64_t>(148 * 4, (cols + 255) / 256)), 256, 0, s>>>(
      part, ny, cols, out);
  return cudaGetLastError();
}

cudaError_t mlp_sgd(float* w, const float* g, int64_t n, float lr, cudaStream_t s) {
  sgd_kernel<<<grid_for(n), kThreads, 0, s>>>(w, g, n, lr);
  return cudaGetLastError();
}

}  // namespace tr
