// K3..K7 elementwise/reduction kernels of MLP training; see mlp_kernels.cu.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "act.cuh"

namespace tr {


cudaError_t mlp_bias_act(float* y, float* a, const float* bias, int64_t rows, int64_t cols, int act, cudaStream_t s);
cudaError_t mlp_act_grad(float* dy, const float* dout, const float* y, const float* a, int64_t n, int act,
                         cudaStream_t s);
cudaError_t mlp_mse_grad(float* dout, const float* pred, const float* target, int64_t n, int64_t n_mean,
                         double* loss_sum, cudaStream_t s);
cudaError_t mlp_colsum(const float* m, int64_t rows, int64_t cols, float* out, cudaStream_t s);
cudaError_t mlp_sgd(float* w, const float* g, int64_t n, float lr, cudaStream_t s);

}  // namespace tr
