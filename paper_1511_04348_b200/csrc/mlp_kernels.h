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
// out[c] = sum_b part[b * cols + c] over n_blocks blocks in order (tr_product.colsum)
cudaError_t mlp_colsum_finish(const float* part, int64_t n_blocks, int64_t cols, float* out, cudaStream_t s);
// 32-row block sums of one output tile (the fallback of a fused colsum):
// part[(r / 32) * ld_part + c] = sum of m[r..r+31][c] over the tile's valid rows
cudaError_t tile_colsum32(const float* m, int64_t ldm, int64_t rows, int64_t cols, float* part, int64_t ld_part,
                          cudaStream_t s);
cudaError_t mlp_sgd(float* w, const float* g, int64_t n, float lr, cudaStream_t s);

}  // namespace tr
