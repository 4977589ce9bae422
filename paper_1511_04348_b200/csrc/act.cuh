// Activations of the reference MLP (ann.py:30-48), shared by the elementwise
// kernels and the fused GEMM epilogues.  act'(.) is written in terms of the
// activation OUTPUT a only: sigmoid' = a(1 - a), relu' = [a > 0] (a > 0 iff
// y > 0), identity' = 1 -- so the pre-activation never has to be stored.
#pragma once

#include <cstdint>

namespace tr {

enum Activation : int32_t { ACT_IDENTITY = 0, ACT_SIGMOID = 1, ACT_RELU = 2 };

#ifdef __CUDACC__
__device__ __forceinline__ float act_fwd(int act, float y) {
  // y clamped at -80 keeps e^-y finite (<= 5.5e34 < 2^126), the range where the
  // fast reciprocal-based division is accurate to 2 ulp; sigmoid(-80) = 1.8e-35,
  // so the clamp moves no result by more than that.
  if (act == ACT_SIGMOID) return __fdividef(1.0f, 1.0f + __expf(-fmaxf(y, -80.f)));
  if (act == ACT_RELU) return y > 0.f ? y : 0.f;
  return y;
}

__device__ __forceinline__ float act_grad_from_out(int act, float a) {
  if (act == ACT_SIGMOID) return a * (1.0f - a);
  if (act == ACT_RELU) return a > 0.f ? 1.f : 0.f;
  return 1.f;
}

#endif  // __CUDACC__

}  // namespace tr
