// Probe: which SMs share a die.  B200 = two dies, each with half the L2;
// addresses are homed on one die at fine grain, and an L2 hit costs more from
// the far die.  Every SM times dependent L2-only loads (ld.global.cg) of 256
// lines 2 KB apart (warm in L2); an SM's near/far pattern over the lines is its
// die's signature.  Also prints where a 2-CTA-cluster launch of 148 CTAs (the
// K1 pair grid) puts each cluster.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kLines = 256, kReps = 32, kStride = 2048 / 8;  // in uint64 units

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void warm(const uint64_t* buf, uint64_t* sink) {
  uint64_t s = 0;
  for (int j = threadIdx.x; j < kLines; j += blockDim.x) s += buf[j * kStride];
  if (s == 12345) *sink = s;
}

__global__ void probe(const uint64_t* buf, float* lat, int* sm_of_block) {
  extern __shared__ char pad[];
  if (threadIdx.x != 0) return;
  const uint32_t sm = smid();
  sm_of_block[blockIdx.x] = static_cast<int>(sm);
  for (int j = 0; j < kLines; ++j) {
    const uint64_t* p = buf + j * kStride;
    uint64_t a = reinterpret_cast<uint64_t>(p);
    // warm this line into the path once
    asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));
    a = reinterpret_cast<uint64_t>(p);
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < kReps; ++r) asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));
    const long long t1 = clock64();
    if (a == 0) sm_of_block[0] = -1;
    lat[sm * kLines + j] = static_cast<float>(t1 - t0) / kReps;
  }
}

__global__ void where(int* sm_of_block) {
  extern __shared__ char pad[];
  if (threadIdx.x == 0) sm_of_block[blockIdx.x] = static_cast<int>(smid());
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<uint64_t> h(static_cast<size_t>(kLines) * kStride, 0);
  uint64_t* buf;
  cudaMalloc(&buf, h.size() * 8);
  for (int j = 0; j < kLines; ++j) h[static_cast<size_t>(j) * kStride] = reinterpret_cast<uint64_t>(buf + j * kStride);
  cudaMemcpy(buf, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  float* lat;
  int* sob;
  uint64_t* sink;
  cudaMalloc(&lat, sizeof(float) * 256 * kLines);
  cudaMalloc(&sob, sizeof(int) * 1024);
  cudaMalloc(&sink, 8);
  cudaMemset(lat, 0, sizeof(float) * 256 * kLines);
  const int smem = 200 * 1024;  // one CTA per SM
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(where, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  warm<<<1, 256>>>(buf, sink);
  probe<<<nsm, 32, smem>>>(buf, lat, sob);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("probe: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> L(256 * kLines);
  cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost);
  // per line: threshold between the two latency modes = midpoint of min and max over SMs
  std::vector<float> thr(kLines);
  for (int j = 0; j < kLines; ++j) {
    float lo = 1e30f, hi = 0;
    for (int s = 0; s < nsm; ++s) { lo = std::min(lo, L[s * kLines + j]); hi = std::max(hi, L[s * kLines + j]); }
    thr[j] = 0.5f * (lo + hi);
  }
  // die of SM s = agreement of its near/far pattern with SM 0's
  std::vector<int> die(nsm);
  float near_sum = 0, far_sum = 0;
  int near_n = 0, far_n = 0;
  for (int s = 0; s < nsm; ++s) {
    int agree = 0;
    for (int j = 0; j < kLines; ++j) agree += (L[s * kLines + j] > thr[j]) == (L[0 * kLines + j] > thr[j]);
    die[s] = agree > kLines / 2 ? 0 : 1;
    for (int j = 0; j < kLines; ++j) {
      if (L[s * kLines + j] > thr[j]) { far_sum += L[s * kLines + j]; ++far_n; }
      else { near_sum += L[s * kLines + j]; ++near_n; }
    }
  }
  printf("latency: near %.1f cycles, far %.1f cycles (mean of the two modes)\n", near_sum / std::max(1, near_n),
         far_sum / std::max(1, far_n));
  int n0 = 0;
  printf("die of smid 0..%d:\n", nsm - 1);
  for (int s = 0; s < nsm; ++s) { printf("%d", die[s]); n0 += die[s] == 0; if (s % 74 == 73) printf("\n"); }
  printf("\ndie sizes: %d / %d\n", n0, nsm - n0);
  // where a 148-CTA, 2-CTA-cluster launch lands
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {
    cudaLaunchKernelEx(&cfg, where, sob);
    cudaDeviceSynchronize();
    std::vector<int> so(nsm);
    cudaMemcpy(so.data(), sob, nsm * 4, cudaMemcpyDeviceToHost);
    printf("cluster launch %d: cluster -> die (smid of its first CTA)\n", rep);
    for (int c = 0; c < nsm / 2; ++c) printf("%d", die[so[2 * c]]);
    printf("\n");
    for (int c = 0; c < nsm / 2; ++c) printf("%d ", so[2 * c]);
    printf("\n");
  }
  return 0;
}
