// Probe: can runtime-API kernels run on a green-context stream with cudaMalloc'd
// memory, confined to a subset of SMs?  Dev tool.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void busy(float* out, int iters) {
  float v = threadIdx.x;
  for (int i = 0; i < iters; ++i) v = v * 1.0000001f + 0.5f;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = v + smid * 0.f + (float)smid;
}

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs: %u\n", all.sm.smCount);
  CUdevResource groups[2], rest;
  unsigned n = 1;
  CK(cuDevSmResourceSplitByCount(groups, &n, &all, &rest, 0, 32));
  printf("group0 SMs: %u, rest %u\n", groups[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc desc;
  CK(cuDevResourceGenerateDesc(&desc, &groups[0], 1));
  CUgreenCtx g;
  CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream gs;
  CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
  float* out;
  RK(cudaMalloc(&out, 4096 * sizeof(float)));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  for (int pass = 0; pass < 2; ++pass) {
    cudaStream_t s = pass == 0 ? (cudaStream_t)0 : (cudaStream_t)gs;
    busy<<<1184, 128, 0, s>>>(out, 200000);
    RK(cudaGetLastError());
    RK(cudaStreamSynchronize(s));
    RK(cudaEventRecord(e0, s));
    busy<<<1184, 128, 0, s>>>(out, 200000);
    RK(cudaEventRecord(e1, s));
    RK(cudaEventSynchronize(e1));
    float ms = 0;
    RK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<float> h(1184);
    RK(cudaMemcpy(h.data(), out, 1184 * 4, cudaMemcpyDeviceToHost));
    std::vector<int> seen(256, 0);
    int distinct = 0;
    for (float v : h) { int sm = (int)v % 256; if (!seen[sm]++) ++distinct; }
    printf("%s: %.2f ms, distinct SMs used %d\n", pass == 0 ? "full GPU (default stream)" : "green ctx stream", ms, distinct);
  }
  printf("OK\n");
  return 0;
}
