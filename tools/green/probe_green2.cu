// Probe: which runtime call invalidates a green-context stream?  Dev tool.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(float* p) { p[threadIdx.x] += 1.f; }
int main(int argc, char** argv) {
  cudaSetDevice(0); cudaFree(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUdevResource all, rest; cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  CUdevResource g[32]; unsigned n = 18;
  cuDevSmResourceSplitByCount(g, &n, &all, &rest, 0, 8);
  CUdevResourceDesc desc; cuDevResourceGenerateDesc(&desc, g, 4);
  CUgreenCtx gc; cuGreenCtxCreate(&gc, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM);
  CUstream cs; cuGreenCtxStreamCreate(&cs, gc, CU_STREAM_NON_BLOCKING, 0);
  cudaStream_t s = (cudaStream_t)cs;
  float* p; cudaMalloc(&p, 1024);
  cudaEvent_t e; cudaEventCreate(&e);
  auto step = [&](const char* what) {
    k<<<1, 32, 0, s>>>(p);
    cudaError_t r1 = cudaGetLastError();
    cudaError_t r2 = cudaEventRecord(e, s);
    cudaError_t r3 = cudaStreamSynchronize(s);
    printf("%-28s launch=%s record=%s sync=%s\n", what, cudaGetErrorString(r1), cudaGetErrorString(r2), cudaGetErrorString(r3));
  };
  step("initial");
  cudaDeviceSynchronize(); step("after cudaDeviceSynchronize");
  float* q; cudaMalloc(&q, 1 << 20); step("after cudaMalloc");
  cudaMemcpy(q, p, 1024, cudaMemcpyDeviceToDevice); step("after cudaMemcpy");
  cudaFree(q); step("after cudaFree");
  cudaSetDevice(0); step("after cudaSetDevice");
  return 0;
}
