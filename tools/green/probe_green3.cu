// Probe: event reuse on a green-context stream after cudaEventElapsedTime /
// cross-thread launches.  Dev tool.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <thread>
__global__ void k(float* p) { p[threadIdx.x] += 1.f; }
#define P(what, x) printf("%-40s %s\n", what, cudaGetErrorString(x))
int main() {
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
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  P("record e0", cudaEventRecord(e0, s));
  k<<<1, 32, 0, s>>>(p);
  P("record e1", cudaEventRecord(e1, s));
  P("sync", cudaStreamSynchronize(s));
  float ms; P("elapsed", cudaEventElapsedTime(&ms, e0, e1));
  P("record e0 again", cudaEventRecord(e0, s));
  P("sync", cudaStreamSynchronize(s));
  std::thread t([&] {
    cudaSetDevice(0);
    k<<<1, 32, 0, s>>>(p);
    P("[thread] launch", cudaGetLastError());
    cudaEvent_t te; cudaEventCreateWithFlags(&te, cudaEventDisableTiming);
    P("[thread] record", cudaEventRecord(te, s));
    P("[thread] sync", cudaStreamSynchronize(s));
  });
  t.join();
  P("main record e0 after thread", cudaEventRecord(e0, s));
  P("main sync", cudaStreamSynchronize(s));
  std::thread t2([&] { cudaSetDevice(0); });
  t2.join();
  P("main record after 2nd thread exit", cudaEventRecord(e0, s));
  return 0;
}
