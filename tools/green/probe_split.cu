// Probe: sequential SM splits on B200.  Dev tool.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  cudaSetDevice(0); cudaFree(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUdevResource all; cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  unsigned counts[] = {96, 48, 64, 32, 16, 8, 74, 100, 104};
  for (unsigned c : counts) {
    CUdevResource g, rest; unsigned n = 1;
    CUresult r = cuDevSmResourceSplitByCount(&g, &n, &all, &rest, 0, c);
    printf("split %u from all: r=%d n=%u group=%u rest=%u\n", c, (int)r, n, r ? 0 : g.sm.smCount, r ? 0 : rest.sm.smCount);
    if (r == 0) {
      CUdevResource g2, rest2; unsigned n2 = 1;
      CUresult r2 = cuDevSmResourceSplitByCount(&g2, &n2, &rest, &rest2, 0, 16);
      printf("   then 16 from rest: r=%d n=%u group=%u rest=%u\n", (int)r2, n2, r2 ? 0 : g2.sm.smCount, r2 ? 0 : rest2.sm.smCount);
      CUdevResource g3; unsigned n3 = 1;
      CUresult r3 = cuDevSmResourceSplitByCount(&g3, &n3, &rest, nullptr, 0, rest.sm.smCount);
      printf("   whole rest: r=%d n=%u group=%u\n", (int)r3, n3, r3 ? 0 : g3.sm.smCount);
    }
  }
  return 0;
}
