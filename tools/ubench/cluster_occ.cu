// How many clusters of size cs can be co-resident (one CTA per SM)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k(int* p) { if (p) p[blockIdx.x] = 1; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d\n", pr.multiProcessorCount);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs * 16); cfg.blockDim = dim3(480); cfg.dynamicSmemBytes = 100000;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cs %2d: max active clusters %d (%d SMs) %s\n", cs, n, n * cs, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
