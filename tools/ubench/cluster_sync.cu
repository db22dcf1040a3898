// Microbenchmark: per-step cost of the cluster engine's synchronisation pattern
// (syncthreads + mbarrier phase wait + st.async halo push), no stencil work.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_04070_b200/csrc/dufwi_cluster_kernels.cuh"
using namespace dufwi;

template <int MODE>  // 0: syncthreads only, 1: + mbarrier/st.async halo, 2: cluster barrier per step
__global__ void __launch_bounds__(512, 1) k(int steps, int nz, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* X = reinterpret_cast<double*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * 4096 * 8);
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  const int rank = (int)cg::this_cluster().block_rank();
  const int cs = (int)cg::this_cluster().num_blocks();
  if (threadIdx.x == 0) { mbar_init(bar[0], 1); mbar_init(bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cluster_sync_all();
  const bool up = rank > 0, dn = rank + 1 < cs;
  const uint32_t txb = (uint32_t)((up ? 1 : 0) + (dn ? 1 : 0)) * nz * 8;
  double v = threadIdx.x;
  for (int t = 0; t < steps; ++t) {
    if (MODE == 2) { cluster_sync_all(); continue; }
    __syncthreads();
    if (MODE == 1) {
      if (t >= 1 && (up || dn)) mbar_wait(bar[(t - 1) & 1], ((t - 1) >> 1) & 1);
      if (threadIdx.x == 0 && (up || dn)) mbar_expect_tx(bar[t & 1], txb);
      double* Xw = X + (t & 1) * 4096;
      v = v * 1.0000001 + X[((t + 1) & 1) * 4096 + (threadIdx.x % nz)];
      if (threadIdx.x < nz) {
        if (up) push_async(mapa_rank(smem_addr(Xw + threadIdx.x), rank - 1), v, mapa_rank(bar[t & 1], rank - 1));
        if (dn) push_async(mapa_rank(smem_addr(Xw + 2048 + threadIdx.x), rank + 1), v, mapa_rank(bar[t & 1], rank + 1));
      }
    }
  }
  if (MODE == 1 && (up || dn)) mbar_wait(bar[(steps - 1) & 1], ((steps - 1) >> 1) & 1);
  cluster_sync_all();
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

template <int MODE>
float run(int steps, int nclusters) {
  double* out; cudaMalloc(&out, 4096 * 8);
  size_t smem = 2 * 4096 * 8 + 64;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(16 * nclusters); cfg.blockDim = dim3(480); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 16; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k<MODE>, steps, 160, out);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<MODE>, steps, 160, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError(); if (err) printf("err %s\n", cudaGetErrorString(err));
  cudaFree(out);
  return ms;
}

int main() {
  for (int nc : {1, 8}) {
    printf("clusters=%d  syncthreads only: %.3f us/step\n", nc, run<0>(10000, nc) * 1e3 / 10000);
    printf("clusters=%d  + mbarrier/st.async halo: %.3f us/step\n", nc, run<1>(10000, nc) * 1e3 / 10000);
    printf("clusters=%d  cluster barrier: %.3f us/step\n", nc, run<2>(10000, nc) * 1e3 / 10000);
  }
  return 0;
}
