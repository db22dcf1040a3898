// Microbenchmark: DRAM bandwidth of the stepwise engine's access pattern (a warp
// streams TX rows of a 128-wide z strip: 2 float4 reads + 1 float4 write per
// lane per row) against a flat copy of the same bytes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void strip_kernel(const float* __restrict__ a, const float* __restrict__ b, float* c,
                             int nx, int nz, int TX, int W) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int zw = 128 * W;  // z cells per warp
  const int z0 = blockIdx.x * zw;
  const int x0 = (blockIdx.y * 4 + warp) * TX;
  const size_t fo = (size_t)blockIdx.z * nx * nz;
  for (int x = x0; x < min(nx, x0 + TX); ++x) {
    for (int w = 0; w < W; ++w) {
      const int z = z0 + 128 * w + 4 * lane;
      if (z >= nz) continue;
      const size_t o = fo + (size_t)x * nz + z;
      const float4 p = __ldg(reinterpret_cast<const float4*>(a + o));
      const float4 q = __ldg(reinterpret_cast<const float4*>(b + o));
      *reinterpret_cast<float4*>(c + o) = make_float4(p.x + q.x, p.y + q.y, p.z + q.z, p.w + q.w);
    }
  }
}
__global__ void flat_kernel(const float4* __restrict__ a, const float4* __restrict__ b, float4* c, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 p = a[i], q = b[i];
    c[i] = make_float4(p.x + q.x, p.y + q.y, p.z + q.z, p.w + q.w);
  }
}
int main() {
  const int nx = 1088, nz = 1088, U = 64;
  const size_t n = (size_t)U * nx * nz;
  float *a, *b, *c;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4);
  cudaMemset(a, 0, n * 4); cudaMemset(b, 0, n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  flat_kernel<<<148 * 8, 256>>>((float4*)a, (float4*)b, (float4*)c, n / 4);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) flat_kernel<<<148 * 8, 256>>>((float4*)a, (float4*)b, (float4*)c, n / 4);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("flat: %.0f GB/s\n", 12.0 * n * 5 / (ms * 1e-3) / 1e9);
  for (int W : {1, 2, 4})
    for (int TX : {4, 8, 16, 32}) {
      dim3 grid((nz + 128 * W - 1) / (128 * W), (nx + 4 * TX - 1) / (4 * TX), U);
      strip_kernel<<<grid, 128>>>(a, b, c, nx, nz, TX, W);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) strip_kernel<<<grid, 128>>>(a, b, c, nx, nz, TX, W);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("strip W=%d (z per warp %d) TX=%2d: %.0f GB/s\n", W, 128 * W, TX, 12.0 * n * 5 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
