// Microbenchmark: dependent-chain latency and throughput of DADD / DFMA and F2F on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + b; x = x + b; x = x + b; x = x + b; }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void latfma(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void latf2f(double* out, float a, int n, long long* cyc) {
  float x = a; double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double d = (double)x; x = (float)(d * 1.0000001); }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void thr(double* out, double a, double b, int n) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
  long long h; int n = 10000;
  lat<<<1, 1>>>(out, 1.0, 1e-9, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  latfma<<<1, 1>>>(out, 1.0, 0.999, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  latf2f<<<1, 1>>>(out, 1.0f, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("F2F f32->f64->DMUL->f32 chain: %.2f cycles/iter\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  thr<<<148 * 4, 512>>>(out, 1.0, 0.999, 100);
  cudaEventRecord(e0); thr<<<148 * 4, 512>>>(out, 1.0, 0.999, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * iters * 148.0 * 4 * 512;
  printf("DFMA throughput: %.1f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", flops / ms / 1e9, flops / 2 / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}
