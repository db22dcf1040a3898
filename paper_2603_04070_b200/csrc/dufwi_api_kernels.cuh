// Field utilities of the public forward API: the reference's `laplacian`
// (forward.py:211-223) and `step_wavefield` (forward.py:237-253) on float64
// fields, one thread per cell.  Every multiply and add is an explicitly rounded
// f64 operation in the reference's order (no FMA contraction), so the results
// are bit-identical to NumPy's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dufwi {

// out = -4u; out += u[x-1]; out += u[x+1]; out += u[z-1]; out += u[z+1]; out /= dx*dx
__device__ __forceinline__ double lap5_ref(const double* __restrict__ u, int nx, int nz, int x,
                                           int z, double dx2) {
  const size_t c = (size_t)x * nz + z;
  double acc = __dmul_rn(-4.0, u[c]);
  if (x > 0) acc = __dadd_rn(acc, u[c - nz]);
  if (x < nx - 1) acc = __dadd_rn(acc, u[c + nz]);
  if (z > 0) acc = __dadd_rn(acc, u[c - 1]);
  if (z < nz - 1) acc = __dadd_rn(acc, u[c + 1]);
  return __ddiv_rn(acc, dx2);
}

__global__ void laplacian_f64_kernel(const double* __restrict__ u, long long batch, int nx, int nz,
                                     double dx2, double* __restrict__ out) {
  const long long n = (long long)nx * nz, total = batch * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / n, k = i - b * n;
    const int x = (int)(k / nz), z = (int)(k - (long long)x * nz);
    out[i] = lap5_ref(u + b * n, nx, nz, x, z, dx2);
  }
}

// step_coefficients (forward.py:226-234) and the update of step_wavefield:
// out = ((a u1 + b u2) + e lap(u1)) + s
__global__ void step_field_f64_kernel(const double* __restrict__ u1, const double* __restrict__ u2,
                                      const double* __restrict__ c, const double* __restrict__ d,
                                      const double* __restrict__ s, int nx, int nz, double dx2,
                                      double dt, double* __restrict__ out) {
  const long long n = (long long)nx * nz;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i / nz), z = (int)(i - (long long)x * nz);
    const double ddt = __dmul_rn(d[i], dt);
    const double den = __dadd_rn(1.0, ddt);
    const double a = __ddiv_rn(__dsub_rn(2.0, __dmul_rn(ddt, ddt)), den);
    const double b = __ddiv_rn(__dsub_rn(ddt, 1.0), den);
    const double e = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(c[i], c[i]), dt), dt), den);
    const double lap = lap5_ref(u1, nx, nz, x, z, dx2);
    const double v = __dadd_rn(__dadd_rn(__dmul_rn(a, u1[i]), __dmul_rn(b, u2[i])),
                               __dmul_rn(e, lap));
    out[i] = __dadd_rn(v, s[i]);
  }
}

}  // namespace dufwi
