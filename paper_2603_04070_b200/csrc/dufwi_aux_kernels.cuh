// Small per-sweep kernels: coefficients, receiver gather, residual/misfit,
// group reduction and gradient finalisation.  None of these is on the per-step
// critical path; each runs once per sweep.
#pragma once

#include "dufwi_common.cuh"

namespace dufwi {

// E/dx^2 and dE/dc per phantom (forward.py:226-234, adjoint.py:116-117), and
// q = 1/rho for the density operator.
__global__ void set_model_kernel(Geo g, const double* __restrict__ c, const double* __restrict__ rho,
                                 double* __restrict__ Ed, double* __restrict__ dEdc,
                                 double* __restrict__ rho_copy, double* __restrict__ q,
                                 float* __restrict__ Edf, float* __restrict__ qf,
                                 double inv_dx2_div, double dx2, size_t total) {
  const size_t N2 = (size_t)g.nx * g.nz;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t cell = i % N2;
    const int x = (int)(cell / g.nz), z = (int)(cell % g.nz);
    const double D = damping_at(g, x, z);
    const double den = 1.0 + D * g.dt;
    const double cv = c[i];
    const double E = cv * cv * g.dt * g.dt / den;
    Ed[i] = E / dx2;
    Edf[i] = (float)(E / dx2);
    dEdc[i] = 2.0 * cv * (g.dt * g.dt) / den;
    if (rho) {
      rho_copy[i] = rho[i];
      q[i] = 1.0 / rho[i];
      qf[i] = (float)(1.0 / rho[i]);
    }
  }
  (void)inv_dx2_div;
}

// Density tables of the lean kernels (see Model): Er = rho * Ed, face factors
// f = 0.5 * (q_c + q_j) as in the oracle's rho_face_weights, outer faces = own q.
__global__ void rho_faces_kernel(Geo g, int B, const double* __restrict__ Ed,
                                 const double* __restrict__ rho, const double* __restrict__ q,
                                 double* __restrict__ Er, double* __restrict__ fxe,
                                 double* __restrict__ fz, double* __restrict__ fz0,
                                 float* __restrict__ Erf) {
  const int nx = g.nx, nz = g.nz;
  const size_t N2 = (size_t)nx * nz, NE = N2 + nz;
  const size_t total = (size_t)B * NE;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / NE);
    const size_t e = i % NE;
    const int r = (int)(e / nz), z = (int)(e % nz);  // r in [0, nx]
    const double* qb = q + (size_t)b * N2;
    fxe[i] = r == 0 ? qb[z] : r == nx ? qb[(size_t)(nx - 1) * nz + z]
                                      : 0.5 * (qb[(size_t)(r - 1) * nz + z] + qb[(size_t)r * nz + z]);
    if (r < nx) {
      const size_t c = (size_t)b * N2 + (size_t)r * nz + z;
      Er[c] = rho[c] * Ed[c];
      Erf[c] = (float)(rho[c] * Ed[c]);
      fz[c] = z == nz - 1 ? q[c] : 0.5 * (q[c] + q[c + 1]);
      if (z == 0) fz0[(size_t)b * nx + r] = q[c];
    }
  }
}

// traces[lu][r][t] = rec[t][lu][slot(s, r)] — the (P,R,nt) ChannelData layout
// (grid.py:164-183).  Flags non-finite samples (forward.py:309-310).
__global__ void gather_traces_kernel(Geo g, int unit_begin, int U, const float* __restrict__ rec,
                                     const int* __restrict__ rx_slot, float* __restrict__ traces,
                                     int* __restrict__ flag) {
  const size_t total = (size_t)U * g.R * g.nt;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i % g.nt);
    const size_t rest = i / g.nt;
    const int r = (int)(rest % g.R);
    const int lu = (int)(rest / g.R);
    const int s = (unit_begin + lu) % g.S;
    const float v = rec[((size_t)t * U + lu) * g.M + rx_slot[s * g.R + r]];
    traces[i] = v;
    if (!isfinite(v)) *flag = 1;
  }
}

// kResidualSplit blocks per unit (blockIdx.x = part, blockIdx.y = unit): resid
// merged per receiver node into rres[t][lu][slot] (duplicates summed in
// receiver order, like np.add.at in adjoint.py:127) and per-part partial
// misfits sum((tr - obs)^2) (adjoint.py:113-114) from fixed-shape block
// reductions, summed in part order later — results do not depend on scheduling.
constexpr int kResidualSplit = 64;

template <int NT>
__global__ void __launch_bounds__(NT) residual_kernel(Geo g, int unit_begin, int U,
                                                      const float* __restrict__ traces,
                                                      const double* __restrict__ obs,
                                                      const int* __restrict__ rx_slot,
                                                      const int* __restrict__ rx_next,
                                                      const unsigned char* __restrict__ rx_head,
                                                      double* __restrict__ rres,
                                                      double* __restrict__ misfit_unit) {
  const int lu = blockIdx.y;
  const int s = (unit_begin + lu) % g.S;
  const size_t base = (size_t)lu * g.R * g.nt;
  const size_t n = (size_t)g.R * g.nt;
  const size_t per = (n + kResidualSplit - 1) / kResidualSplit;
  const size_t i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  double sq = 0.0;
  for (size_t i = i0 + threadIdx.x; i < i1; i += NT) {
    const int r = (int)(i / g.nt), t = (int)(i % g.nt);
    const double d = (double)traces[base + i] - obs[base + i];
    sq += d * d;
    if (rx_head[s * g.R + r]) {
      double v = 2.0 * d;
      for (int r2 = rx_next[s * g.R + r]; r2 >= 0; r2 = rx_next[s * g.R + r2]) {
        const size_t j = base + (size_t)r2 * g.nt + t;
        v += 2.0 * ((double)traces[j] - obs[j]);
      }
      rres[((size_t)t * U + lu) * g.M + rx_slot[s * g.R + r]] = v;
    }
  }
  __shared__ double red[NT];
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) misfit_unit[(size_t)lu * kResidualSplit + blockIdx.x] = red[0];
}

// misfit[b] += sum over the chunk's units of phantom b, in unit order.  One warp:
// lane l sums the parts of units l, l + 32, ... (part order, loads of different
// units in flight together), lane 0 then adds the unit sums in unit order — the
// same additions in the same order as a serial loop.
__global__ void misfit_sum_kernel(Geo g, int unit_begin, int U, const double* __restrict__ mu,
                                  double* __restrict__ misfit) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  __shared__ double unit_sum[32];
  for (int base = 0; base < U; base += 32) {
    const int lu = base + threadIdx.x;
    double m = 0.0;
    if (lu < U)
      for (int k = 0; k < kResidualSplit; ++k) m += mu[(size_t)lu * kResidualSplit + k];
    unit_sum[threadIdx.x] = m;
    __syncwarp();
    if (threadIdx.x == 0) {
      const int n = min(32, U - base);
      for (int j = 0; j < n; ++j) misfit[(unit_begin + base + j) / g.S] += unit_sum[j];
    }
    __syncwarp();
  }
}

// acc[b] += sum of acc_part[g] over phantom b's groups, in group order.  Group
// numbering follows shot_group(): `first` groups for the chunk's first phantom,
// then `gpp` per further phantom (empty tail groups hold zeros).
__global__ void reduce_groups_kernel(Geo g, int b0, int nb, int first, int gpp,
                                     const double* __restrict__ acc_part,
                                     double* __restrict__ acc, const double* __restrict__ scale) {
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t total = (size_t)nb * N2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int bl = (int)(i / N2);
    const size_t cell = i % N2;
    const int g0 = bl == 0 ? 0 : first + (bl - 1) * gpp;
    const int g1 = bl == 0 ? first : g0 + gpp;
    double sum = 0.0;
    for (int k = g0; k < g1; ++k) sum += acc_part[(size_t)k * N2 + cell];
    // scale: rho for the lean density kernels, whose imaging sums D(u) lam (L_rho = rho D)
    if (scale) sum = scale[(size_t)(b0 + bl) * N2 + cell] * sum;
    acc[(size_t)(b0 + bl) * N2 + cell] += sum;
  }
}

// grad = keep ? dE/dc * (acc / dx^2) : 0, keep = D == 0 and farther than guard
// from every element (adjoint.py:75-91, 133-137).
// (ex0..ez1: bounding box of the elements, so cells farther than guard from the
// box skip the element loop.)
__global__ void finalize_kernel(Geo g, const double* __restrict__ acc, const double* __restrict__ dEdc,
                                const int* __restrict__ elements, int n_el, int ex0, int ex1,
                                int ez0, int ez1, int apply_mask, int guard, double dx2,
                                double* __restrict__ grad, int* __restrict__ flag) {
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t total = (size_t)g.B * N2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t cell = i % N2;
    const int x = (int)(cell / g.nz), z = (int)(cell % g.nz);
    const double a = acc[i];
    if (!isfinite(a)) *flag = 1;
    bool keep = true;
    if (apply_mask) {
      keep = damping_at(g, x, z) == 0.0;
      const long g2 = (long)guard * guard;
      const bool near = x >= ex0 - guard && x <= ex1 + guard && z >= ez0 - guard && z <= ez1 + guard;
      for (int e = 0; e < n_el && keep && near; ++e) {
        const long ddx = x - elements[2 * e], ddz = z - elements[2 * e + 1];
        if (ddx * ddx + ddz * ddz <= g2) keep = false;
      }
    }
    grad[i] = keep ? dEdc[i] * (a / dx2) : 0.0;
  }
}

}  // namespace dufwi
