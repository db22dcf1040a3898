// Stepwise engine: one launch per time step over every unit of a chunk.
//
// Used for grids whose per-unit state does not fit a thread-block cluster's
// shared memory (configs 2-4).  Each launch is HBM-bound: per forward cell
// update it reads u[t-1] (neighbours come from L1/L2), u[t-2], writes u[t]
// = 12 B of DRAM traffic + the per-phantom coefficient (L2-resident, shared by
// all shots of the phantom).
//
// Reference semantics: forward.py:273-313 (update -> inject -> sample -> store)
// and adjoint.py:119-131 (update -> add.at residual -> imaging for t >= 1).
#pragma once

#include "dufwi_common.cuh"

namespace dufwi {

constexpr int kTileZ = 32;  // threads along z (contiguous axis): one warp per row
constexpr int kTileX = 8;   // rows per CTA

__device__ __forceinline__ double ld_or0(const float* p, size_t i, bool ok) {
  return ok ? (double)__ldg(p + i) : 0.0;
}

// ---------------------------------------------------------------------------
// forward step.  MODE 0: no history (uo aliases u2), 1: full history (uo is
// hist[t]), 2: strips (uo aliases u2, ring cells also written to strip_t).
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kTileZ* kTileX)
    fwd_step_kernel(Geo g, Model m, int t, int unit_begin, const float* __restrict__ u1,
                    const float* u2, float* uo, float* __restrict__ rec_t,
                    float* __restrict__ strip_t, int has1, int has2) {
  const int z = blockIdx.x * kTileZ + threadIdx.x;
  const int x = blockIdx.y * kTileX + threadIdx.y;
  if (x >= g.nx || z >= g.nz) return;
  const int lu = blockIdx.z;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t c = (size_t)x * g.nz + z;
  const size_t pb = (size_t)b * N2;

  double uc = 0.0, lap = 0.0;
  if (has1) {
    const float* f = u1 + (size_t)lu * N2;
    uc = (double)__ldg(f + c);
    const double xm = ld_or0(f, c - g.nz, x > 0);
    const double xp = ld_or0(f, c + g.nz, x < g.nx - 1);
    const double zm = ld_or0(f, c - 1, z > 0);
    const double zp = ld_or0(f, c + 1, z < g.nz - 1);
    if (RHO) {
      const RhoW w = rho_weights(m.rho + pb, m.q + pb, g.nx, g.nz, x, z);
      lap = (((-w.W * uc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp;
    } else {
      lap = (((-4.0 * uc + xm) + xp) + zm) + zp;
    }
  }
  const double u2c = has2 ? (double)u2[(size_t)lu * N2 + c] : 0.0;
  double A, Bc;
  ab_coeffs(damping_at(g, x, z), g.dt, A, Bc);
  double v = A * uc + Bc * u2c + __ldg(m.Ed + pb + c) * lap;
  if (x == __ldg(g.tx + 2 * s) && z == __ldg(g.tx + 2 * s + 1)) v += __ldg(g.pulse + t);
  const float vf = (float)v;
  uo[(size_t)lu * N2 + c] = vf;
  if (__ldg(g.row_flag + x)) {
    const int slot = __ldg(g.node_slot + c);
    if (slot >= 0) rec_t[(size_t)lu * g.M + slot] = vf;
  }
  if (MODE == 2) {
    float* st = strip_t + (size_t)lu * g.SL;
    if (z >= g.z_lo && z <= g.z_hi) {
      if (x == g.x_lo - 1) st[z - g.z_lo] = vf;
      if (x == g.x_hi + 1) st[g.Lz + z - g.z_lo] = vf;
    }
    if (x >= g.x_lo && x <= g.x_hi) {
      if (z == g.z_lo - 1) st[2 * g.Lz + x - g.x_lo] = vf;
      if (z == g.z_hi + 1) st[2 * g.Lz + g.Lx + x - g.x_lo] = vf;
    }
  }
}

// ---------------------------------------------------------------------------
// adjoint step over one shot group of one phantom (blockIdx.z = group id).
// lam[t] = A lam[t+1] + L^T(E lam[t+1]) + B lam[t+2] (+ merged residual at
// receiver nodes), written in place over lam[t+2].  Imaging for t >= 1:
// acc_part[group] += sum_shots L(u[t-1]) * lam[t]  (f64, fixed shot order).
// MODE 1: u[t-1] from the full history.  MODE 2: u[t-1] held in a buffer, its
// ring neighbours from strips[t-1]; the same kernel reconstructs u[t-2] =
// 2u[t-1] + E L u[t-1] + s[t] delta_tx - u[t] in place over u[t] (interior).
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kTileZ* kTileX)
    adj_step_kernel(Geo g, Model m, int t, int unit_begin, int U, int gs, int b0, int gpp,
                    const float* __restrict__ l1, float* l2o, const float* __restrict__ F,
                    float* ut, const float* __restrict__ utm1,
                    const float* __restrict__ strip_tm1, const double* __restrict__ rres_t,
                    double* __restrict__ acc_part, int has1, int has2, int do_img, int do_recon) {
  const int z = blockIdx.x * kTileZ + threadIdx.x;
  const int x = blockIdx.y * kTileX + threadIdx.y;
  if (x >= g.nx || z >= g.nz) return;
  const int gid = blockIdx.z;
  const int b = b0 + gid / gpp;
  const int s_first = (gid % gpp) * gs;
  const int u_first = max(b * g.S + s_first, unit_begin);
  const int u_last = min(b * g.S + min(s_first + gs, g.S), unit_begin + U);
  if (u_first >= u_last) return;

  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t c = (size_t)x * g.nz + z;
  const size_t pb = (size_t)b * N2;
  const bool okxm = x > 0, okxp = x < g.nx - 1, okzm = z > 0, okzp = z < g.nz - 1;

  // Per-phantom coefficients, hoisted out of the shot loop.
  double A, Bc;
  ab_coeffs(damping_at(g, x, z), g.dt, A, Bc);
  const double* Ed = m.Ed + pb;
  const double Ec = __ldg(Ed + c);
  // incoming weights (neighbour j -> c) times E_j for the transposed operator
  double kc, kxm = 0.0, kxp = 0.0, kzm = 0.0, kzp = 0.0;
  RhoW w{1.0, 1.0, 1.0, 1.0, 4.0};
  if (RHO) {
    const double* rho = m.rho + pb;
    const double* q = m.q + pb;
    w = rho_weights(rho, q, g.nx, g.nz, x, z);
    kc = -w.W * Ec;
    if (okxm) kxm = rho_in_weight(rho, q, c, c - g.nz) * __ldg(Ed + c - g.nz);
    if (okxp) kxp = rho_in_weight(rho, q, c, c + g.nz) * __ldg(Ed + c + g.nz);
    if (okzm) kzm = rho_in_weight(rho, q, c, c - 1) * __ldg(Ed + c - 1);
    if (okzp) kzp = rho_in_weight(rho, q, c, c + 1) * __ldg(Ed + c + 1);
  } else {
    kc = -4.0 * Ec;
    if (okxm) kxm = __ldg(Ed + c - g.nz);
    if (okxp) kxp = __ldg(Ed + c + g.nz);
    if (okzm) kzm = __ldg(Ed + c - 1);
    if (okzp) kzp = __ldg(Ed + c + 1);
  }
  const int slot = __ldg(g.row_flag + x) ? __ldg(g.node_slot + c) : -1;
  const bool interior =
      MODE == 2 ? (x >= g.x_lo && x <= g.x_hi && z >= g.z_lo && z <= g.z_hi) : true;
  const bool img = do_img && interior;
  const double pulse_t = __ldg(g.pulse + t);

  double local = 0.0;
  for (int u = u_first; u < u_last; ++u) {
    const int lu = u - unit_begin;
    const size_t fo = (size_t)lu * N2;
    double lam = 0.0;
    if (has1) {
      const float* L = l1 + fo;
      const double lc = (double)__ldg(L + c);
      // L^T(E lam1): reference order (-4 (E lam)_c + x-1 + x+1 + z-1 + z+1) / dx^2
      const double adj = RHO ? ((((kc * lc + kxm * ld_or0(L, c - g.nz, okxm)) +
                                  kxp * ld_or0(L, c + g.nz, okxp)) +
                                 kzm * ld_or0(L, c - 1, okzm)) +
                                kzp * ld_or0(L, c + 1, okzp))
                             : ((((kc * lc + kxm * ld_or0(L, c - g.nz, okxm)) +
                                  kxp * ld_or0(L, c + g.nz, okxp)) +
                                 kzm * ld_or0(L, c - 1, okzm)) +
                                kzp * ld_or0(L, c + 1, okzp));
      lam = A * lc + adj;
    }
    if (has2) lam += Bc * (double)l2o[fo + c];
    if (slot >= 0) lam += __ldg(rres_t + (size_t)lu * g.M + slot);
    l2o[fo + c] = (float)lam;

    if (img) {
      double lapu;
      if (MODE == 1) {
        const float* f = F + fo;
        const double fc = (double)__ldg(f + c);
        const double xm = ld_or0(f, c - g.nz, okxm), xp = ld_or0(f, c + g.nz, okxp);
        const double zm = ld_or0(f, c - 1, okzm), zp = ld_or0(f, c + 1, okzp);
        lapu = RHO ? ((((-w.W * fc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp)
                   : ((((-4.0 * fc + xm) + xp) + zm) + zp);
      } else {
        // u[t-1]: interior cells from the buffer, ring cells from strips[t-1]
        const float* f = utm1 + fo;
        const float* st = strip_tm1 + (size_t)lu * g.SL;
        const double fc = (double)f[c];
        const double xm = x > g.x_lo ? (double)f[c - g.nz]
                                     : (x > 0 ? (double)__ldg(st + z - g.z_lo) : 0.0);
        const double xp = x < g.x_hi ? (double)f[c + g.nz]
                                     : (x < g.nx - 1 ? (double)__ldg(st + g.Lz + z - g.z_lo) : 0.0);
        const double zm = z > g.z_lo ? (double)f[c - 1]
                                     : (z > 0 ? (double)__ldg(st + 2 * g.Lz + x - g.x_lo) : 0.0);
        const double zp = z < g.z_hi ? (double)f[c + 1]
                                     : (z < g.nz - 1 ? (double)__ldg(st + 2 * g.Lz + g.Lx + x - g.x_lo) : 0.0);
        lapu = RHO ? ((((-w.W * fc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp)
                   : ((((-4.0 * fc + xm) + xp) + zm) + zp);
        if (do_recon) {
          const int s = u - b * g.S;
          double prev = 2.0 * fc + Ec * lapu - (double)ut[fo + c];
          if (x == __ldg(g.tx + 2 * s) && z == __ldg(g.tx + 2 * s + 1)) prev += pulse_t;
          ut[fo + c] = (float)prev;
        }
      }
      local += lapu * lam;
    }
  }
  if (img) acc_part[(size_t)gid * N2 + c] += local;
}

}  // namespace dufwi
