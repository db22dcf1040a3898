// Shared device-side types and helpers for the DUFWI sm_100a kernels.
//
// Arithmetic model: wavefields are stored in f32 in HBM, every
// per-cell update is evaluated in f64 registers from the f32 inputs and rounded
// once when stored.  The cluster engine and the first-generation stepwise
// kernels read f64 coefficients (E/dx^2, dE/dc, density); the lean stepwise
// kernels stream f32 copies of E/dx^2, rho E/dx^2 and 1/rho (Model::Edf/Erf/qf,
// half the bytes) and widen them to f64 before the arithmetic.  Damping
// profiles, (A, B) tables and the pulse are f64 everywhere.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dufwi {

// Undamped-box + slot tables, shared by all units of a plan.
struct Geo {
  int nx, nz, nt;
  int S, R, M, B;
  int x_lo, x_hi, z_lo, z_hi;  // inclusive undamped box (strip mode)
  int Lx, Lz, SL;              // box extents and ring length per step (2Lz + 2Lx)
  double dt;
  const double* px;            // [nx] separable damping, or nullptr
  const double* pz;            // [nz]
  const double* d2d;           // [nx][nz] general damping if px == nullptr
  const double* pulse;         // [nt]
  const int* tx;               // [S][2]
  const int* node_slot;        // [nx][nz] receiver-node slot or -1
  const unsigned char* row_flag;  // [nx] 1 if the row holds any slot
  const unsigned char* col_flag;  // [nz] 1 if the column holds any slot
};

// Per-phantom coefficient arrays.
struct Model {
  const double* Ed;    // [B][nx][nz]  c^2 dt^2 / (1 + D dt) / dx^2
  const double* rho;   // [B][nx][nz]  density or nullptr
  const double* q;     // [B][nx][nz]  1/rho
  // density operator tables of the lean stepwise kernels (dufwi_lean_kernels.cuh)
  const double* Er;    // [B][nx][nz]    rho E / dx^2
  const double* fxe;   // [B][nx+1][nz]  x faces (q_{x-1} + q_x)/2; rows 0 and nx: outer = own q
  const double* fz;    // [B][nx][nz]    z faces (q_z + q_{z+1})/2; z = nz-1: outer = own q
  const double* fz0;   // [B][nx]        outer z face left of z = 0: q(x, 0)
  // f32 copies streamed by the lean kernels (arithmetic stays f64): Ed, Er, q
  const float* Edf;
  const float* Erf;
  const float* qf;
};

__device__ __forceinline__ double damping_at(const Geo& g, int x, int z) {
  return g.px ? fmax(__ldg(g.px + x), __ldg(g.pz + z)) : __ldg(g.d2d + (size_t)x * g.nz + z);
}

// A, B of the damped update (forward.py:226-234); exactly (2, -1) where D == 0.
__device__ __forceinline__ void ab_coeffs(double D, double dt, double& A, double& Bc) {
  if (D == 0.0) {
    A = 2.0;
    Bc = -1.0;
    return;
  }
  const double ddt = D * dt;
  const double den = 1.0 + ddt;
  A = (2.0 - ddt * ddt) / den;
  Bc = (ddt - 1.0) / den;
}

// Face weights of the variable-density operator at cell (x,z) of phantom
// arrays rho/q (oracle/dufwi_oracle.py rho_face_weights): w_j = rho_c (q_c + q_j)/2,
// outer faces use q_j := q_c.
struct RhoW {
  double xm, xp, zm, zp, W;
};

__device__ __forceinline__ RhoW rho_weights(const double* rho, const double* q, int nx, int nz,
                                            int x, int z) {
  const size_t c = (size_t)x * nz + z;
  const double rc = __ldg(rho + c), qc = __ldg(q + c);
  const double qxm = x > 0 ? __ldg(q + c - nz) : qc;
  const double qxp = x < nx - 1 ? __ldg(q + c + nz) : qc;
  const double qzm = z > 0 ? __ldg(q + c - 1) : qc;
  const double qzp = z < nz - 1 ? __ldg(q + c + 1) : qc;
  RhoW w;
  w.xm = rc * (0.5 * (qc + qxm));
  w.xp = rc * (0.5 * (qc + qxp));
  w.zm = rc * (0.5 * (qc + qzm));
  w.zp = rc * (0.5 * (qc + qzp));
  w.W = ((w.xm + w.xp) + w.zm) + w.zp;
  return w;
}

// Weight of the face (j -> c) as seen from neighbour j: rho_j (q_j + q_c)/2.
__device__ __forceinline__ double rho_in_weight(const double* rho, const double* q, size_t c,
                                                size_t j) {
  return __ldg(rho + j) * (0.5 * (__ldg(q + j) + __ldg(q + c)));
}

// ------------------------------------------------------------ f64 arithmetic
// Explicit roundings, shared by the fast and the generic step so both produce
// the same bits: the reference's 5-point sum (((-4c + xm) + xp) + zm) + zp and
// the update A u1 + B u2 + E lap (forward.py:301-308).
__device__ __forceinline__ double lap5(double c, double xm, double xp, double zm, double zp) {
  return __dadd_rn(__dadd_rn(__dadd_rn(__fma_rn(-4.0, c, xm), xp), zm), zp);
}
__device__ __forceinline__ double fwd_update(double A, double B, double u1, double u2, double e,
                                             double lap) {
  return __fma_rn(e, lap, __fma_rn(A, u1, __dmul_rn(B, u2)));
}
// (A, B) = (2, -1): B u2 = -u2 exactly, so this equals fwd_update bit for bit.
__device__ __forceinline__ double fwd_update_free(double u1, double u2, double e, double lap) {
  return __fma_rn(e, lap, __fma_rn(2.0, u1, -u2));
}
// lam = (A lam1 + L^T(E lam1)) + B lam2 (adjoint.py:119-131)
__device__ __forceinline__ double adj_update(double A, double B, double l1, double l2,
                                             double adj) {
  return __fma_rn(B, l2, __fma_rn(A, l1, adj));
}
__device__ __forceinline__ double adj_update_free(double l1, double l2, double adj) {
  return __dadd_rn(__fma_rn(2.0, l1, adj), -l2);
}
// u[t-2] = 2 u[t-1] + E L u[t-1] - u[t] (+ source), the forward step solved backwards
__device__ __forceinline__ double recon(double ub, double ua, double e, double lapu) {
  return __dadd_rn(__fma_rn(e, lapu, 2.0 * ub), -ua);
}

}  // namespace dufwi
