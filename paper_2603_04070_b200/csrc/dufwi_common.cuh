// Shared device-side types and helpers for the DUFWI sm_100a kernels.
//
// Arithmetic model: wavefields are stored in f32 in HBM.  The
// default sweep kernels (cluster engine with T = float, dufwi_tile_kernels.cuh)
// evaluate every update in f32 in the increment form defined below, which has
// the error of "f64 arithmetic, f32 storage"; imaging sums are folded into f64.
// DUFWI_ARITH_F64 plans (cluster engine with T = double, the lean / vec / stream
// stepwise kernels) evaluate every update in f64 registers in the reference's
// operation order and round once when storing; they read f64 coefficients
// (E/dx^2, dE/dc, density) or, the lean kernels, f32 copies widened to f64.
// Damping profiles and the pulse are f64 on the device; the f32 kernels use
// pairs / tables rounded once from f64.
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

// ------------------------------------------------------------ f32 arithmetic
// Increment form of the same updates, evaluated entirely in f32 (the sweep
// kernels' arithmetic).  The reference's u[t] = A u1 + B u2 + E L(u1) is
// rewritten as
//   u[t] = u1 + ((u1 - u2) + (A - 2) u1 + (B + 1) u2 + E L(u1)),
//   L(u1) = ((xm - c) + (xp - c)) + ((zm - c) + (zp - c)).
// Neighbouring values of a resolved wavefield are close, so the differences are
// (nearly) exact, the increment is ~ omega dt = 0.13 of |u|, and the only
// rounding at the scale of |u| is the final add — the one rounding that f32
// storage of the field costs anyway.  Measured against the f64 reference this
// form has the error of "f64 arithmetic, f32 storage" (config 0: traces 4.9e-7,
// fixed-observation gradient 5.4e-6; the naive f32 form A u1 + B u2 + E lap is
// 3x worse on traces); DESIGN.md section 4.0.  (a2, b1) = (A - 2, B + 1) are
// formed in f64 and rounded once; both are exactly 0 where D == 0.
__device__ __forceinline__ float lap5f(float c, float xm, float xp, float zm, float zp) {
  return __fadd_rn(__fadd_rn(__fsub_rn(xm, c), __fsub_rn(xp, c)),
                   __fadd_rn(__fsub_rn(zm, c), __fsub_rn(zp, c)));
}
// undamped cell: u1 + ((u1 - u2) + e lap)
__device__ __forceinline__ float inc_update_free(float u1, float u2, float e, float lap) {
  return __fadd_rn(u1, __fmaf_rn(e, lap, __fsub_rn(u1, u2)));
}
__device__ __forceinline__ float inc_update(float a2, float b1, float u1, float u2, float e,
                                            float lap) {
  const float d = __fadd_rn(__fsub_rn(u1, u2), __fmaf_rn(a2, u1, __fmul_rn(b1, u2)));
  return __fadd_rn(u1, __fmaf_rn(e, lap, d));
}
// lam = l1 + ((l1 - l2) + L(E l1)) (+ damping terms); adj = L(E l1)
__device__ __forceinline__ float inc_adj_free(float l1, float l2, float adj) {
  return __fadd_rn(l1, __fadd_rn(__fsub_rn(l1, l2), adj));
}
__device__ __forceinline__ float inc_adj(float a2, float b1, float l1, float l2, float adj) {
  const float d = __fadd_rn(__fsub_rn(l1, l2), __fmaf_rn(a2, l1, __fmul_rn(b1, l2)));
  return __fadd_rn(l1, __fadd_rn(d, adj));
}
// u[t-2] = u[t-1] + ((u[t-1] - u[t]) + E L u[t-1]) (+ source), undamped cells
__device__ __forceinline__ float inc_recon(float ub, float ua, float e, float lapu) {
  return __fadd_rn(ub, __fmaf_rn(e, lapu, __fsub_rn(ub, ua)));
}
// (A - 2, B + 1) of the damped update, rounded once from f64
__device__ __forceinline__ float2 ab_inc(double D, double dt) {
  double A, B;
  ab_coeffs(D, dt, A, B);
  return make_float2((float)(A - 2.0), (float)(B + 1.0));
}

// ------------------------------------------------- arithmetic by scalar type
// The cluster sweeps are written once over the scalar type T: float selects
// the f32 increment form above (DUFWI_ARITH_F32, the default), double the
// reference's operation order in f64 (DUFWI_ARITH_F64).  The per-cell
// damping pair is (A - 2, B + 1) for float and (A, B) for double.
template <class T> struct Pair;
template <> struct Pair<float> { typedef float2 type; };
template <> struct Pair<double> { typedef double2 type; };
template <class T> using pair_t = typename Pair<T>::type;

template <class T> __device__ __forceinline__ pair_t<T> ab_pair(double D, double dt);
template <> __device__ __forceinline__ float2 ab_pair<float>(double D, double dt) {
  return ab_inc(D, dt);
}
template <> __device__ __forceinline__ double2 ab_pair<double>(double D, double dt) {
  double A, B;
  ab_coeffs(D, dt, A, B);
  return make_double2(A, B);
}
// the pair of an undamped cell
template <class T> __device__ __forceinline__ pair_t<T> free_pair();
template <> __device__ __forceinline__ float2 free_pair<float>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ double2 free_pair<double>() { return make_double2(2.0, -1.0); }

__device__ __forceinline__ float mul_s(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_s(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_s(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_s(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float fma_s(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_s(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ float lap_s(float c, float xm, float xp, float zm, float zp) {
  return lap5f(c, xm, xp, zm, zp);
}
__device__ __forceinline__ double lap_s(double c, double xm, double xp, double zm, double zp) {
  return lap5(c, xm, xp, zm, zp);
}
__device__ __forceinline__ float step_free(float u1, float u2, float e, float lap) {
  return inc_update_free(u1, u2, e, lap);
}
__device__ __forceinline__ double step_free(double u1, double u2, double e, double lap) {
  return fwd_update_free(u1, u2, e, lap);
}
__device__ __forceinline__ float step_ab(float2 ab, float u1, float u2, float e, float lap) {
  return inc_update(ab.x, ab.y, u1, u2, e, lap);
}
__device__ __forceinline__ double step_ab(double2 ab, double u1, double u2, double e, double lap) {
  return fwd_update(ab.x, ab.y, u1, u2, e, lap);
}
__device__ __forceinline__ float adjs_free(float l1, float l2, float adj) {
  return inc_adj_free(l1, l2, adj);
}
__device__ __forceinline__ double adjs_free(double l1, double l2, double adj) {
  return adj_update_free(l1, l2, adj);
}
__device__ __forceinline__ float adjs_ab(float2 ab, float l1, float l2, float adj) {
  return inc_adj(ab.x, ab.y, l1, l2, adj);
}
__device__ __forceinline__ double adjs_ab(double2 ab, double l1, double l2, double adj) {
  return adj_update(ab.x, ab.y, l1, l2, adj);
}
__device__ __forceinline__ float recon_s(float ub, float ua, float e, float lapu) {
  return inc_recon(ub, ua, e, lapu);
}
__device__ __forceinline__ double recon_s(double ub, double ua, double e, double lapu) {
  return recon(ub, ua, e, lapu);
}

}  // namespace dufwi
