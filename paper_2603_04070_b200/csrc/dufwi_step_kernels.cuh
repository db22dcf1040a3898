// Stepwise engine: one launch per time step over every unit of a chunk.
//
// Used for grids whose per-unit state does not fit a thread-block cluster
// (configs 2-4).  Each launch is HBM-bound, so the kernels are shaped for
// memory-level parallelism and for reading every byte once:
//   * a warp owns a 32-lane z strip — lanes 1..30 compute, lanes 0 and 31 only
//     load the z halo — so each row access is one coalesced segment and the
//     z-neighbours come from warp shuffles of f64 registers;
//   * a thread computes RX consecutive x-rows for NS shots of one phantom and
//     issues ALL its loads (RX+2 rows of u[t-1], RX rows of u[t-2], per NS
//     shot) before any arithmetic, so ~20 independent loads are in flight per
//     thread; the 8 warps of a CTA stack along x so the x-halo rows a warp
//     re-reads were just loaded by its neighbour (L1 hits);
//   * per-phantom coefficients (E/dx^2, density) are loaded once per NS shots;
//     every f32 value is converted to f64 once.
// DRAM traffic per forward cell update: read u[t-1] and u[t-2], write u[t] = 12 B.
//
// Reference semantics: forward.py:273-313 (update -> inject -> sample -> store)
// and adjoint.py:119-131 (update -> add.at residual -> imaging for t >= 1).
#pragma once

#include "dufwi_common.cuh"

namespace dufwi {

constexpr int kStripZ = 30;  // computed z per warp
constexpr int kWarpsX = 8;   // warps per CTA, stacked along x
constexpr int kRXF = 4;      // x-rows per thread, forward
constexpr int kRXA = 2;      // x-rows per thread, adjoint (more live fields per row)
constexpr int kNSF = 2;      // shots per thread, forward
constexpr int kNSA = 1;      // shots per thread, adjoint

// (A, B) of cell (x, z) from 1-D tables: D = max(px, pz), so A(D) is the table
// entry of whichever axis ramp is larger (identical to ab_coeffs(max(px, pz))).
struct ABTables {
  const double *px, *pz, *Ax, *Bx, *Az, *Bz;  // separable damping
  const double *A2, *B2;                      // general damping map
};

__device__ __forceinline__ void ab_at(const ABTables& T, int x, double pzz, double Azz, double Bzz,
                                      size_t cell, double& A, double& B) {
  if (T.px) {
    const bool xs = __ldg(T.px + x) >= pzz;
    A = xs ? __ldg(T.Ax + x) : Azz;
    B = xs ? __ldg(T.Bx + x) : Bzz;
  } else {
    A = __ldg(T.A2 + cell);
    B = __ldg(T.B2 + cell);
  }
}

__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// Shot group gid of the chunk [unit_begin, unit_begin+U): up to gs shots of one
// phantom.  Groups are enumerated phantom by phantom over the chunk's actual
// units (the first and last phantom may be partial), so no group is empty
// except possibly the tail groups of a partial last phantom.
struct ShotGroup {
  int b, lu0, n;  // phantom, first chunk-local unit, count
};

__device__ __forceinline__ ShotGroup shot_group(const Geo& g, int gid, int unit_begin, int U,
                                                int gs) {
  ShotGroup sg;
  const int b0 = unit_begin / g.S;
  const int n_first = min(U, (b0 + 1) * g.S - unit_begin);
  const int gpp_first = (n_first + gs - 1) / gs;
  int b, start, end;
  if (gid < gpp_first) {
    b = b0;
    start = unit_begin + gid * gs;
    end = min(unit_begin + n_first, start + gs);
  } else {
    const int gpp = (g.S + gs - 1) / gs;
    const int k = gid - gpp_first;
    b = b0 + 1 + k / gpp;
    start = b * g.S + (k % gpp) * gs;
    end = min(min((b + 1) * g.S, unit_begin + U), start + gs);
  }
  sg.b = b;
  sg.lu0 = start - unit_begin;
  sg.n = max(0, end - start);
  return sg;
}

// Density weights of one cell: outgoing w_{c->j} = rho_c (q_c + q_j)/2 and
// incoming w_{j->c} = rho_j (q_j + q_c)/2 (oracle rho_face_weights / lap_rho_T).
struct RhoW2 {
  double wxm, wxp, wzm, wzp, W, ixm, ixp, izm, izp;
};

__device__ __forceinline__ RhoW2 rho_w2(double rc, double qc, double rm, double qm, double rp,
                                        double qp, double rzm, double qzm, double rzp, double qzp,
                                        bool okxm, bool okxp, bool okzm, bool okzp) {
  RhoW2 r;
  r.wxm = rc * (0.5 * (qc + (okxm ? qm : qc)));
  r.wxp = rc * (0.5 * (qc + (okxp ? qp : qc)));
  r.wzm = rc * (0.5 * (qc + (okzm ? qzm : qc)));
  r.wzp = rc * (0.5 * (qc + (okzp ? qzp : qc)));
  r.W = ((r.wxm + r.wxp) + r.wzm) + r.wzp;
  r.ixm = okxm ? rm * (0.5 * (qm + qc)) : 0.0;
  r.ixp = okxp ? rp * (0.5 * (qp + qc)) : 0.0;
  r.izm = okzm ? rzm * (0.5 * (qzm + qc)) : 0.0;
  r.izp = okzp ? rzp * (0.5 * (qzp + qc)) : 0.0;
  return r;
}

// Thread geometry shared by both kernels.
struct Lane {
  int lane, z, x0;  // z of this lane; first of the thread's RX rows
  bool zin, comp;   // inside the grid / computes (lanes 1..30 inside the grid)
};

__device__ __forceinline__ Lane lane_geo(const Geo& g, int rx) {
  Lane L;
  L.lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  L.z = blockIdx.x * kStripZ - 1 + L.lane;
  L.x0 = (blockIdx.y * kWarpsX + warp) * rx;
  L.zin = L.z >= 0 && L.z < g.nz;
  L.comp = L.zin && L.lane >= 1 && L.lane <= kStripZ;
  return L;
}

// ---------------------------------------------------------------------------
// forward step.  MODE 0: no history (uo aliases u2), 1: full history (uo is
// hist[t]), 2: strips (uo aliases u2; ring cells also written to strip_t).
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kWarpsX * 32)
    fwd_stream_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int U, int gs,
                      const float* __restrict__ u1, const float* u2, float* uo,
                      float* __restrict__ rec_t, float* __restrict__ strip_t, int has1, int has2) {
  const Lane L = lane_geo(g, kRXF);
  if (L.x0 >= g.nx) return;  // warp-uniform
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  const int nz = g.nz;
  const size_t N2 = (size_t)g.nx * nz;
  const size_t pb = (size_t)sg.b * N2;
  const int zc = L.zin ? L.z : 0;

  // ---- all loads first
  double u[kNSF][kRXF + 2], w2[kNSF][kRXF];
#pragma unroll
  for (int k = 0; k < kNSF; ++k) {
    const bool ak = k < sg.n;
    const size_t fo = (size_t)(sg.lu0 + (ak ? k : 0)) * N2;
#pragma unroll
    for (int r = 0; r < kRXF + 2; ++r) {
      const int x = L.x0 - 1 + r;
      u[k][r] = (has1 && ak && L.zin && x >= 0 && x < g.nx) ? (double)__ldg(u1 + fo + (size_t)x * nz + zc) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kRXF; ++r) {
      const int x = L.x0 + r;
      w2[k][r] = (has2 && ak && L.comp && x < g.nx) ? (double)u2[fo + (size_t)x * nz + L.z] : 0.0;
    }
  }
  double ed[kRXF];
#pragma unroll
  for (int r = 0; r < kRXF; ++r) {
    const int x = L.x0 + r;
    ed[r] = (L.comp && x < g.nx) ? __ldg(m.Ed + pb + (size_t)x * nz + L.z) : 0.0;
  }
  double qv[kRXF + 2], rv[kRXF + 2];
  if (RHO) {
#pragma unroll
    for (int r = 0; r < kRXF + 2; ++r) {
      const int x = L.x0 - 1 + r;
      const bool ok = L.zin && x >= 0 && x < g.nx;
      qv[r] = ok ? __ldg(m.q + pb + (size_t)x * nz + zc) : 0.0;
      rv[r] = ok ? __ldg(m.rho + pb + (size_t)x * nz + zc) : 0.0;
    }
  }
  double pzz = 0.0, Azz = 2.0, Bzz = -1.0;
  if (T.px && L.zin) { pzz = __ldg(T.pz + L.z); Azz = __ldg(T.Az + L.z); Bzz = __ldg(T.Bz + L.z); }
  const double pulse_t = __ldg(g.pulse + t);
  int txr[kNSF];
#pragma unroll
  for (int k = 0; k < kNSF; ++k) {
    const int s = (unit_begin + sg.lu0 + (k < sg.n ? k : 0)) % g.S;
    txr[k] = (k < sg.n && __ldg(g.tx + 2 * s + 1) == L.z) ? __ldg(g.tx + 2 * s) - L.x0 : -1;
  }

  // ---- compute and store
#pragma unroll
  for (int r = 0; r < kRXF; ++r) {
    const int x = L.x0 + r;
    const size_t cell = (size_t)x * nz + L.z;
    double A, B;
    ab_at(T, min(x, g.nx - 1), pzz, Azz, Bzz, (size_t)min(x, g.nx - 1) * nz + zc, A, B);
    RhoW2 w{};
    if (RHO) {
      const double qzm = shfl_up1(qv[r + 1]), qzp = shfl_dn1(qv[r + 1]);
      const double rzm = shfl_up1(rv[r + 1]), rzp = shfl_dn1(rv[r + 1]);
      w = rho_w2(rv[r + 1], qv[r + 1], rv[r], qv[r], rv[r + 2], qv[r + 2], rzm, qzm, rzp, qzp,
                 x > 0, x + 1 < g.nx, L.z > 0, L.z < nz - 1);
    }
    int slot = -1;
    if (L.comp && x < g.nx && __ldg(g.row_flag + x)) slot = __ldg(g.node_slot + cell);
#pragma unroll
    for (int k = 0; k < kNSF; ++k) {
      const double c0 = u[k][r + 1];
      const double zm = shfl_up1(c0), zp = shfl_dn1(c0);
      const double lap = RHO ? ((((-w.W * c0 + w.wxm * u[k][r]) + w.wxp * u[k][r + 2]) + w.wzm * zm) + w.wzp * zp)
                             : ((((-4.0 * c0 + u[k][r]) + u[k][r + 2]) + zm) + zp);
      double v = A * c0 + B * w2[k][r] + ed[r] * lap;
      if (txr[k] == r) v += pulse_t;
      if (L.comp && x < g.nx && k < sg.n) {
        const int lu = sg.lu0 + k;
        const float vf = (float)v;
        uo[(size_t)lu * N2 + cell] = vf;
        if (slot >= 0) rec_t[(size_t)lu * g.M + slot] = vf;
        if (MODE == 2) {
          float* st = strip_t + (size_t)lu * g.SL;
          const int z = L.z;
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
    }
  }
}

// ---------------------------------------------------------------------------
// adjoint step over one shot group of one phantom (blockIdx.z = group id); a
// thread walks the group's shots kNSA at a time, sums the imaging term of all
// of them in registers, then does one read-modify-write of acc_part[group].
// lam[t] = A lam[t+1] + L^T(E lam[t+1]) + B lam[t+2] (+ merged residual),
// written in place over lam[t+2].  Imaging for t >= 1 with L(u[t-1]):
// MODE 1 from the full history, MODE 2 from the buffer u[t-1] (ring cells from
// strips[t-1]) while reconstructing u[t-2] = 2u[t-1] + E L u[t-1] + s[t] d_tx
// - u[t] in place over u[t] on the undamped box.
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kWarpsX * 32)
    adj_stream_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int U, int gs,
                      const float* __restrict__ l1, float* l2o,
                      const float* __restrict__ F, float* ut, const float* __restrict__ utm1,
                      const float* __restrict__ strip_tm1, const double* __restrict__ rres_t,
                      double* __restrict__ acc_part, int has1, int has2, int do_img, int do_recon) {
  const Lane L = lane_geo(g, kRXA);
  if (L.x0 >= g.nx) return;
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  const int nz = g.nz;
  const size_t N2 = (size_t)g.nx * nz;
  const size_t pb = (size_t)sg.b * N2;
  const int zc = L.zin ? L.z : 0;
  const int z = L.z;
  const bool zbox = z >= g.z_lo && z <= g.z_hi;
  // ring columns inside the grid only (no PML: the ring lies outside, = 0)
  const int ringz = !L.zin ? -1 : (z == g.z_lo - 1) ? 2 * g.Lz : (z == g.z_hi + 1) ? 2 * g.Lz + g.Lx : -1;

  // per-phantom coefficients (shared by every shot of the group)
  double edv[kRXA + 2];
#pragma unroll
  for (int r = 0; r < kRXA + 2; ++r) {
    const int x = L.x0 - 1 + r;
    edv[r] = (L.zin && x >= 0 && x < g.nx) ? __ldg(m.Ed + pb + (size_t)x * nz + zc) : 0.0;
  }
  double qv[kRXA + 2], rv[kRXA + 2];
  if (RHO) {
#pragma unroll
    for (int r = 0; r < kRXA + 2; ++r) {
      const int x = L.x0 - 1 + r;
      const bool ok = L.zin && x >= 0 && x < g.nx;
      qv[r] = ok ? __ldg(m.q + pb + (size_t)x * nz + zc) : 0.0;
      rv[r] = ok ? __ldg(m.rho + pb + (size_t)x * nz + zc) : 0.0;
    }
  }
  double pzz = 0.0, Azz = 2.0, Bzz = -1.0;
  if (T.px && L.zin) { pzz = __ldg(T.pz + L.z); Azz = __ldg(T.Az + L.z); Bzz = __ldg(T.Bz + L.z); }
  double Ar[kRXA], Br[kRXA];
  int slot[kRXA];
#pragma unroll
  for (int r = 0; r < kRXA; ++r) {
    const int x = min(L.x0 + r, g.nx - 1);
    ab_at(T, x, pzz, Azz, Bzz, (size_t)x * nz + zc, Ar[r], Br[r]);
    slot[r] = -1;
    if (L.comp && L.x0 + r < g.nx && __ldg(g.row_flag + x)) slot[r] = __ldg(g.node_slot + (size_t)x * nz + z);
  }
  const double pulse_t = __ldg(g.pulse + t);
  double acc[kRXA];
#pragma unroll
  for (int r = 0; r < kRXA; ++r) acc[r] = 0.0;

  for (int k0 = 0; k0 < sg.n; k0 += kNSA) {
    // ---- all loads of this shot batch first
    double lv[kNSA][kRXA + 2], l2v[kNSA][kRXA], fv[kNSA][kRXA + 2], utv[kNSA][kRXA], rr[kNSA][kRXA];
    int txr[kNSA];
#pragma unroll
    for (int k = 0; k < kNSA; ++k) {
      const bool ak = k0 + k < sg.n;
      const int lu = sg.lu0 + (ak ? k0 + k : 0);
      const size_t fo = (size_t)lu * N2;
      const int s = (unit_begin + lu) % g.S;
      txr[k] = (ak && __ldg(g.tx + 2 * s + 1) == z) ? __ldg(g.tx + 2 * s) - L.x0 : -1;
#pragma unroll
      for (int r = 0; r < kRXA + 2; ++r) {
        const int x = L.x0 - 1 + r;
        const bool okx = L.zin && x >= 0 && x < g.nx && ak;
        lv[k][r] = (has1 && okx) ? (double)__ldg(l1 + fo + (size_t)x * nz + zc) : 0.0;
        double f = 0.0;
        if (do_img && okx) {
          if (MODE == 1) {
            f = (double)__ldg(F + fo + (size_t)x * nz + zc);
          } else {
            const bool xbox = x >= g.x_lo && x <= g.x_hi;
            const float* st = strip_tm1 + (size_t)lu * g.SL;
            if (xbox && zbox) f = (double)utm1[fo + (size_t)x * nz + z];
            else if (zbox && x == g.x_lo - 1) f = (double)__ldg(st + z - g.z_lo);
            else if (zbox && x == g.x_hi + 1) f = (double)__ldg(st + g.Lz + z - g.z_lo);
            else if (xbox && ringz >= 0) f = (double)__ldg(st + ringz + x - g.x_lo);
          }
        }
        fv[k][r] = f;
      }
#pragma unroll
      for (int r = 0; r < kRXA; ++r) {
        const int x = L.x0 + r;
        const bool okc = L.comp && x < g.nx && ak;
        l2v[k][r] = (has2 && okc) ? (double)l2o[fo + (size_t)x * nz + z] : 0.0;
        utv[k][r] = (MODE == 2 && do_recon && okc) ? (double)ut[fo + (size_t)x * nz + z] : 0.0;
        rr[k][r] = (okc && slot[r] >= 0) ? __ldg(rres_t + (size_t)lu * g.M + slot[r]) : 0.0;
      }
    }
    // ---- compute and store
#pragma unroll
    for (int k = 0; k < kNSA; ++k) {
      const bool ak = k0 + k < sg.n;
      const size_t fo = (size_t)(sg.lu0 + (ak ? k0 + k : 0)) * N2;
      double el[kRXA + 2];
#pragma unroll
      for (int r = 0; r < kRXA + 2; ++r) el[r] = edv[r] * lv[k][r];
#pragma unroll
      for (int r = 0; r < kRXA; ++r) {
        const int x = L.x0 + r;
        const size_t cell = (size_t)x * nz + z;
        RhoW2 w{};
        if (RHO) {
          const double qzm = shfl_up1(qv[r + 1]), qzp = shfl_dn1(qv[r + 1]);
          const double rzm = shfl_up1(rv[r + 1]), rzp = shfl_dn1(rv[r + 1]);
          w = rho_w2(rv[r + 1], qv[r + 1], rv[r], qv[r], rv[r + 2], qv[r + 2], rzm, qzm, rzp, qzp,
                     x > 0, x + 1 < g.nx, z > 0, z < nz - 1);
        }
        const double ec = el[r + 1];
        const double ezm = shfl_up1(ec), ezp = shfl_dn1(ec);
        const double adj = RHO ? ((((-w.W * ec + w.ixm * el[r]) + w.ixp * el[r + 2]) + w.izm * ezm) + w.izp * ezp)
                               : ((((-4.0 * ec + el[r]) + el[r + 2]) + ezm) + ezp);
        const double lam = ((Ar[r] * lv[k][r + 1] + adj) + Br[r] * l2v[k][r]) + rr[k][r];
        const double fc = fv[k][r + 1];
        const double fzm = shfl_up1(fc), fzp = shfl_dn1(fc);
        if (L.comp && x < g.nx && ak) {
          l2o[fo + cell] = (float)lam;
          const bool interior = MODE == 2 ? (zbox && x >= g.x_lo && x <= g.x_hi) : true;
          if (do_img && interior) {
            const double lapu = RHO ? ((((-w.W * fc + w.wxm * fv[k][r]) + w.wxp * fv[k][r + 2]) + w.wzm * fzm) + w.wzp * fzp)
                                    : ((((-4.0 * fc + fv[k][r]) + fv[k][r + 2]) + fzm) + fzp);
            acc[r] += lapu * lam;
            if (MODE == 2 && do_recon) {
              double prev = 2.0 * fc + edv[r + 1] * lapu - utv[k][r];
              if (txr[k] == r) prev += pulse_t;
              ut[fo + cell] = (float)prev;
            }
          }
        }
      }
    }
  }
  if (do_img && L.comp) {
    double* dst = acc_part + (size_t)blockIdx.z * N2;
#pragma unroll
    for (int r = 0; r < kRXA; ++r) {
      const int x = L.x0 + r;
      if (x < g.nx) dst[(size_t)x * nz + z] += acc[r];
    }
  }
}

}  // namespace dufwi
