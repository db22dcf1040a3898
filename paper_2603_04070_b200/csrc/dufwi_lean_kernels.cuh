// Stepwise engine, lean streaming kernels (nz % 4 == 0, separable damping with
// a rectangular undamped box: every BASELINE config, configs 2/3 with density).
//
// A warp owns a 128-wide z strip (4 cells per lane, float4 loads/stores) and
// walks x-rows, rows ahead streaming through a per-lane cp.async ring of 3
// slots.  Shaped for instruction count, which ncu showed to be the limiter of
// the first stepwise kernels (~420 warp instructions per 128-cell row,
// issue-bound at 27% of DRAM peak):
//   * the x loop is unrolled by the ring depth (a multiple of 3), so ring slots
//     are immediate offsets and the 3-row register window (x-1, x, x+1)
//     rotates by renaming instead of register moves;
//   * addresses are one IMAD.WIDE from an opaque per-lane base and a 32-bit
//     row offset;
//   * per-lane constants hoisted out of the loop: (A, B) of the z-damping band
//     (only for warps touching it, template switch), receiver / ring columns,
//     source cell; per-row work is warp-uniform compares;
//   * one edge value per lane per row (lane 0: z0-1, lane 31: z0+128);
//   * 128-register cap: 4 CTAs of 4 warps per SM.
//
// Variable density (RHO).  The oracle's operator is
// L_rho u = rho_c sum_j f_cj (u_j - u_c) with face factors f_cj = (q_c + q_j)/2,
// q = 1/rho, outer faces f = q_c and u = 0 outside (oracle rho_face_weights).
// Writing D u = sum_j f_cj u_j - S_c u_c (S_c = sum of the 4 face factors),
// L_rho = diag(rho) D with D symmetric, so per phantom two maps are streamed:
// Er = rho E / dx^2 and q; the face factors of D are formed in registers from
// the q rows (QRing, rho_row):
//   forward   u[t]  = A u1 + B u2 + Er * D(u1)
//   adjoint   lam   = A l1 + B l2 + D(Er * l1)        ((E L_rho)^T = D diag(Er))
//   imaging   acc  += D(u[t-1]) * lam, scaled by rho once in reduce_groups
//   recon     u[t-2] = 2 u1 + Er * D(u1) - u[t] (+ source)
// The same f64 values as the oracle up to summation order (parity by tolerance).
//
// Arithmetic: explicitly rounded f64 (dufwi_common.cuh), lap5 / fwd_update /
// adj_update as in the cluster engine.  The coefficient maps (E/dx^2, or Er
// and q) are streamed as f32 copies written by set_model (a relative change of
// the medium below 6e-8, far inside the 1e-4 parity bar): 4 B instead of 8 B
// per cell and map through L2 and the ring, one cp.async instead of two.
// DRAM per cell update: forward 12 B (read u[t-1], u[t-2], write u[t]); lam
// update 12 B; imaging + reconstruction 16 B (+16 B / gs accumulator);
// coefficient maps come from L2 (shared by the phantom's shots).
#pragma once

#include "dufwi_vec_kernels.cuh"

namespace dufwi {

#ifndef DUFWI_LEAN_WARPS
#define DUFWI_LEAN_WARPS 4
#endif
#ifndef DUFWI_LEAN_MINB
#define DUFWI_LEAN_MINB 4
#endif
constexpr int kLeanWarps = DUFWI_LEAN_WARPS;  // warps per CTA
#ifndef DUFWI_LEAN_MINB_RHO
#define DUFWI_LEAN_MINB_RHO 3
#endif
constexpr int kLeanMinB = DUFWI_LEAN_MINB;        // min resident CTAs per SM (register cap)
constexpr int kLeanMinBRho = DUFWI_LEAN_MINB_RHO;  // density kernels: more live f64 state
constexpr int kLeanT = kLeanWarps * 32;
// Lane groups: a warp is kSPW groups of kLS lanes, each group on a kSW-wide z
// strip (4 cells per lane).  kSW = 64: two groups per warp, so a grid whose
// last strip is partial idles at most 15 lanes per group (560 columns: 97% of
// the lanes busy instead of 87.5% with 128-wide strips; 296: 92.5% vs 77%;
// 1088: 100% vs 94%).  The forward and lam update put two units in a warp,
// the imaging kernel two row blocks of the same shot group.
#ifndef DUFWI_LEAN_SW
#define DUFWI_LEAN_SW 64
#endif
constexpr int kSW = DUFWI_LEAN_SW;
constexpr int kLS = kSW / 4;    // lanes per group (the shuffle width)
constexpr int kSPW = 32 / kLS;  // groups per warp
static_assert(kSW == 64 || kSW == 128, "lane-group strip width");
constexpr int kNSL = 3;                       // ring slots (measured best: 3 > 6)
#ifndef DUFWI_FWD_NSL
#define DUFWI_FWD_NSL 3
#endif
constexpr int kFwdNSL = DUFWI_FWD_NSL;         // forward ring slots (>3: runtime slot index)

// Per-lane constants of a 4-cell z segment.
struct LaneInfo {
  int z4;
  bool on;           // the lane group has work (a unit / row block)
  bool act;          // on, and the lane's cells lie in the grid
  unsigned rxk;      // cells on a receiver column
  unsigned boxk;     // cells with z in [z_lo, z_hi]
  int ringl, ringr;  // cell index on ring column z_lo-1 / z_hi+1, or -1
  bool zd;           // any cell in the z damping band
};

__device__ __forceinline__ LaneInfo lane_info(const Geo& g, const ABTables& T, int z4, bool on) {
  LaneInfo L;
  L.z4 = z4;
  L.on = on;
  L.act = on && z4 < g.nz;
  L.rxk = L.boxk = 0u;
  L.ringl = L.ringr = -1;
  L.zd = false;
  if (L.act) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int z = z4 + k;
      if (__ldg(g.col_flag + z)) L.rxk |= 1u << k;
      if (z >= g.z_lo && z <= g.z_hi) L.boxk |= 1u << k;
      if (z == g.z_lo - 1) L.ringl = k;
      if (z == g.z_hi + 1) L.ringr = k;
      if (__ldg(T.pz + z) != 0.0) L.zd = true;
    }
  }
  return L;
}

// Hide a per-lane base pointer from re-association, so base + 32-bit row
// offset compiles to one IMAD.WIDE instead of a 64-bit add chain.
template <class P>
__device__ __forceinline__ P* opaque(P* p) {
  asm volatile("" : "+l"(p));
  return p;
}

// (A, B) of cell (x, z) in a damped row: D = max(px[x], pz[z]) picks the table.
__device__ __forceinline__ double2 ab_row_damped(const ABTables& T, double pxx, double Axx,
                                                 double Bxx, int z) {
  return pxx >= __ldg(T.pz + z) ? make_double2(Axx, Bxx)
                                : make_double2(__ldg(T.Az + z), __ldg(T.Bz + z));
}

// D(u)_c = sum_j f_cj u_j - S_c u_c (variable-density operator without rho_c).
__device__ __forceinline__ double lapf(double c, double xm, double xp, double zm, double zp,
                                       double fxm, double fxp, double fzm, double fzp) {
  const double S = __dadd_rn(__dadd_rn(__dadd_rn(fxm, fxp), fzm), fzp);
  return __fma_rn(fzp, zp, __fma_rn(fzm, zm, __fma_rn(fxp, xp, __fma_rn(fxm, xm, __dmul_rn(-S, c)))));
}

// q = 1/rho rows of the density operator, streamed alongside the fields.  The
// face factors are formed in registers as 0.5 * (q_c + q_j): the expression
// (hence the bits) of the oracle's rho_face_weights and of rho_faces_kernel's
// tables; an outer face is 0.5 * (q_c + q_c) == q_c exactly.  One f64 stream
// (8 B per cell) instead of the two face tables (16 B), and 40 B instead of
// 72 B of ring per lane and slot.
template <int NSL>
struct QRing {
  float4 q[NSL][kLeanT];   // q row (f32 copy; the face arithmetic is f64)
  float qe[NSL][kLeanT];   // q at the lane's edge column
};
template <int NSL, bool RHO>
struct QRingOpt {};
template <int NSL>
struct QRingOpt<NSL, true> {
  QRing<NSL> r;
};

// Per-lane view of one phantom's q map.
struct QLane {
  const float* q;   // q + zc (row r at r * nz)
  const float* qe;  // q + edge column (first lane of a group: z0-1, last: z0+kSW)
  bool edge;         // the lane has an edge column inside the grid
  bool lo, hi;       // the lane's first / last cell is z = 0 / z = nz-1 (outer faces)
};

__device__ __forceinline__ QLane q_lane(const Model& m, const Geo& g, int b, int zc, int z0,
                                        int l, int z4, bool on) {
  QLane Q;
  const float* qb = m.qf + (size_t)b * g.nx * g.nz;
  const bool el = on && l == 0 && z0 > 0, er = on && l == kLS - 1 && z0 + kSW < g.nz;
  Q.q = opaque(qb + zc);
  Q.qe = opaque(qb + (el ? z0 - 1 : er ? z0 + kSW : 0));
  Q.edge = el || er;
  Q.lo = z4 == 0;
  Q.hi = z4 + 4 >= g.nz;
  return Q;
}

template <int NSL>
__device__ __forceinline__ void issue_q(QRing<NSL>& R, const QLane& Q, int tid, int sl, int r,
                                        bool ok, bool act, int nz) {
  cp16(&R.q[sl][tid], Q.q + r * nz, ok && act);
  cp4(&R.qe[sl][tid], Q.qe + r * nz, ok && Q.edge);
}

template <int NSL>
__device__ __forceinline__ void read_q(const QRing<NSL>& R, int tid, int sl, double (&q)[4],
                                       double& qe) {
  const float4 a = R.q[sl][tid];
  q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
  qe = R.qe[sl][tid];
}

__device__ __forceinline__ double face(double a, double b) {
  return __dmul_rn(0.5, __dadd_rn(a, b));
}

// z faces of a lane's 4 cells in one row: fz[k] lies between cells k-1 and k
// (fz[0] / fz[4]: the neighbours in lanes -1 / +1, the edge column, or outer).
__device__ __forceinline__ void zfaces(const QLane& Q, int l, const double (&q)[4], double qe,
                                       double (&fz)[5]) {
  double ql = __shfl_up_sync(0xffffffffu, q[3], 1, kLS);
  double qr = __shfl_down_sync(0xffffffffu, q[0], 1, kLS);
  if (l == 0) ql = qe;
  if (l == kLS - 1) qr = qe;
  if (Q.lo) ql = q[0];
  if (Q.hi) qr = q[3];
  fz[0] = face(ql, q[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) fz[k] = face(q[k - 1], q[k]);
  fz[4] = face(q[3], qr);
}

// Row-walk state at the first row x0: q of row x0 (+ edge column) and the
// x face above it, fxe[x0] = face(q[x0-1], q[x0]) (outer at x0 = 0: q[0]).
__device__ __forceinline__ void rho_prologue(const QLane& Q, bool act, int x0, int nz,
                                             double (&qc)[4], double& qce, double (&fx)[4]) {
  if (act) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(Q.q + x0 * nz));
    qc[0] = a.x; qc[1] = a.y; qc[2] = a.z; qc[3] = a.w;
  }
  if (Q.edge) qce = __ldg(Q.qe + x0 * nz);
  double qm[4] = {qc[0], qc[1], qc[2], qc[3]};
  if (act && x0 >= 1) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(Q.q + (x0 - 1) * nz));
    qm[0] = a.x; qm[1] = a.y; qm[2] = a.z; qm[3] = a.w;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) fx[k] = face(qm[k], qc[k]);
}

// One row x of the walk: q of row x+1 from ring slot sl (outer below the last
// row: q of row x again) gives the x face below row x; the z faces of row x come
// from the carried q of row x, which then advances to row x+1.
template <int NSL>
__device__ __forceinline__ void rho_row(const QRing<NSL>& R, const QLane& Q, int tid, int sl,
                                        int l, bool has_next, double (&qc)[4], double& qce,
                                        double (&fxp)[4], double (&fz)[5]) {
  double qn[4], qen;
  read_q(R, tid, sl, qn, qen);
  if (!has_next) {
#pragma unroll
    for (int k = 0; k < 4; ++k) qn[k] = qc[k];
    qen = qce;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) fxp[k] = face(qc[k], qn[k]);
  zfaces(Q, l, qc, qce, fz);
#pragma unroll
  for (int k = 0; k < 4; ++k) qc[k] = qn[k];
  qce = qen;
}

// ----------------------------------------------------------------- forward
template <int NSL, bool RHO>
struct LeanFwdRing {
  float4 u1[NSL][kLeanT];   // u[t-1] row r+1
  float4 u2[NSL][kLeanT];   // u[t-2] row r
  float4 e[NSL][kLeanT];    // E (RHO: Er) row r, f32 copy
  float edge[NSL][kLeanT];  // u[t-1] row r+1 at the group's edge column (z0-1 / z0+kSW)
  QRingOpt<NSL, RHO> fr;    // RHO: q row r+1
};

template <int MODE, bool RHO, bool ZD>
__device__ __forceinline__ void fwd_lean_rows(const Geo& g, const ABTables& T, const LaneInfo& L,
                                              LeanFwdRing<kFwdNSL, RHO>& ring, const QLane& QL,
                                              int tid, int lane, int z0, int x0, int x1, int lu,
                                              int txx, int tk, double pulse_t, const float* f1,
                                              const float* f2, const float* Ec, float* fo,
                                              float* rec_t, float* strip_t, bool has1, bool has2,
                                              bool wrx, bool wring) {
  constexpr int NSL = kFwdNSL;
  const int nz = g.nz, nx = g.nx;
  const int zc = L.act ? L.z4 : 0;
  const bool edge_l = L.on && lane == 0 && z0 > 0;
  const bool edge_r = L.on && lane == kLS - 1 && z0 + kSW < g.nz;
  const int ze = edge_l ? z0 - 1 : edge_r ? z0 + kSW : 0;
  const bool has_edge = has1 && (edge_l || edge_r);
  const bool ok1 = has1 && L.act, ok2 = has2 && L.act;
  const float* b1 = opaque(f1 + zc);
  const float* b2 = opaque(f2 + zc);
  const float* be = opaque(Ec + zc);
  const float* bl = opaque(f1 + ze);
  float* bo = opaque(fo + zc);
  double Az[4], Bz[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Az[k] = 2.0;
    Bz[k] = -1.0;
    if (ZD && L.act && L.zd) {
      Az[k] = __ldg(T.Az + L.z4 + k);
      Bz[k] = __ldg(T.Bz + L.z4 + k);
    }
  }
  // copies of "row r": u[t-1] row r+1 (+ edge), u[t-2] row r, E row r (+ faces)
  auto issue = [&](int r, int sl) {
    const bool okn = r + 1 < nx;
    const int on = okn ? (r + 1) * nz : 0;
    const int orr = r * nz;
    cp16(&ring.u1[sl][tid], b1 + on, ok1 && okn);
    cp16(&ring.u2[sl][tid], b2 + orr, ok2);
    cp16(&ring.e[sl][tid], be + orr, L.act);
    cp4(&ring.edge[sl][tid], bl + on, has_edge && okn);
    if constexpr (RHO) issue_q(ring.fr.r, QL, tid, sl, r + 1, okn, L.act, nz);
  };
  // register windows: slot (k) % 3 = row x-1, (k+1) % 3 = row x, (k+2) % 3 = row x+1;
  // FX[s] = x face above the row of slot s (fxe[row]); qc / qce: q of row x
  double W[3][4], Eg[3], FX[3][4], qc[4] = {0.0, 0.0, 0.0, 0.0}, qce = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) W[0][k] = W[1][k] = W[2][k] = FX[0][k] = FX[1][k] = FX[2][k] = 0.0;
  Eg[0] = Eg[1] = Eg[2] = 0.0;
  if (has1) {
    if (x0 >= 1 && L.act) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(b1 + (x0 - 1) * nz));
      W[0][0] = f.x; W[0][1] = f.y; W[0][2] = f.z; W[0][3] = f.w;
    }
    if (L.act) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(b1 + x0 * nz));
      W[1][0] = f.x; W[1][1] = f.y; W[1][2] = f.z; W[1][3] = f.w;
    }
    if (edge_l || edge_r) Eg[1] = (double)__ldg(bl + x0 * nz);
  }
  if constexpr (RHO) rho_prologue(QL, L.act, x0, nz, qc, qce, FX[1]);
#pragma unroll
  for (int k = 0; k < NSL - 1; ++k) {
    if (x0 + k < x1) issue(x0 + k, k);
    cp_commit();
  }
  // unrolled by 3 (the register window); with NSL == 3 the ring slot is the
  // unroll index, deeper rings index their slot at run time
  constexpr int UNR = 3;
  int sr = 0, si = NSL - 1;
  for (int xb = x0; xb < x1; xb += UNR) {
#pragma unroll
    for (int k0 = 0; k0 < UNR; ++k0) {
      const int x = xb + k0;
      if (x >= x1) break;
      const int k = NSL == 3 ? k0 : sr;
      const int im = k0 % 3, ic = (k0 + 1) % 3, ip = (k0 + 2) % 3;
      if (x + NSL - 1 < x1) issue(x + NSL - 1, NSL == 3 ? (k0 + NSL - 1) % NSL : si);
      cp_commit();
      cp_wait<NSL - 1>();  // the group of row x has landed
      if (NSL != 3) {
        sr = sr + 1 == NSL ? 0 : sr + 1;
        si = si + 1 == NSL ? 0 : si + 1;
      }
      {
        const float4 f = ring.u1[k][tid];
        W[ip][0] = f.x; W[ip][1] = f.y; W[ip][2] = f.z; W[ip][3] = f.w;
        Eg[ip] = (double)ring.edge[k][tid];
      }
      const float4 w2 = ring.u2[k][tid];
      const float4 ef = ring.e[k][tid];
      const double u2v[4] = {w2.x, w2.y, w2.z, w2.w};
      const double ed[4] = {ef.x, ef.y, ef.z, ef.w};
      double zl = __shfl_up_sync(0xffffffffu, W[ic][3], 1, kLS);
      double zr = __shfl_down_sync(0xffffffffu, W[ic][0], 1, kLS);
      if (lane == 0) zl = Eg[ic];
      if (lane == kLS - 1) zr = Eg[ic];
      double lap[4];
      if constexpr (RHO) {
        double fz[5];
        rho_row(ring.fr.r, QL, tid, k, lane, x + 1 < nx, qc, qce, FX[ip], fz);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double zm = c == 0 ? zl : W[ic][c - 1];
          const double zp = c == 3 ? zr : W[ic][c + 1];
          lap[c] = lapf(W[ic][c], W[im][c], W[ip][c], zm, zp, FX[ic][c], FX[ip][c], fz[c], fz[c + 1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double zm = c == 0 ? zl : W[ic][c - 1];
          const double zp = c == 3 ? zr : W[ic][c + 1];
          lap[c] = lap5(W[ic][c], W[im][c], W[ip][c], zm, zp);
        }
      }
      double v[4];
      if (x >= g.x_lo && x <= g.x_hi) {  // undamped row: (A, B) of the lane's z band
#pragma unroll
        for (int c = 0; c < 4; ++c)
          v[c] = ZD ? fwd_update(Az[c], Bz[c], W[ic][c], u2v[c], ed[c], lap[c])
                    : fwd_update_free(W[ic][c], u2v[c], ed[c], lap[c]);
      } else {  // damped row (x band of the PML)
        const double pxx = __ldg(T.px + x), Axx = __ldg(T.Ax + x), Bxx = __ldg(T.Bx + x);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 ab = ab_row_damped(T, pxx, Axx, Bxx, min(L.z4 + c, nz - 1));
          v[c] = fwd_update(ab.x, ab.y, W[ic][c], u2v[c], ed[c], lap[c]);
        }
      }
      if (x == txx) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c == tk) v[c] = __dadd_rn(v[c], pulse_t);
      }
      if (L.act) {
        const int orow = x * nz;
        *reinterpret_cast<float4*>(bo + orow) =
            make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
        if (wrx && L.rxk && __ldg(g.row_flag + x)) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (L.rxk & (1u << c)) {
              const int slot = __ldg(g.node_slot + orow + L.z4 + c);
              if (slot >= 0) rec_t[(size_t)lu * g.M + slot] = (float)v[c];
            }
        }
        if (MODE == 2) {
          float* st = strip_t + (size_t)lu * g.SL;
          if (x == g.x_lo - 1 || x == g.x_hi + 1) {
            const int base = (x == g.x_lo - 1 ? 0 : g.Lz) - g.z_lo + L.z4;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (L.boxk & (1u << c)) st[base + c] = (float)v[c];
          } else if (wring && x >= g.x_lo && x <= g.x_hi) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (c == L.ringl) st[2 * g.Lz + x - g.x_lo] = (float)v[c];
              if (c == L.ringr) st[2 * g.Lz + g.Lx + x - g.x_lo] = (float)v[c];
            }
          }
        }
      }
    }
  }
  cp_wait<0>();
}

template <int MODE, bool RHO>
__global__ void __launch_bounds__(kLeanT, RHO ? kLeanMinBRho : kLeanMinB)
    fwd_lean_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int U, int TX,
                    const float* __restrict__ u1, const float* u2, float* uo,
                    float* __restrict__ rec_t, float* __restrict__ strip_t, int has1, int has2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& ring = *reinterpret_cast<LeanFwdRing<kFwdNSL, RHO>*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int l = lane % kLS;  // lane within its group; group lane / kLS works on its own unit
  const int z0 = blockIdx.x * kSW;
  const int x0 = (blockIdx.y * kLeanWarps + warp) * TX;
  if (x0 >= g.nx) return;  // warp-uniform
  const int x1 = min(g.nx, x0 + TX);
  const int lu0 = blockIdx.z * kSPW + lane / kLS;
  const bool on = lu0 < U;
  const int lu = on ? lu0 : U - 1;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * g.nz;
  const LaneInfo L = lane_info(g, T, z0 + 4 * l, on);
  const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
  const int tk = (L.act && txz >= L.z4 && txz < L.z4 + 4) ? txz - L.z4 : -1;
  const double pulse_t = __ldg(g.pulse + t);
  const bool wrx = __any_sync(0xffffffffu, L.rxk != 0u);
  const bool wring = __any_sync(0xffffffffu, L.ringl >= 0 || L.ringr >= 0);
  const bool wzd = __any_sync(0xffffffffu, L.zd);
  const float* f1 = u1 + (size_t)lu * N2;
  const float* f2 = u2 + (size_t)lu * N2;
  float* fo = uo + (size_t)lu * N2;
  const float* Ec = (RHO ? m.Erf : m.Edf) + (size_t)b * N2;
  QLane QL{};
  if constexpr (RHO) QL = q_lane(m, g, b, L.act ? L.z4 : 0, z0, l, L.z4, on);
  if (wzd)
    fwd_lean_rows<MODE, RHO, true>(g, T, L, ring, QL, tid, l, z0, x0, x1, lu, txx, tk, pulse_t,
                                   f1, f2, Ec, fo, rec_t, strip_t, has1, has2, wrx, wring);
  else
    fwd_lean_rows<MODE, RHO, false>(g, T, L, ring, QL, tid, l, z0, x0, x1, lu, txx, tk, pulse_t,
                                    f1, f2, Ec, fo, rec_t, strip_t, has1, has2, wrx, wring);
}

// --------------------------------------------------------------- lam update
// lam[t] = A lam[t+1] + L^T(E lam[t+1]) + B lam[t+2] (+ merged residual at the
// receiver nodes), in place over lam[t+2] (adjoint.py:119-131).  RHO:
// L^T(E lam) = D(Er lam).
template <int NSL, bool RHO>
struct LeanAdjRing {
  float4 l1[NSL][kLeanT];    // lam[t+1] row r+1
  float4 e[NSL][kLeanT];     // E (RHO: Er) row r+1, f32 copy
  float4 l2[NSL][kLeanT];    // lam[t+2] row r
  float edl[NSL][kLeanT];    // lam[t+1] row r+1 at the lane's edge column
  float ede[NSL][kLeanT];    // E row r+1 at the lane's edge column
  QRingOpt<NSL, RHO> fr;     // RHO: q row r+1
};

template <bool RHO, bool ZD>
__device__ __forceinline__ void adjlam_lean_rows(const Geo& g, const ABTables& T,
                                                 const LaneInfo& L, LeanAdjRing<kNSL, RHO>& ring,
                                                 const QLane& QL, int tid, int lane, int z0,
                                                 int x0, int x1, int lu, const float* L1,
                                                 float* L2, const float* Ec,
                                                 const double* rres_t, bool has1, bool has2,
                                                 bool wrx) {
  constexpr int NSL = kNSL;
  const int nz = g.nz, nx = g.nx;
  const int zc = L.act ? L.z4 : 0;
  const bool edge_l = L.on && lane == 0 && z0 > 0;
  const bool edge_r = L.on && lane == kLS - 1 && z0 + kSW < g.nz;
  const bool has_edge = edge_l || edge_r;
  const int ze = edge_l ? z0 - 1 : edge_r ? z0 + kSW : 0;
  const bool ok1 = has1 && L.act, ok2 = has2 && L.act;
  const float* b1 = opaque(L1 + zc);
  float* b2 = opaque(L2 + zc);
  const float* be = opaque(Ec + zc);
  const float* bl = opaque(L1 + ze);
  const float* bel = opaque(Ec + ze);
  double Az[4], Bz[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Az[k] = 2.0;
    Bz[k] = -1.0;
    if (ZD && L.act && L.zd) {
      Az[k] = __ldg(T.Az + L.z4 + k);
      Bz[k] = __ldg(T.Bz + L.z4 + k);
    }
  }
  auto issue = [&](int r, int sl) {
    const bool okn = r + 1 < nx;
    const int on = okn ? (r + 1) * nz : 0;
    const int orr = r * nz;
    cp16(&ring.l1[sl][tid], b1 + on, ok1 && okn);
    cp16(&ring.e[sl][tid], be + on, L.act && okn);
    cp16(&ring.l2[sl][tid], b2 + orr, ok2);
    cp4(&ring.edl[sl][tid], bl + on, has1 && has_edge && okn);
    cp4(&ring.ede[sl][tid], bel + on, has_edge && okn);
    if constexpr (RHO) issue_q(ring.fr.r, QL, tid, sl, r + 1, okn, L.act, nz);
  };
  // windows of E*lam1 (EL) and raw lam1 (RL), slot (k)%3 = row x-1, (k+1)%3 = x,
  // (k+2)%3 = x+1; FX[s] = x face above the row of slot s; qc / qce: q of row x
  double EL[3][4], RL[3][4], EG[3], FX[3][4], qc[4] = {0.0, 0.0, 0.0, 0.0}, qce = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    EL[0][k] = EL[1][k] = EL[2][k] = RL[0][k] = RL[1][k] = RL[2][k] = FX[0][k] = FX[1][k] =
        FX[2][k] = 0.0;
  EG[0] = EG[1] = EG[2] = 0.0;
  if (has1) {
    auto ld = [&](int x, int w) {
      if (L.act) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(b1 + x * nz));
        const float4 a = __ldg(reinterpret_cast<const float4*>(be + x * nz));
        RL[w][0] = f.x; RL[w][1] = f.y; RL[w][2] = f.z; RL[w][3] = f.w;
        EL[w][0] = __dmul_rn(a.x, RL[w][0]);
        EL[w][1] = __dmul_rn(a.y, RL[w][1]);
        EL[w][2] = __dmul_rn(a.z, RL[w][2]);
        EL[w][3] = __dmul_rn(a.w, RL[w][3]);
      }
      if (has_edge) EG[w] = __dmul_rn((double)__ldg(bel + x * nz), (double)__ldg(bl + x * nz));
    };
    if (x0 >= 1) ld(x0 - 1, 0);
    ld(x0, 1);
  }
  if constexpr (RHO) rho_prologue(QL, L.act, x0, nz, qc, qce, FX[1]);
#pragma unroll
  for (int k = 0; k < NSL - 1; ++k) {
    if (x0 + k < x1) issue(x0 + k, k);
    cp_commit();
  }
  for (int xb = x0; xb < x1; xb += NSL) {
#pragma unroll
    for (int k = 0; k < NSL; ++k) {
      const int x = xb + k;
      if (x >= x1) break;
      const int im = k % 3, ic = (k + 1) % 3, ip = (k + 2) % 3;
      if (x + NSL - 1 < x1) issue(x + NSL - 1, (k + NSL - 1) % NSL);
      cp_commit();
      cp_wait<NSL - 1>();
      {
        const float4 f = ring.l1[k][tid];
        const float4 a = ring.e[k][tid];
        RL[ip][0] = f.x; RL[ip][1] = f.y; RL[ip][2] = f.z; RL[ip][3] = f.w;
        EL[ip][0] = __dmul_rn(a.x, RL[ip][0]);
        EL[ip][1] = __dmul_rn(a.y, RL[ip][1]);
        EL[ip][2] = __dmul_rn(a.z, RL[ip][2]);
        EL[ip][3] = __dmul_rn(a.w, RL[ip][3]);
        EG[ip] = __dmul_rn((double)ring.ede[k][tid], (double)ring.edl[k][tid]);
      }
      const float4 w2 = ring.l2[k][tid];
      const double l2v[4] = {w2.x, w2.y, w2.z, w2.w};
      double zl = __shfl_up_sync(0xffffffffu, EL[ic][3], 1, kLS);
      double zr = __shfl_down_sync(0xffffffffu, EL[ic][0], 1, kLS);
      if (lane == 0) zl = EG[ic];
      if (lane == kLS - 1) zr = EG[ic];
      double adj[4];
      if constexpr (RHO) {
        double fz[5];
        rho_row(ring.fr.r, QL, tid, k, lane, x + 1 < nx, qc, qce, FX[ip], fz);
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
          const double zm = c2 == 0 ? zl : EL[ic][c2 - 1];
          const double zp = c2 == 3 ? zr : EL[ic][c2 + 1];
          adj[c2] = lapf(EL[ic][c2], EL[im][c2], EL[ip][c2], zm, zp, FX[ic][c2], FX[ip][c2], fz[c2],
                         fz[c2 + 1]);
        }
      } else {
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
          const double zm = c2 == 0 ? zl : EL[ic][c2 - 1];
          const double zp = c2 == 3 ? zr : EL[ic][c2 + 1];
          adj[c2] = lap5(EL[ic][c2], EL[im][c2], EL[ip][c2], zm, zp);
        }
      }
      double lam[4];
      if (x >= g.x_lo && x <= g.x_hi) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          lam[c] = ZD ? adj_update(Az[c], Bz[c], RL[ic][c], l2v[c], adj[c])
                      : adj_update_free(RL[ic][c], l2v[c], adj[c]);
      } else {
        const double pxx = __ldg(T.px + x), Axx = __ldg(T.Ax + x), Bxx = __ldg(T.Bx + x);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 ab = ab_row_damped(T, pxx, Axx, Bxx, min(L.z4 + c, nz - 1));
          lam[c] = adj_update(ab.x, ab.y, RL[ic][c], l2v[c], adj[c]);
        }
      }
      if (L.act) {
        const int orow = x * nz;
        if (wrx && L.rxk && __ldg(g.row_flag + x)) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (L.rxk & (1u << c)) {
              const int slot = __ldg(g.node_slot + orow + L.z4 + c);
              if (slot >= 0) lam[c] = __dadd_rn(lam[c], __ldg(rres_t + (size_t)lu * g.M + slot));
            }
        }
        *reinterpret_cast<float4*>(b2 + orow) =
            make_float4((float)lam[0], (float)lam[1], (float)lam[2], (float)lam[3]);
      }
    }
  }
  cp_wait<0>();
}

template <bool RHO>
__global__ void __launch_bounds__(kLeanT, RHO ? kLeanMinBRho : kLeanMinB)
    adjlam_lean_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int U, int TX,
                       const float* __restrict__ l1, float* l2o, const double* __restrict__ rres_t,
                       int has1, int has2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& ring = *reinterpret_cast<LeanAdjRing<kNSL, RHO>*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int l = lane % kLS;  // lane within its group; group lane / kLS works on its own unit
  const int z0 = blockIdx.x * kSW;
  const int x0 = (blockIdx.y * kLeanWarps + warp) * TX;
  if (x0 >= g.nx) return;  // warp-uniform
  const int x1 = min(g.nx, x0 + TX);
  const int lu0 = blockIdx.z * kSPW + lane / kLS;
  const bool on = lu0 < U;
  const int lu = on ? lu0 : U - 1;
  const int b = (unit_begin + lu) / g.S;
  const size_t N2 = (size_t)g.nx * g.nz;
  const LaneInfo L = lane_info(g, T, z0 + 4 * l, on);
  const bool wrx = __any_sync(0xffffffffu, L.rxk != 0u);
  const bool wzd = __any_sync(0xffffffffu, L.zd);
  const float* L1 = l1 + (size_t)lu * N2;
  float* L2 = l2o + (size_t)lu * N2;
  const float* Ec = (RHO ? m.Erf : m.Edf) + (size_t)b * N2;
  QLane QL{};
  if constexpr (RHO) QL = q_lane(m, g, b, L.act ? L.z4 : 0, z0, l, L.z4, on);
  if (wzd)
    adjlam_lean_rows<RHO, true>(g, T, L, ring, QL, tid, l, z0, x0, x1, lu, L1, L2, Ec, rres_t,
                                has1, has2, wrx);
  else
    adjlam_lean_rows<RHO, false>(g, T, L, ring, QL, tid, l, z0, x0, x1, lu, L1, L2, Ec, rres_t,
                                 has1, has2, wrx);
}

// ------------------------------------------------------ imaging + reconstruction
// sum_t L(u[t-1]) lam[t] over a group of gs shots of one phantom (adjoint.py:128-130)
// and, MODE 2, the reconstruction u[t-2] = 2 u[t-1] + E L u[t-1] + s[t] d_tx - u[t]
// in place over u[t] on the undamped box.
//
// A warp owns a 128-wide z strip x kImgTX box rows and walks the group's shots
// one after the other as ONE stream of ring items (kImgTX + 2 per shot): item i
// of a shot carries u[t-1] row x0-1+i (+ the lane's edge value, + RHO x faces)
// and, for i >= 2, lam[t], u[t], E and RHO z faces of row x0+i-2, so the
// pipeline never drains between shots.  The imaging sums of the warp's
// kImgTX x 4 cells per lane stay in registers for the whole group; one f64
// read-modify-write of acc_part[group] per cell at the end.
//
// MODE 2 keeps u[t-1] complete on the box AND its 1-cell ring in the field
// buffer: the reconstruction writes the box cells of u[t-2], and the ring cells
// of u[t-2] are copied from strips[t-2] (lanes on ring columns inline, the first
// and last warps for the ring rows).  The forward leaves u[nt-1], u[nt-2] complete,
// so the stencil of every box cell reads the field buffer only.
// MODE 1 reads u[t-1] from the full history (F = hist[t-1]) over the whole grid.
// DRAM per cell update: MODE 2 read u[t-1], u[t], lam[t], write u[t-2] = 16 B
// (+16 B / gs for the accumulator); MODE 1 read u[t-1], lam[t] = 8 B.
constexpr int kImgTX = 4;
constexpr int kImgItems = kImgTX + 2;  // ring items per shot (multiple of 3)
static_assert(kImgItems % 3 == 0 && kImgItems % kNSL == 0, "ring/window rotation");

template <bool RHO>
struct LeanImgRing {
  float4 u1[kNSL][kLeanT];    // u[t-1] row x0-1+i
  float4 lam[kNSL][kLeanT];   // lam[t] row x0+i-2
  float4 ut[kNSL][kLeanT];    // u[t] row x0+i-2 (MODE 2)
  float4 e[kNSL][kLeanT];     // E (RHO: Er) row x0+i-2, f32 copy (MODE 2)
  float edge[kNSL][kLeanT];   // u[t-1] row x0-1+i at the lane's edge column
  QRingOpt<kNSL, RHO> fr;     // RHO: q row x0-1+i
};

// PW: every lane of the warp has its 4 cells inside the box columns (no ring
// column, no cell outside the imaging region): the per-cell box / ring
// predicates and the ring-strip loads compile away (ncu: 36% of the kernel's
// instructions were ISETP / FSEL / SEL).
template <int MODE, bool RHO, bool PW>
__device__ __forceinline__ void img_lean_body(const Geo& g, const Model& m, int t, int unit_begin,
                                              int U, int gs, const float* __restrict__ lam_t,
                                              const float* __restrict__ F, float* ut,
                                              const float* __restrict__ utm1,
                                              const float* __restrict__ strip_tm2,
                                              double* __restrict__ acc_part, int do_recon) {
  constexpr int NSL = kNSL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& ring = *reinterpret_cast<LeanImgRing<RHO>*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nz = g.nz, nx = g.nx;
  const int l = lane % kLS;  // lane within its group; group lane / kLS takes its own row block
  const int z0 = blockIdx.x * kSW;
  const int rlo = MODE == 2 ? g.x_lo : 0, rhi = MODE == 2 ? g.x_hi + 1 : nx;  // rows [rlo, rhi)
  const int x0 = rlo + ((blockIdx.y * kLeanWarps + warp) * kSPW + lane / kLS) * kImgTX;
  const bool on = x0 < rhi;
  if (!__any_sync(0xffffffffu, on)) return;  // warp-uniform
  const int x1 = on ? min(rhi, x0 + kImgTX) : x0;  // an idle group walks no rows
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  const size_t N2 = (size_t)nx * nz;
  const int z4 = z0 + 4 * l;
  const bool act = PW || (on && z4 < nz);
  const int zc = act ? z4 : 0;
  const bool edge_l = on && l == 0 && z0 > 0, edge_r = on && l == kLS - 1 && z0 + kSW < nz;
  const bool has_edge = edge_l || edge_r;
  const int ze = edge_l ? z0 - 1 : edge_r ? z0 + kSW : 0;
  unsigned boxk = 0u;
  int ringl = -1, ringr = -1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int z = z4 + k;
    if (MODE == 1 ? act : (act && z >= g.z_lo && z <= g.z_hi)) boxk |= 1u << k;
    if (MODE == 2 && act && z == g.z_lo - 1) ringl = k;
    if (MODE == 2 && act && z == g.z_hi + 1) ringr = k;
  }
  if (PW) {
    boxk = 0xFu;
    ringl = ringr = -1;
  }
  const bool recon_on = MODE == 2 && do_recon;
  const double pulse_t = __ldg(g.pulse + t);
  const float* Ec = (RHO ? m.Erf : m.Edf) + (size_t)sg.b * N2;
  const float* be = opaque(Ec + zc);
  QLane QL{};
  if constexpr (RHO) QL = q_lane(m, g, sg.b, zc, z0, l, z4, on);
  const float* U1 = MODE == 1 ? F : utm1;
  auto issue = [&](int k, int i, int sl) {  // item i of the group's k-th shot
    if (k >= sg.n) return;
    const size_t fo = (size_t)(sg.lu0 + k) * N2;
    const int ru = x0 - 1 + i;  // u[t-1] row
    const bool oku = ru >= 0 && ru < nx && (MODE == 1 || (ru >= g.x_lo - 1 && ru <= g.x_hi + 1));
    const int ou = oku ? ru * nz : 0;
    cp16(&ring.u1[sl][tid], U1 + fo + zc + ou, oku && act);
    cp4(&ring.edge[sl][tid], U1 + fo + ze + ou, oku && has_edge);
    const int rx = x0 + i - 2;
    const bool okx = i >= 2 && rx < x1;
    if constexpr (RHO) {
      const bool okq = ru >= 0 && ru < nx;
      issue_q(ring.fr.r, QL, tid, sl, okq ? ru : 0, okq, act, nz);
    }
    if (i >= 2) {
      const int ox = okx ? rx * nz : 0;
      cp16(&ring.lam[sl][tid], lam_t + fo + zc + ox, okx && act);
      if (recon_on) {
        cp16(&ring.ut[sl][tid], ut + fo + zc + ox, okx && act);
        cp16(&ring.e[sl][tid], be + ox, okx && act);
      }
    }
  };
  double acc[kImgTX][4];
#pragma unroll
  for (int r = 0; r < kImgTX; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  // prologue: items 0 .. NSL-2 of shot 0
#pragma unroll
  for (int i = 0; i < NSL - 1; ++i) {
    issue(0, i, i);
    cp_commit();
  }
  // FX[s]: x face above the u[t-1] row of slot s; qp / qpe: q of the previous item's row
  double W[3][4], Eg[3], FX[3][4], qp[4] = {0.0, 0.0, 0.0, 0.0}, qpe = 0.0;
  for (int k = 0; k < sg.n; ++k) {
    const int lu = sg.lu0 + k;
    const int s = (unit_begin + lu) % g.S;
    const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
    const int tk = (act && txz >= z4 && txz < z4 + 4) ? txz - z4 : -1;
    float* uo = ut + (size_t)lu * N2 + zc;
    const float* st = MODE == 2 ? strip_tm2 + (size_t)lu * g.SL : nullptr;
#pragma unroll
    for (int i = 0; i < kImgItems; ++i) {
      const int sl = i % NSL, wi = i % 3;
      // keep NSL-1 items in flight: item i+NSL-1 of this shot or of the next one
      if (i + NSL - 1 < kImgItems) issue(k, i + NSL - 1, (i + NSL - 1) % NSL);
      else issue(k + 1, i + NSL - 1 - kImgItems, (i + NSL - 1) % NSL);
      cp_commit();
      cp_wait<NSL - 1>();
      {
        const float4 f = ring.u1[sl][tid];
        W[wi][0] = f.x; W[wi][1] = f.y; W[wi][2] = f.z; W[wi][3] = f.w;
        Eg[wi] = (double)ring.edge[sl][tid];
      }
      double fz[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // z faces of row x0+i-2
      if constexpr (RHO) {
        const int ru = x0 - 1 + i;
        double qn[4], qen;
        read_q(ring.fr.r, tid, sl, qn, qen);
        if (ru == 0) {  // outer face above row 0
#pragma unroll
          for (int c = 0; c < 4; ++c) qp[c] = qn[c];
          qpe = qen;
        }
        if (ru >= nx) {  // outer face below row nx-1
#pragma unroll
          for (int c = 0; c < 4; ++c) qn[c] = qp[c];
          qen = qpe;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) FX[wi][c] = face(qp[c], qn[c]);
        if (i >= 2) zfaces(QL, l, qp, qpe, fz);  // warp-uniform
#pragma unroll
        for (int c = 0; c < 4; ++c) qp[c] = qn[c];
        qpe = qen;
      }
      if (i < 2) continue;
      const int r = i - 2;
      const int x = x0 + r;
      const int im = (i + 1) % 3, ic = (i + 2) % 3, ip = i % 3;  // rows x-1, x, x+1
      double zl = __shfl_up_sync(0xffffffffu, W[ic][3], 1, kLS);
      double zr = __shfl_down_sync(0xffffffffu, W[ic][0], 1, kLS);
      if (l == 0) zl = Eg[ic];
      if (l == kLS - 1) zr = Eg[ic];
      if (x >= x1) continue;  // warp-uniform (last row block)
      const float4 lf = ring.lam[sl][tid];
      const double lam[4] = {lf.x, lf.y, lf.z, lf.w};
      double lapu[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double zm = c == 0 ? zl : W[ic][c - 1];
        const double zp = c == 3 ? zr : W[ic][c + 1];
        if constexpr (RHO)
          lapu[c] = lapf(W[ic][c], W[im][c], W[ip][c], zm, zp, FX[ic][c], FX[ip][c], fz[c],
                         fz[c + 1]);
        else
          lapu[c] = lap5(W[ic][c], W[im][c], W[ip][c], zm, zp);
        if (boxk & (1u << c)) acc[r][c] = __fma_rn(lapu[c], lam[c], acc[r][c]);
      }
      if (recon_on && act) {
        const float4 uf = ring.ut[sl][tid];
        const float4 ef = ring.e[sl][tid];
        const double ua[4] = {uf.x, uf.y, uf.z, uf.w};
        const double ed[4] = {ef.x, ef.y, ef.z, ef.w};
        float o[4] = {uf.x, uf.y, uf.z, uf.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (boxk & (1u << c)) {
            double prev = recon(W[ic][c], ua[c], ed[c], lapu[c]);
            if (x == txx && c == tk) prev = __dadd_rn(prev, pulse_t);
            o[c] = (float)prev;
          }
          if (c == ringl) o[c] = __ldg(st + 2 * g.Lz + x - g.x_lo);
          if (c == ringr) o[c] = __ldg(st + 2 * g.Lz + g.Lx + x - g.x_lo);
        }
        *reinterpret_cast<float4*>(uo + x * nz) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    if (recon_on && act) {  // ring rows of u[t-2]
      if (x0 == g.x_lo && g.x_lo > 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (boxk & (1u << c)) uo[(g.x_lo - 1) * nz + c] = __ldg(st + z4 + c - g.z_lo);
      }
      if (x1 == g.x_hi + 1 && g.x_hi + 1 < nx) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (boxk & (1u << c)) uo[(g.x_hi + 1) * nz + c] = __ldg(st + g.Lz + z4 + c - g.z_lo);
      }
    }
  }
  cp_wait<0>();
  if (act) {
    double* dst = acc_part + (size_t)blockIdx.z * N2 + zc;
#pragma unroll
    for (int r = 0; r < kImgTX; ++r) {
      if (x0 + r >= x1) break;
      double2* p = reinterpret_cast<double2*>(dst + (x0 + r) * nz);
      double2 a = p[0], b = p[1];
      a.x += acc[r][0]; a.y += acc[r][1]; b.x += acc[r][2]; b.y += acc[r][3];
      p[0] = a;
      p[1] = b;
    }
  }
}

template <int MODE, bool RHO>
__global__ void __launch_bounds__(kLeanT, RHO ? kLeanMinBRho : kLeanMinB)
    img_lean_kernel(Geo g, Model m, int t, int unit_begin, int U, int gs,
                    const float* __restrict__ lam_t, const float* __restrict__ F, float* ut,
                    const float* __restrict__ utm1, const float* __restrict__ strip_tm2,
                    double* __restrict__ acc_part, int do_recon) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = lane % kLS;
  const int z4 = blockIdx.x * kSW + 4 * l;
  const int rlo = MODE == 2 ? g.x_lo : 0, rhi = MODE == 2 ? g.x_hi + 1 : g.nx;
  const int x0 = rlo + ((blockIdx.y * kLeanWarps + warp) * kSPW + lane / kLS) * kImgTX;
  const bool plain = x0 < rhi && (MODE == 1 ? z4 < g.nz : (z4 >= g.z_lo && z4 + 3 <= g.z_hi));
  if (__all_sync(0xffffffffu, plain))
    img_lean_body<MODE, RHO, true>(g, m, t, unit_begin, U, gs, lam_t, F, ut, utm1, strip_tm2,
                                   acc_part, do_recon);
  else
    img_lean_body<MODE, RHO, false>(g, m, t, unit_begin, U, gs, lam_t, F, ut, utm1, strip_tm2,
                                    acc_part, do_recon);
}

}  // namespace dufwi
