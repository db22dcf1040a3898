// Stepwise engine, constant density: the adjoint step as ONE streaming kernel.
//
// The split adjoint (dufwi_lean_kernels.cuh) writes lam[t] in adjlam_lean_kernel
// and reads it back in img_lean_kernel: 4 B of DRAM per cell update that this
// kernel saves.  A lane group owns kImgTX rows x a 64-wide z strip of the WHOLE
// grid (the lam update covers the PML too) and walks its shot group as the
// imaging kernel does, one stream of ring items (kImgTX + 2 per shot).  Item i
// of a shot carries row x0-1+i of lam[t+1] and E (and of u[t-1] inside the
// imaging rows) and, for i >= 2, row x = x0+i-2 of lam[t+2] and u[t].  Per row x:
//   lam[t]  = A lam1 + L(E lam1) + B lam2 (+ residual), stored in place over lam[t+2]
//   acc    += L(u[t-1]) * lam[t]          (lam[t] rounded to f32 first, as the split
//                                           path reads it back: same bits)
//   u[t-2]  = 2 u[t-1] + E L(u[t-1]) - u[t] (+ source)   (MODE 2, box cells)
// The f64 operations and their order are those of adjlam_lean_rows and
// img_lean_body, so the outputs are bit-identical to the split path.
// DRAM per cell update: MODE 2 read lam[t+1], lam[t+2], u[t-1], u[t], write
// lam[t], u[t-2] = 24 B (split: 28 B); + 16 B / gs for the accumulator.
// Halo rows of lam[t+1], E and u[t-1] (6 rows per 4) come from L1/L2.
#pragma once

#include "dufwi_lean_kernels.cuh"

namespace dufwi {

struct FusedAdjRing {
  float4 l1[kNSL][kLeanT];   // lam[t+1] row x0-1+i
  float4 e[kNSL][kLeanT];    // E row x0-1+i (f32 copy)
  float4 u1[kNSL][kLeanT];   // u[t-1] row x0-1+i (imaging rows)
  float4 l2[kNSL][kLeanT];   // lam[t+2] row x0+i-2
  float4 ut[kNSL][kLeanT];   // u[t] row x0+i-2 (MODE 2 reconstruction)
  float edl[kNSL][kLeanT];   // lam[t+1] at the lane's edge column
  float ede[kNSL][kLeanT];   // E at the lane's edge column
  float edu[kNSL][kLeanT];   // u[t-1] at the lane's edge column
  double2 acc[kImgTX][2][kLeanT];  // the lane's imaging sums over the shot group
};

// PW: every cell of the warp lies in the box (columns and rows): no damping,
// no ring columns, every row images.  ZD: some lane touches the z damping band.
template <int MODE, bool PW, bool ZD>
__device__ __forceinline__ void adjimg_body(const Geo& g, const Model& m, const ABTables& T, int t,
                                            int unit_begin, int U, int gs,
                                            const float* __restrict__ l1b, float* l2b,
                                            const double* __restrict__ rres_t, int has1, int has2,
                                            const float* __restrict__ F, float* ut,
                                            const float* __restrict__ utm1,
                                            const float* __restrict__ strip_tm2,
                                            double* __restrict__ acc_part, int do_recon) {
  constexpr int NSL = kNSL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& ring = *reinterpret_cast<FusedAdjRing*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nz = g.nz, nx = g.nx;
  const int l = lane % kLS;
  const int z0 = blockIdx.x * kSW;
  const int x0 = ((blockIdx.y * kLeanWarps + warp) * kSPW + lane / kLS) * kImgTX;
  const bool on = x0 < nx;
  if (!__any_sync(0xffffffffu, on)) return;  // warp-uniform
  const int x1 = on ? min(nx, x0 + kImgTX) : x0;
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  const size_t N2 = (size_t)nx * nz;
  const int z4 = z0 + 4 * l;
  const bool act = PW || (on && z4 < nz);
  const int zc = act ? z4 : 0;
  const bool edge_l = on && l == 0 && z0 > 0, edge_r = on && l == kLS - 1 && z0 + kSW < nz;
  const bool has_edge = edge_l || edge_r;
  const int ze = edge_l ? z0 - 1 : edge_r ? z0 + kSW : 0;
  // imaging rows [ilo, ihi]; u[t-1] is read on [ilo-1, ihi+1] (MODE 2: the box and its ring)
  const int ilo = MODE == 2 ? g.x_lo : 0, ihi = MODE == 2 ? g.x_hi : nx - 1;
  unsigned boxk = 0u, rxk = 0u;
  int ringl = -1, ringr = -1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int z = z4 + k;
    if (act) {
      if (MODE == 1 || (z >= g.z_lo && z <= g.z_hi)) boxk |= 1u << k;
      if (MODE == 2 && z == g.z_lo - 1) ringl = k;
      if (MODE == 2 && z == g.z_hi + 1) ringr = k;
      if (__ldg(g.col_flag + z)) rxk |= 1u << k;
    }
  }
  if (PW) {
    boxk = 0xFu;
    ringl = ringr = -1;
  }
  const bool wrx = __any_sync(0xffffffffu, rxk != 0u);
  const bool do_img = t >= 1;
  const bool recon_on = MODE == 2 && do_recon;
  const double pulse_t = __ldg(g.pulse + t);
  const float* Ec = m.Edf + (size_t)sg.b * N2;
  const float* be = opaque(Ec + zc);
  const float* bel = opaque(Ec + ze);
  const float* U1 = MODE == 1 ? F : utm1;
  auto issue = [&](int k, int i, int sl) {  // item i of the group's k-th shot
    if (k >= sg.n) return;
    const size_t fo = (size_t)(sg.lu0 + k) * N2;
    const int ru = x0 - 1 + i;
    const bool okr = ru >= 0 && ru < nx;
    const int orr = okr ? ru * nz : 0;
    cp16(&ring.l1[sl][tid], l1b + fo + zc + orr, has1 && okr && act);
    cp4(&ring.edl[sl][tid], l1b + fo + ze + orr, has1 && okr && has_edge);
    cp16(&ring.e[sl][tid], be + orr, okr && act);
    cp4(&ring.ede[sl][tid], bel + orr, okr && has_edge);
    const bool oku = do_img && okr && ru >= ilo - 1 && ru <= ihi + 1;
    cp16(&ring.u1[sl][tid], U1 + fo + zc + orr, oku && act);
    cp4(&ring.edu[sl][tid], U1 + fo + ze + orr, oku && has_edge);
    if (i >= 2) {
      const int rx = x0 + i - 2;
      const bool okx = rx < x1;
      const int ox = okx ? rx * nz : 0;
      cp16(&ring.l2[sl][tid], l2b + fo + zc + ox, has2 && okx && act);
      if (recon_on)
        cp16(&ring.ut[sl][tid], ut + fo + zc + ox, okx && act && rx >= ilo && rx <= ihi);
    }
  };
  // imaging sums in shared memory (registers would spill at 168)
#pragma unroll
  for (int r = 0; r < kImgTX; ++r) ring.acc[r][0][tid] = ring.acc[r][1][tid] = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < NSL - 1; ++i) {
    issue(0, i, i);
    cp_commit();
  }
  // windows over rows x-1, x, x+1: u[t-1] (W, edge Eg), E lam[t+1] (EL, edge EG),
  // raw lam[t+1] (RL) and E (EW) as loaded
  double W[3][4], Eg[3], EL[3][4], EG[3];
  float4 RL[3], EW[3];
  for (int k = 0; k < sg.n; ++k) {
    const int lu = sg.lu0 + k;
    const int s = (unit_begin + lu) % g.S;
    const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
    const int tk = (act && txz >= z4 && txz < z4 + 4) ? txz - z4 : -1;
    float* uo = ut + (size_t)lu * N2 + zc;
    float* lo = l2b + (size_t)lu * N2 + zc;
    const float* st = MODE == 2 ? strip_tm2 + (size_t)lu * g.SL : nullptr;
    const double* rr = rres_t + (size_t)lu * g.M;
#pragma unroll
    for (int i = 0; i < kImgItems; ++i) {
      const int sl = i % NSL, wi = i % 3;
      if (i + NSL - 1 < kImgItems) issue(k, i + NSL - 1, (i + NSL - 1) % NSL);
      else issue(k + 1, i + NSL - 1 - kImgItems, (i + NSL - 1) % NSL);
      cp_commit();
      cp_wait<NSL - 1>();
      {
        const float4 f = ring.l1[sl][tid];
        const float4 a = ring.e[sl][tid];
        RL[wi] = f;
        EW[wi] = a;
        EL[wi][0] = __dmul_rn(a.x, f.x);
        EL[wi][1] = __dmul_rn(a.y, f.y);
        EL[wi][2] = __dmul_rn(a.z, f.z);
        EL[wi][3] = __dmul_rn(a.w, f.w);
        EG[wi] = __dmul_rn((double)ring.ede[sl][tid], (double)ring.edl[sl][tid]);
        if (do_img) {
          const float4 u = ring.u1[sl][tid];
          W[wi][0] = u.x; W[wi][1] = u.y; W[wi][2] = u.z; W[wi][3] = u.w;
          Eg[wi] = (double)ring.edu[sl][tid];
        }
      }
      if (i < 2) continue;
      const int r = i - 2;
      const int x = x0 + r;
      const int im = (i + 1) % 3, ic = (i + 2) % 3, ip = i % 3;  // rows x-1, x, x+1
      double zl = __shfl_up_sync(0xffffffffu, EL[ic][3], 1, kLS);
      double zr = __shfl_down_sync(0xffffffffu, EL[ic][0], 1, kLS);
      if (l == 0) zl = EG[ic];
      if (l == kLS - 1) zr = EG[ic];
      double wl = 0.0, wr = 0.0;
      if (do_img) {  // launch-uniform
        wl = __shfl_up_sync(0xffffffffu, W[ic][3], 1, kLS);
        wr = __shfl_down_sync(0xffffffffu, W[ic][0], 1, kLS);
        if (l == 0) wl = Eg[ic];
        if (l == kLS - 1) wr = Eg[ic];
      }
      if (x >= x1) continue;  // the grid's last row block
      // ---- lam[t] row x (adjlam_lean_rows)
      const float4 w2 = ring.l2[sl][tid];
      const double l2v[4] = {w2.x, w2.y, w2.z, w2.w};
      const double rl[4] = {RL[ic].x, RL[ic].y, RL[ic].z, RL[ic].w};
      double lam[4];
      {
        double adj[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double zm = c == 0 ? zl : EL[ic][c - 1];
          const double zp = c == 3 ? zr : EL[ic][c + 1];
          adj[c] = lap5(EL[ic][c], EL[im][c], EL[ip][c], zm, zp);
        }
        if (PW || (x >= g.x_lo && x <= g.x_hi)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (ZD) {  // undamped row: D = pz[z], (A, B) of the z band (L1-resident tables)
              const int z = min(z4 + c, nz - 1);
              lam[c] = adj_update(__ldg(T.Az + z), __ldg(T.Bz + z), rl[c], l2v[c], adj[c]);
            } else {
              lam[c] = adj_update_free(rl[c], l2v[c], adj[c]);
            }
          }
        } else {
          const double pxx = __ldg(T.px + x), Axx = __ldg(T.Ax + x), Bxx = __ldg(T.Bx + x);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double2 ab = ab_row_damped(T, pxx, Axx, Bxx, min(z4 + c, nz - 1));
            lam[c] = adj_update(ab.x, ab.y, rl[c], l2v[c], adj[c]);
          }
        }
      }
      if (!act) continue;
      const int orow = x * nz;
      if (wrx && rxk && __ldg(g.row_flag + x)) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (rxk & (1u << c)) {
            const int slot = __ldg(g.node_slot + orow + z4 + c);
            if (slot >= 0) lam[c] = __dadd_rn(lam[c], __ldg(rr + slot));
          }
      }
      const float4 lf = make_float4((float)lam[0], (float)lam[1], (float)lam[2], (float)lam[3]);
      *reinterpret_cast<float4*>(lo + orow) = lf;
      if (!do_img) continue;
      // ---- imaging and reconstruction of row x (img_lean_body)
      if (PW || (x >= ilo && x <= ihi)) {
        const double lm[4] = {lf.x, lf.y, lf.z, lf.w};
        const double* wc = W[ic];
        double lapu[4];
        double2 a0 = ring.acc[r][0][tid], a1 = ring.acc[r][1][tid];
        double acc[4] = {a0.x, a0.y, a1.x, a1.y};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double zm = c == 0 ? wl : wc[c - 1];
          const double zp = c == 3 ? wr : wc[c + 1];
          lapu[c] = lap5(wc[c], W[im][c], W[ip][c], zm, zp);
          if (boxk & (1u << c)) acc[c] = __fma_rn(lapu[c], lm[c], acc[c]);
        }
        ring.acc[r][0][tid] = make_double2(acc[0], acc[1]);
        ring.acc[r][1][tid] = make_double2(acc[2], acc[3]);
        if (recon_on) {
          const float4 uf = ring.ut[sl][tid];
          const double ua[4] = {uf.x, uf.y, uf.z, uf.w};
          const double ed[4] = {EW[ic].x, EW[ic].y, EW[ic].z, EW[ic].w};
          float o[4] = {uf.x, uf.y, uf.z, uf.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (boxk & (1u << c)) {
              double prev = recon(wc[c], ua[c], ed[c], lapu[c]);
              if (x == txx && c == tk) prev = __dadd_rn(prev, pulse_t);
              o[c] = (float)prev;
            }
            if (c == ringl) o[c] = __ldg(st + 2 * g.Lz + x - g.x_lo);
            if (c == ringr) o[c] = __ldg(st + 2 * g.Lz + g.Lx + x - g.x_lo);
          }
          *reinterpret_cast<float4*>(uo + orow) = make_float4(o[0], o[1], o[2], o[3]);
        }
      } else if (!PW && recon_on && boxk && (x == g.x_lo - 1 || x == g.x_hi + 1)) {
        // ring rows of u[t-2], box columns
        const float* sr = st + (x == g.x_lo - 1 ? 0 : g.Lz) + z4 - g.z_lo;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (boxk & (1u << c)) uo[orow + c] = __ldg(sr + c);
      }
    }
  }
  cp_wait<0>();
  if (act && do_img) {
    double* dst = acc_part + (size_t)blockIdx.z * N2 + zc;
#pragma unroll
    for (int r = 0; r < kImgTX; ++r) {
      const int x = x0 + r;
      if (x >= x1) break;
      if (!PW && (x < ilo || x > ihi)) continue;
      double2* p = reinterpret_cast<double2*>(dst + x * nz);
      double2 a = p[0], b = p[1];
      const double2 s0 = ring.acc[r][0][tid], s1 = ring.acc[r][1][tid];
      a.x += s0.x; a.y += s0.y; b.x += s1.x; b.y += s1.y;
      p[0] = a;
      p[1] = b;
    }
  }
}

// MINB: resident CTAs per SM (register cap 168 at 3, 255 at 2)
template <int MODE, int MINB>
__global__ void __launch_bounds__(kLeanT, MINB)
    adjimg_lean_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int U, int gs,
                       const float* __restrict__ l1, float* l2o, const double* __restrict__ rres_t,
                       int has1, int has2, const float* __restrict__ F, float* ut,
                       const float* __restrict__ utm1, const float* __restrict__ strip_tm2,
                       double* __restrict__ acc_part, int do_recon) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = lane % kLS;
  const int z4 = blockIdx.x * kSW + 4 * l;
  const int x0 = ((blockIdx.y * kLeanWarps + warp) * kSPW + lane / kLS) * kImgTX;
  const bool plain = x0 >= g.x_lo && x0 + kImgTX - 1 <= g.x_hi && z4 >= g.z_lo &&
                     z4 + 3 <= g.z_hi;
  bool zd = false;
  if (z4 < g.nz)
#pragma unroll
    for (int k = 0; k < 4; ++k) zd |= __ldg(T.pz + min(z4 + k, g.nz - 1)) != 0.0;
#define DUFWI_ADJIMG(PW, ZD)                                                                     \
  adjimg_body<MODE, PW, ZD>(g, m, T, t, unit_begin, U, gs, l1, l2o, rres_t, has1, has2, F, ut,  \
                            utm1, strip_tm2, acc_part, do_recon)
  if (__all_sync(0xffffffffu, plain)) DUFWI_ADJIMG(true, false);
  else if (__any_sync(0xffffffffu, zd)) DUFWI_ADJIMG(false, true);
  else DUFWI_ADJIMG(false, false);
#undef DUFWI_ADJIMG
}

}  // namespace dufwi
