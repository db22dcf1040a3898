// Stepwise engine, f32 tile kernels (DUFWI_ARITH_F32): one launch per time
// step, TMA-staged stencil tiles.
//
// A CTA owns one kTX x kTZ tile of the grid.  One thread issues
// cp.async.bulk.tensor loads of the tile's operands into shared memory — the
// stencil operand with its 1-cell halo as a (kTX+2) x (kTZ+8) box (4 columns
// either side keep every box row a multiple of 16 bytes), the others as plain
// kTX x kTZ boxes — and the copies complete on an mbarrier.  The tensor maps
// are 4-D over a workspace region, [slot][unit][x][z], so the same map serves
// every step, unit and ping-pong slot; out-of-grid elements are zero-filled by
// the TMA unit, which IS the reference's boundary condition (u = 0 outside,
// forward.py:211-223), so the stencil carries no boundary predicates and no
// per-lane address arithmetic.  Latency is hidden across CTAs (3-8 resident
// per SM), not inside one.
//
// Threads: 16 lanes x 4 cells cover a tile row (float4 shared loads and global
// stores), a thread walks kTRPT consecutive rows with a 3-row register window.
// A tile is classified once per CTA: tiles inside the undamped box run the
// branch-free body (no damping terms, no ring strips); border tiles pick
// (A-2, B+1) per cell from the separable ramps.  Receiver sampling only in
// tiles the plan flags as holding receiver nodes.
//
// Arithmetic: f32 increment form (dufwi_common.cuh).  Variable density
// (SURVEY §0.1 G3): D(u)_c = sum_j f_cj (u_j - u_c), f_cj = h_c + h_j with
// h = q/2 streamed from a replicate-padded map ([nx+2][nz+8], so outer faces
// are f = q_c as in the oracle's rho_face_weights); forward u += Er D(u1),
// adjoint lam += D(Er l1), imaging sums D(u) lam (scaled by rho in
// reduce_groups), as in the lean kernels.
//
// DRAM per cell update: forward 12 B, lam update 12 B, imaging +
// reconstruction 16 B (+16 B / gs accumulator); coefficient tiles come from L2
// and, in the imaging kernel, are loaded once per shot group.
#pragma once

#include <cuda.h>

#include "dufwi_cluster_kernels.cuh"  // mbarrier helpers
#include "dufwi_step_kernels.cuh"     // ShotGroup

namespace dufwi {

constexpr int kTZ = 64;                 // tile columns
constexpr int kTX = 32;                 // tile rows
constexpr int kTHZ = kTZ + 8;           // halo'd tile row length (floats)
constexpr int kTHX = kTX + 2;           // halo'd tile rows
constexpr int kTRPT = 4;                // rows per thread
constexpr int kTLanes = kTZ / 4;        // lanes per tile row
constexpr int kTT = kTLanes * (kTX / kTRPT);  // threads per CTA
constexpr uint32_t kHaloBytes = kTHX * kTHZ * 4;
constexpr uint32_t kPlainBytes = kTX * kTZ * 4;
constexpr uint32_t kHaloSlot = (kHaloBytes + 127) / 128 * 128;  // shared-memory slot sizes
constexpr uint32_t kPlainSlot = kPlainBytes;
static_assert(kTX % kTRPT == 0 && kPlainBytes % 128 == 0, "tile shape");

// f32 tables of the separable damping for the increment form: ramps and the
// pairs (A - 2, B + 1) along x and z.
struct TileTabs {
  const float *px, *pz, *a2x, *b1x, *a2z, *b1z;
  const unsigned char* tile_rx;  // [tiles_x][tiles_z]: the tile holds a receiver node
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                            int c2, int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tile_bar_init(uint32_t bar, int n) {
  for (int i = 0; i < n; ++i) mbar_init(bar + 8u * i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  fence_proxy_async();
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

struct F4 {
  float v[4];
  __device__ __forceinline__ F4() {}
  __device__ __forceinline__ F4(const float4& a) { v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; }
};

// Per-thread view of a tile: lane l covers columns z4 .. z4+3, rows xb .. xb+kTRPT-1.
struct TileThread {
  int l, rg, z0, x0, z4, xb, r0;
  bool zact;
};
__device__ __forceinline__ TileThread tile_thread(const Geo& g, int z0, int x0) {
  TileThread t;
  t.l = threadIdx.x % kTLanes;
  t.rg = threadIdx.x / kTLanes;
  t.z0 = z0;
  t.x0 = x0;
  t.z4 = z0 + 4 * t.l;
  t.r0 = t.rg * kTRPT;
  t.xb = x0 + t.r0;
  t.zact = t.z4 < g.nz;
  return t;
}

// The tile lies inside the undamped box: no damping terms, no ring cells.
__device__ __forceinline__ bool tile_in_box(const Geo& g, int z0, int x0) {
  return x0 >= g.x_lo && x0 + kTX - 1 <= g.x_hi && z0 >= g.z_lo && z0 + kTZ - 1 <= g.z_hi;
}

// (A - 2, B + 1) per lane cell along z, and the ramp values for the x/z choice.
struct LanePml {
  float pz[4], a2[4], b1[4];
};
__device__ __forceinline__ LanePml lane_pml(const Geo& g, const TileTabs& T, int z4) {
  LanePml P;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int z = min(z4 + k, g.nz - 1);
    P.pz[k] = __ldg(T.pz + z);
    P.a2[k] = __ldg(T.a2z + z);
    P.b1[k] = __ldg(T.b1z + z);
  }
  return P;
}

// Face factors of a thread's row from the h = q/2 window (hm, hc, hp: rows
// x-1, x, x+1; hzl / hzr: the row's z neighbours of the lane's 4 cells).
struct Faces {
  float xm[4], xp[4], z[5];
};
__device__ __forceinline__ void faces_row(const F4& hc, const F4& hp, float hzl, float hzr,
                                          Faces& f) {
#pragma unroll
  for (int k = 0; k < 4; ++k) f.xp[k] = __fadd_rn(hc.v[k], hp.v[k]);
  f.z[0] = __fadd_rn(hzl, hc.v[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) f.z[k] = __fadd_rn(hc.v[k - 1], hc.v[k]);
  f.z[4] = __fadd_rn(hc.v[3], hzr);
}

// L(w) (RHO: D(w)) of the lane's 4 cells of the centre row.
template <bool RHO>
__device__ __forceinline__ void stencil_row(const F4& wm, const F4& wc, const F4& wp, float zl,
                                            float zr, const Faces& f, float (&out)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float c = wc.v[k];
    const float zm = k == 0 ? zl : wc.v[k - 1];
    const float zp = k == 3 ? zr : wc.v[k + 1];
    if (RHO) {
      const float a = __fmul_rn(f.xm[k], __fsub_rn(wm.v[k], c));
      const float b = __fmaf_rn(f.xp[k], __fsub_rn(wp.v[k], c), a);
      const float d = __fmaf_rn(f.z[k], __fsub_rn(zm, c), b);
      out[k] = __fmaf_rn(f.z[k + 1], __fsub_rn(zp, c), d);
    } else {
      out[k] = lap5f(c, wm.v[k], wp.v[k], zm, zp);
    }
  }
}

// Density window of a thread: h rows x-1 and x and the x face between them.
template <bool RHO>
struct HWin {
  F4 hc;
  Faces f;
  const float* ph;
  __device__ __forceinline__ void init(const float* sH, const TileThread& t) {
    if (RHO) {
      ph = sH + t.r0 * kTHZ + 4 + 4 * t.l;
      const F4 hm(lds4(ph));
      hc = F4(lds4(ph + kTHZ));
#pragma unroll
      for (int k = 0; k < 4; ++k) f.xm[k] = __fadd_rn(hm.v[k], hc.v[k]);
    }
  }
  // faces of row j (centre row r0 + j), then advance the window
  __device__ __forceinline__ void row(int j) {
    if (RHO) {
      const float* hr = ph + (j + 1) * kTHZ;
      const F4 hp(lds4(hr + kTHZ));
      faces_row(hc, hp, hr[-1], hr[4], f);
      hc = hp;
    }
  }
  __device__ __forceinline__ void next() {
    if (RHO) {
#pragma unroll
      for (int k = 0; k < 4; ++k) f.xm[k] = f.xp[k];
    }
  }
};

// ----------------------------------------------------------------- forward
// u[t] = u1 + ((u1 - u2) + damping terms + E L(u1)) (+ source), forward.py:301-308.
struct TileFwdSmem {
  static constexpr uint32_t u1 = 0, u2 = kHaloSlot, e = u2 + kPlainSlot, h = e + kPlainSlot;
  __host__ __device__ static constexpr uint32_t bar(bool rho) { return h + (rho ? kHaloSlot : 0u); }
  __host__ __device__ static constexpr uint32_t bytes(bool rho) { return bar(rho) + 16u; }
};

template <bool RHO, int MODE, bool PML, bool RX>
__device__ __forceinline__ void tile_fwd_compute(const Geo& g, const TileTabs& T,
                                                 const TileThread& t, const float* sU1,
                                                 const float* sU2, const float* sE, const float* sH,
                                                 int lu, int txx, int txz, float pulse_t,
                                                 float* __restrict__ uo, float* __restrict__ rec_t,
                                                 float* __restrict__ strip_t) {
  const int nz = g.nz, nx = g.nx;
  const float* pu = sU1 + t.r0 * kTHZ + 4 + 4 * t.l;  // halo row r0 = grid row xb - 1
  F4 wm(lds4(pu)), wc(lds4(pu + kTHZ));
  HWin<RHO> H;
  H.init(sH, t);
  LanePml P;
  if (PML) P = lane_pml(g, T, t.z4);
  unsigned rxk = 0u, boxk = 0u;
  int ringl = -1, ringr = -1;
  if (t.zact) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int z = t.z4 + k;
      if (RX && __ldg(g.col_flag + z)) rxk |= 1u << k;
      if (MODE == 2 && PML) {
        if (z >= g.z_lo && z <= g.z_hi) boxk |= 1u << k;
        if (z == g.z_lo - 1) ringl = k;
        if (z == g.z_hi + 1) ringr = k;
      }
    }
  }
  const int tk = (txz >= t.z4 && txz < t.z4 + 4) ? txz - t.z4 : -1;
#pragma unroll
  for (int j = 0; j < kTRPT; ++j) {
    const int x = t.xb + j;
    const float* pr = pu + (j + 1) * kTHZ;
    const F4 wp(lds4(pr + kTHZ));
    const float zl = pr[-1], zr = pr[4];
    const F4 w2(lds4(sU2 + (t.r0 + j) * kTZ + 4 * t.l));
    const F4 e4(lds4(sE + (t.r0 + j) * kTZ + 4 * t.l));
    H.row(j);
    float lap[4], v[4];
    stencil_row<RHO>(wm, wc, wp, zl, zr, H.f, lap);
    if (PML) {
      const int xx = min(x, nx - 1);
      const float pxx = __ldg(T.px + xx), a2x = __ldg(T.a2x + xx), b1x = __ldg(T.b1x + xx);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ux = pxx >= P.pz[k];
        v[k] = inc_update(ux ? a2x : P.a2[k], ux ? b1x : P.b1[k], wc.v[k], w2.v[k], e4.v[k], lap[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = inc_update_free(wc.v[k], w2.v[k], e4.v[k], lap[k]);
    }
    if (x == txx && tk >= 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k == tk) v[k] = __fadd_rn(v[k], pulse_t);
    }
    if (t.zact && x < nx) {
      const int orow = x * nz;
      *reinterpret_cast<float4*>(uo + orow + t.z4) = make_float4(v[0], v[1], v[2], v[3]);
      if (RX && rxk && __ldg(g.row_flag + x)) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rxk & (1u << k)) {
            const int slot = __ldg(g.node_slot + orow + t.z4 + k);
            if (slot >= 0) rec_t[(size_t)lu * g.M + slot] = v[k];
          }
      }
      if (MODE == 2 && PML) {  // ring cells lie outside the box: border tiles only
        float* st = strip_t + (size_t)lu * g.SL;
        if (x == g.x_lo - 1 || x == g.x_hi + 1) {
          const int base = (x == g.x_lo - 1 ? 0 : g.Lz) - g.z_lo + t.z4;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (boxk & (1u << k)) st[base + k] = v[k];
        } else if (x >= g.x_lo && x <= g.x_hi) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k == ringl) st[2 * g.Lz + x - g.x_lo] = v[k];
            if (k == ringr) st[2 * g.Lz + g.Lx + x - g.x_lo] = v[k];
          }
        }
      }
    }
    wm = wc;
    wc = wp;
    H.next();
  }
}

// Zero a shared-memory slot whose operand does not exist yet (t < 2 / the
// adjoint's first steps): the stencil reads zeros, like the reference's initial state.
__device__ __forceinline__ void zero_slot(float* s, uint32_t bytes) {
  for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<float4*>(s)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// mU1: halo'd boxes of the region holding u[t-1] (slot s1), mU2: plain boxes
// of the region holding u[t-2] (slot s2); uo: where u[t] goes (unit 0 of its slot).
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kTT)
    tile_fwd_kernel(const __grid_constant__ CUtensorMap mU1, const __grid_constant__ CUtensorMap mU2,
                    const __grid_constant__ CUtensorMap mE, const __grid_constant__ CUtensorMap mH,
                    Geo g, TileTabs T, int t, int unit_begin, int s1, int s2, int has1, int has2,
                    float* __restrict__ uo, float* __restrict__ rec_t,
                    float* __restrict__ strip_t) {
  extern __shared__ __align__(128) unsigned char tsm[];
  float* sU1 = reinterpret_cast<float*>(tsm + TileFwdSmem::u1);
  float* sU2 = reinterpret_cast<float*>(tsm + TileFwdSmem::u2);
  float* sE = reinterpret_cast<float*>(tsm + TileFwdSmem::e);
  float* sH = reinterpret_cast<float*>(tsm + TileFwdSmem::h);
  const uint32_t bar = smem_addr(tsm + TileFwdSmem::bar(RHO));
  const int z0 = blockIdx.x * kTZ, x0 = blockIdx.y * kTX, lu = blockIdx.z;
  const int u = unit_begin + lu;
  const int b = u / g.S, s = u - b * g.S;
  if (threadIdx.x == 0) {
    tile_bar_init(bar, 1);
    mbar_expect_tx(bar, (has1 ? kHaloBytes : 0u) + (has2 ? kPlainBytes : 0u) + kPlainBytes +
                            (RHO ? kHaloBytes : 0u));
    if (has1) tma_load_4d(smem_addr(sU1), &mU1, z0 - 4, x0 - 1, lu, s1, bar);
    if (has2) tma_load_4d(smem_addr(sU2), &mU2, z0, x0, lu, s2, bar);
    tma_load_3d(smem_addr(sE), &mE, z0, x0, b, bar);
    if (RHO) tma_load_3d(smem_addr(sH), &mH, z0, x0, b, bar);
  }
  if (!has1) zero_slot(sU1, kHaloSlot);
  if (!has2) zero_slot(sU2, kPlainSlot);
  const TileThread tt = tile_thread(g, z0, x0);
  const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
  const float pulse_t = (float)__ldg(g.pulse + t);
  const bool pml = !tile_in_box(g, z0, x0);
  const bool rx = __ldg(T.tile_rx + blockIdx.y * gridDim.x + blockIdx.x) != 0;
  float* uu = uo + (size_t)lu * g.nx * g.nz;
  __syncthreads();  // barrier initialised (and zero fills done) before anyone waits / reads
  mbar_wait(bar, 0);
#define DUFWI_TF(P, R)                                                                          \
  tile_fwd_compute<RHO, MODE, P, R>(g, T, tt, sU1, sU2, sE, sH, lu, txx, txz, pulse_t, uu, rec_t, \
                                    strip_t)
  if (pml) {
    if (rx) DUFWI_TF(true, true); else DUFWI_TF(true, false);
  } else {
    if (rx) DUFWI_TF(false, true); else DUFWI_TF(false, false);
  }
#undef DUFWI_TF
}

// --------------------------------------------------------------- lam update
// lam[t] = l1 + ((l1 - l2) + damping terms + L^T(E l1)) (+ merged residual at
// the receiver nodes), in place over lam[t+2] (adjoint.py:119-131); RHO:
// L^T(E lam) = D(Er lam).  E (Er) is staged with its halo: the operand of the
// stencil is the product E l1.
struct TileAdjSmem {
  static constexpr uint32_t l1 = 0, e = kHaloSlot, l2 = 2 * kHaloSlot, h = l2 + kPlainSlot;
  __host__ __device__ static constexpr uint32_t bar(bool rho) { return h + (rho ? kHaloSlot : 0u); }
  __host__ __device__ static constexpr uint32_t bytes(bool rho) { return bar(rho) + 16u; }
};

__device__ __forceinline__ F4 mul4(const F4& a, const F4& b) {
  F4 r;
#pragma unroll
  for (int k = 0; k < 4; ++k) r.v[k] = __fmul_rn(a.v[k], b.v[k]);
  return r;
}

template <bool RHO, bool PML, bool RX>
__device__ __forceinline__ void tile_adj_compute(const Geo& g, const TileTabs& T,
                                                 const TileThread& t, const float* sL1,
                                                 const float* sE, const float* sL2, const float* sH,
                                                 int lu, float* __restrict__ lo,
                                                 const double* __restrict__ rres_t) {
  const int nz = g.nz, nx = g.nx;
  const int o = t.r0 * kTHZ + 4 + 4 * t.l;
  const float* pl = sL1 + o;
  const float* pe = sE + o;
  F4 elm = mul4(F4(lds4(pe)), F4(lds4(pl)));
  F4 lc(lds4(pl + kTHZ));
  F4 elc = mul4(F4(lds4(pe + kTHZ)), lc);
  HWin<RHO> H;
  H.init(sH, t);
  LanePml P;
  if (PML) P = lane_pml(g, T, t.z4);
  unsigned rxk = 0u;
  if (RX && t.zact) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (__ldg(g.col_flag + t.z4 + k)) rxk |= 1u << k;
  }
#pragma unroll
  for (int j = 0; j < kTRPT; ++j) {
    const int x = t.xb + j;
    const float* lr = pl + (j + 1) * kTHZ;
    const float* er = pe + (j + 1) * kTHZ;
    const F4 lp(lds4(lr + kTHZ));
    const F4 elp = mul4(F4(lds4(er + kTHZ)), lp);
    const float zl = __fmul_rn(er[-1], lr[-1]), zr = __fmul_rn(er[4], lr[4]);
    const F4 w2(lds4(sL2 + (t.r0 + j) * kTZ + 4 * t.l));
    H.row(j);
    float adj[4], lam[4];
    stencil_row<RHO>(elm, elc, elp, zl, zr, H.f, adj);
    if (PML) {
      const int xx = min(x, nx - 1);
      const float pxx = __ldg(T.px + xx), a2x = __ldg(T.a2x + xx), b1x = __ldg(T.b1x + xx);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ux = pxx >= P.pz[k];
        lam[k] = inc_adj(ux ? a2x : P.a2[k], ux ? b1x : P.b1[k], lc.v[k], w2.v[k], adj[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) lam[k] = inc_adj_free(lc.v[k], w2.v[k], adj[k]);
    }
    if (t.zact && x < nx) {
      const int orow = x * nz;
      if (RX && rxk && __ldg(g.row_flag + x)) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rxk & (1u << k)) {
            const int slot = __ldg(g.node_slot + orow + t.z4 + k);
            if (slot >= 0)
              lam[k] = __fadd_rn(lam[k], (float)__ldg(rres_t + (size_t)lu * g.M + slot));
          }
      }
      *reinterpret_cast<float4*>(lo + orow + t.z4) = make_float4(lam[0], lam[1], lam[2], lam[3]);
    }
    elm = elc;
    elc = elp;
    lc = lp;
    H.next();
  }
}

template <bool RHO>
__global__ void __launch_bounds__(kTT)
    tile_adj_kernel(const __grid_constant__ CUtensorMap mL1, const __grid_constant__ CUtensorMap mL2,
                    const __grid_constant__ CUtensorMap mEh, const __grid_constant__ CUtensorMap mH,
                    Geo g, TileTabs T, int unit_begin, int s1, int s2, int has1, int has2,
                    float* __restrict__ lo, const double* __restrict__ rres_t) {
  extern __shared__ __align__(128) unsigned char tsm[];
  float* sL1 = reinterpret_cast<float*>(tsm + TileAdjSmem::l1);
  float* sE = reinterpret_cast<float*>(tsm + TileAdjSmem::e);
  float* sL2 = reinterpret_cast<float*>(tsm + TileAdjSmem::l2);
  float* sH = reinterpret_cast<float*>(tsm + TileAdjSmem::h);
  const uint32_t bar = smem_addr(tsm + TileAdjSmem::bar(RHO));
  const int z0 = blockIdx.x * kTZ, x0 = blockIdx.y * kTX, lu = blockIdx.z;
  const int b = (unit_begin + lu) / g.S;
  if (threadIdx.x == 0) {
    tile_bar_init(bar, 1);
    mbar_expect_tx(bar, (has1 ? kHaloBytes : 0u) + (has2 ? kPlainBytes : 0u) + kHaloBytes +
                            (RHO ? kHaloBytes : 0u));
    if (has1) tma_load_4d(smem_addr(sL1), &mL1, z0 - 4, x0 - 1, lu, s1, bar);
    if (has2) tma_load_4d(smem_addr(sL2), &mL2, z0, x0, lu, s2, bar);
    tma_load_3d(smem_addr(sE), &mEh, z0 - 4, x0 - 1, b, bar);
    if (RHO) tma_load_3d(smem_addr(sH), &mH, z0, x0, b, bar);
  }
  if (!has1) zero_slot(sL1, kHaloSlot);
  if (!has2) zero_slot(sL2, kPlainSlot);
  const TileThread tt = tile_thread(g, z0, x0);
  const bool pml = !tile_in_box(g, z0, x0);
  const bool rx = __ldg(T.tile_rx + blockIdx.y * gridDim.x + blockIdx.x) != 0;
  float* ll = lo + (size_t)lu * g.nx * g.nz;
  __syncthreads();
  mbar_wait(bar, 0);
#define DUFWI_TA(P, R) tile_adj_compute<RHO, P, R>(g, T, tt, sL1, sE, sL2, sH, lu, ll, rres_t)
  if (pml) {
    if (rx) DUFWI_TA(true, true); else DUFWI_TA(true, false);
  } else {
    if (rx) DUFWI_TA(false, true); else DUFWI_TA(false, false);
  }
#undef DUFWI_TA
}

// ------------------------------------------------ imaging + reconstruction
// sum_t L(u[t-1]) lam[t] over a group of gs shots of one phantom
// (adjoint.py:128-130) and, MODE 2, the reconstruction
// u[t-2] = u[t-1] + ((u[t-1] - u[t]) + E L u[t-1]) (+ s[t] at the source) in
// place over u[t] on the undamped box; the 1-cell ring of u[t-2] comes from
// strips[t-2] (border tiles), so the field buffer always holds box + ring.
// MODE 1 reads u[t-1] from the full history over the whole grid.
//
// A CTA walks the group's shots through a 2-stage pipeline (stage = u[t-1]
// with halo, lam[t], u[t]); the coefficient tiles E (and h) are loaded once
// per CTA, the imaging sums stay in f32 registers for the group (gs terms) and
// are added to the group's f64 accumulator once.
#ifndef DUFWI_IMG_STAGES
#define DUFWI_IMG_STAGES 2
#endif
constexpr int kImgStages = DUFWI_IMG_STAGES;  // 1: latency hidden across CTAs only; N: N-1 shots prefetched
static_assert(kImgStages >= 1 && kImgStages <= 4, "imaging pipeline depth");
struct TileImgSmem {
  static constexpr uint32_t stage = kHaloSlot + 2 * kPlainSlot;  // u1, lam, ut
  static constexpr uint32_t e = kImgStages * stage, h = e + kPlainSlot;
  __host__ __device__ static constexpr uint32_t bar(bool rho) { return h + (rho ? kHaloSlot : 0u); }
  __host__ __device__ static constexpr uint32_t bytes(bool rho) { return bar(rho) + 48u; }
};

template <bool RHO, int MODE, bool BORDER>
__device__ __forceinline__ void tile_img_shot(const Geo& g, const TileThread& t, const float* sU1,
                                              const float* sLam, const float* sUt, const float* sE,
                                              const float* sH, int txx, int txz, float pulse_t,
                                              bool recon_on, float* __restrict__ uo,
                                              const float* __restrict__ st,
                                              float (&acc)[kTRPT][4]) {
  const int nz = g.nz, nx = g.nx;
  const float* pu = sU1 + t.r0 * kTHZ + 4 + 4 * t.l;
  F4 wm(lds4(pu)), wc(lds4(pu + kTHZ));
  HWin<RHO> H;
  H.init(sH, t);
  unsigned boxk = 0xFu;
  int ringl = -1, ringr = -1;
  if (BORDER) {
    boxk = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int z = t.z4 + k;
      if (z >= g.z_lo && z <= g.z_hi) boxk |= 1u << k;
      if (z == g.z_lo - 1) ringl = k;
      if (z == g.z_hi + 1) ringr = k;
    }
  }
  const int tk = (txz >= t.z4 && txz < t.z4 + 4) ? txz - t.z4 : -1;
#pragma unroll
  for (int j = 0; j < kTRPT; ++j) {
    const int x = t.xb + j;
    const float* pr = pu + (j + 1) * kTHZ;
    const F4 wp(lds4(pr + kTHZ));
    const float zl = pr[-1], zr = pr[4];
    const F4 lam(lds4(sLam + (t.r0 + j) * kTZ + 4 * t.l));
    H.row(j);
    float lapu[4];
    stencil_row<RHO>(wm, wc, wp, zl, zr, H.f, lapu);
    // MODE 1: every grid cell; MODE 2: the undamped box
    const bool rowbox = MODE == 1 ? x < nx : (!BORDER || (x >= g.x_lo && x <= g.x_hi));
    const unsigned m = MODE == 1 ? (t.zact ? 0xFu : 0u) : (rowbox ? boxk : 0u);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (m & (1u << k)) acc[j][k] = __fmaf_rn(lapu[k], lam.v[k], acc[j][k]);
    if (MODE == 2 && recon_on) {
      const F4 ua(lds4(sUt + (t.r0 + j) * kTZ + 4 * t.l));
      const F4 e4(lds4(sE + (t.r0 + j) * kTZ + 4 * t.l));
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float prev = inc_recon(wc.v[k], ua.v[k], e4.v[k], lapu[k]);
        if (x == txx && k == tk) prev = __fadd_rn(prev, pulse_t);
        o[k] = (m & (1u << k)) ? prev : ua.v[k];
      }
      bool wr = !BORDER;
      if (BORDER && t.zact && x < nx) {
        if (rowbox) {
          wr = boxk != 0u || ringl >= 0 || ringr >= 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k == ringl) o[k] = __ldg(st + 2 * g.Lz + x - g.x_lo);
            if (k == ringr) o[k] = __ldg(st + 2 * g.Lz + g.Lx + x - g.x_lo);
          }
        } else if (x == g.x_lo - 1 || x == g.x_hi + 1) {  // ring rows
          wr = boxk != 0u;
          const int base = (x == g.x_lo - 1 ? 0 : g.Lz) - g.z_lo + t.z4;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (boxk & (1u << k)) o[k] = __ldg(st + base + k);
        }
      }
      if (wr) *reinterpret_cast<float4*>(uo + x * nz + t.z4) = make_float4(o[0], o[1], o[2], o[3]);
    }
    wm = wc;
    wc = wp;
    H.next();
  }
}

// mU1: halo'd boxes of the region holding u[t-1] (slot su1); mLam / mUt: plain
// boxes of lam[t] (slot sl) and u[t] (slot sut); ut: u[t]'s buffer (unit 0),
// rewritten in place; (tx0, tz0): first tile of the launch's tile range.
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kTT)
    tile_img_kernel(const __grid_constant__ CUtensorMap mU1, const __grid_constant__ CUtensorMap mLam,
                    const __grid_constant__ CUtensorMap mUt, const __grid_constant__ CUtensorMap mE,
                    const __grid_constant__ CUtensorMap mH, Geo g, int t, int unit_begin, int U, int gs,
                    int su1, int sl, int sut, int tx0, int tz0, float* __restrict__ ut,
                    const float* __restrict__ strip_tm2, double* __restrict__ acc_part,
                    int do_recon) {
  extern __shared__ __align__(128) unsigned char tsm[];
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  float* sE = reinterpret_cast<float*>(tsm + TileImgSmem::e);
  float* sH = reinterpret_cast<float*>(tsm + TileImgSmem::h);
  const uint32_t bar = smem_addr(tsm + TileImgSmem::bar(RHO));  // [0 .. 3]: stages, [4]: coefficients
  const uint32_t cbar = bar + 32u;
  const int z0 = (tz0 + blockIdx.x) * kTZ, x0 = (tx0 + blockIdx.y) * kTX;
  const bool recon_on = MODE == 2 && do_recon;
  const size_t N2 = (size_t)g.nx * g.nz;
  const uint32_t stage_bytes = kHaloBytes + kPlainBytes + (recon_on ? kPlainBytes : 0u);
  auto issue = [&](int k) {  // thread 0: the operands of the group's k-th shot
    unsigned char* sb = tsm + (k % kImgStages) * TileImgSmem::stage;
    const uint32_t bk = bar + 8u * (k % kImgStages);
    const int lu = sg.lu0 + k;
    mbar_expect_tx(bk, stage_bytes);
    tma_load_4d(smem_addr(sb), &mU1, z0 - 4, x0 - 1, lu, su1, bk);
    tma_load_4d(smem_addr(sb + kHaloSlot), &mLam, z0, x0, lu, sl, bk);
    if (recon_on) tma_load_4d(smem_addr(sb + kHaloSlot + kPlainSlot), &mUt, z0, x0, lu, sut, bk);
  };
  if (threadIdx.x == 0) {
    tile_bar_init(bar, 5);
    const uint32_t cb = (recon_on ? kPlainBytes : 0u) + (RHO ? kHaloBytes : 0u);
    if (cb) {
      mbar_expect_tx(cbar, cb);
      if (recon_on) tma_load_3d(smem_addr(sE), &mE, z0, x0, sg.b, cbar);
      if (RHO) tma_load_3d(smem_addr(sH), &mH, z0, x0, sg.b, cbar);
    }
    issue(0);
    for (int k = 1; k < kImgStages - 1 && k < sg.n; ++k) issue(k);
  }
  const TileThread tt = tile_thread(g, z0, x0);
  const bool border = MODE == 2 && !tile_in_box(g, z0, x0);
  const float pulse_t = (float)__ldg(g.pulse + t);
  float acc[kTRPT][4];
#pragma unroll
  for (int j = 0; j < kTRPT; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[j][k] = 0.f;
  __syncthreads();
  if (recon_on || RHO) mbar_wait(cbar, 0);
  for (int k = 0; k < sg.n; ++k) {
    // shot k + N - 1 goes into the stage shot k - 1 used (free since the last barrier)
    if (kImgStages >= 2 && threadIdx.x == 0 && k + kImgStages - 1 < sg.n) issue(k + kImgStages - 1);
    mbar_wait(bar + 8u * (k % kImgStages), (uint32_t)(k / kImgStages) & 1u);
    const unsigned char* sb = tsm + (k % kImgStages) * TileImgSmem::stage;
    const float* sU1 = reinterpret_cast<const float*>(sb);
    const float* sLam = reinterpret_cast<const float*>(sb + kHaloSlot);
    const float* sUt = reinterpret_cast<const float*>(sb + kHaloSlot + kPlainSlot);
    const int lu = sg.lu0 + k;
    const int s = (unit_begin + lu) % g.S;
    const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
    float* uo = ut + (size_t)lu * N2;
    const float* st = MODE == 2 ? strip_tm2 + (size_t)lu * g.SL : nullptr;
    if (border)
      tile_img_shot<RHO, MODE, true>(g, tt, sU1, sLam, sUt, sE, sH, txx, txz, pulse_t, recon_on, uo,
                                     st, acc);
    else
      tile_img_shot<RHO, MODE, false>(g, tt, sU1, sLam, sUt, sE, sH, txx, txz, pulse_t, recon_on,
                                      uo, st, acc);
    __syncthreads();  // every thread is done with the stage: it may be refilled
    if (kImgStages == 1 && threadIdx.x == 0 && k + 1 < sg.n) issue(k + 1);
  }
  if (tt.zact) {
    double* dst = acc_part + (size_t)blockIdx.z * N2 + tt.z4;
#pragma unroll
    for (int j = 0; j < kTRPT; ++j) {
      const int x = tt.xb + j;
      if (x >= g.nx) break;
      if (MODE == 2 && (x < g.x_lo || x > g.x_hi)) continue;
      double2* p = reinterpret_cast<double2*>(dst + (size_t)x * g.nz);
      double2 a = p[0], c = p[1];
      a.x += (double)acc[j][0];
      a.y += (double)acc[j][1];
      c.x += (double)acc[j][2];
      c.y += (double)acc[j][3];
      p[0] = a;
      p[1] = c;
    }
  }
}

// h = q / 2 on the replicate-padded grid [B][nx+2][nz+8] (cell (x, z) at
// [x+1][z+4]): the outer faces h_c + h_c = q_c of the oracle's rho_face_weights.
__global__ void hq_pad_kernel(Geo g, int B, const float* __restrict__ qf, float* __restrict__ hq) {
  const int px = g.nx + 2, pz = g.nz + 8;
  const size_t total = (size_t)B * px * pz;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / ((size_t)px * pz));
    const int r = (int)(i % ((size_t)px * pz));
    const int x = min(max(r / pz - 1, 0), g.nx - 1), z = min(max(r % pz - 4, 0), g.nz - 1);
    hq[i] = 0.5f * qf[((size_t)b * g.nx + x) * g.nz + z];
  }
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// f32 tensor [d3][d2][nx_][nz_] (d3 = 0: rank 3) with boxes of bx rows x bz columns.
inline bool make_tile_map(CUtensorMap* m, const float* base, int nz_, int nx_, size_t d2, size_t d3,
                          bool halo) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15u)) return false;
  const cuuint32_t rank = d3 ? 4 : 3;
  const cuuint64_t dim[4] = {(cuuint64_t)nz_, (cuuint64_t)nx_, (cuuint64_t)d2, (cuuint64_t)(d3 ? d3 : 1)};
  const cuuint64_t str[3] = {(cuuint64_t)nz_ * 4, (cuuint64_t)nz_ * nx_ * 4,
                             (cuuint64_t)nz_ * nx_ * d2 * 4};
  const cuuint32_t box[4] = {(cuuint32_t)(halo ? kTHZ : kTZ), (cuuint32_t)(halo ? kTHX : kTX), 1, 1};
  const cuuint32_t est[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), dim, str, box, est,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace dufwi
