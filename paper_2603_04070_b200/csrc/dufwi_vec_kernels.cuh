// Stepwise engine, vectorised kernels (nz % 4 == 0, constant density).
//
// A warp owns a 128-wide z strip — each lane 4 consecutive cells, loaded and
// stored as one float4 — and walks TX x-rows of ONE shot, keeping rows x-1,
// x, x+1 in f64 registers (every f32 value converted once).  The rows ahead
// stream through a per-lane cp.async ring of kPipe row slots in shared memory,
// so every warp keeps kPipe-1 rows of loads in flight while it computes.
// z-neighbours come from f64 warp shuffles; the strip's outer neighbours
// (z0-1, z0+128) travel in the same ring.
// DRAM per cell update: forward read u[t-1], u[t-2], write u[t] = 12 B
// (E is read once per phantom per step and shared by its shots through L2).
#pragma once

#include "dufwi_step_kernels.cuh"

namespace dufwi {


struct Row4 {
  double v[4];
};

__device__ __forceinline__ Row4 to_d(float4 f) {
  Row4 r;
  r.v[0] = f.x;
  r.v[1] = f.y;
  r.v[2] = f.z;
  r.v[3] = f.w;
  return r;
}

// (A, B) of one cell in the damping band: the 1-D tables (or the 2-D map).
// Kept out of line (returned in registers) so the undamped fast path carries
// none of its address arithmetic.
__device__ __noinline__ double2 ab_damped(ABTables T, int x, int z, int nz) {
  if (T.px) {
    const bool xs = __ldg(T.px + x) >= __ldg(T.pz + z);
    return make_double2(xs ? __ldg(T.Ax + x) : __ldg(T.Az + z),
                        xs ? __ldg(T.Bx + x) : __ldg(T.Bz + z));
  }
  const size_t i = (size_t)x * nz + z;
  return make_double2(__ldg(T.A2 + i), __ldg(T.B2 + i));
}

// (A, B) for the 4 cells of a lane: (2, -1) when the row and the lane's cells
// are undamped, else per cell from the tables.
__device__ __forceinline__ void ab4(const ABTables& T, int x, int z4, int nz, bool lane_damped,
                                    double (&A)[4], double (&B)[4]) {
  if (T.px && !lane_damped && __ldg(T.px + x) == 0.0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { A[k] = 2.0; B[k] = -1.0; }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 ab = ab_damped(T, x, min(z4 + k, nz - 1), nz);
      A[k] = ab.x;
      B[k] = ab.y;
    }
  }
}

// cp.async helpers: per-lane asynchronous global->shared copies; src_size 0
// zero-fills (rows outside the grid).  Each lane reads back only what it
// copied, so the pipeline needs no inter-lane synchronisation.
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
#ifdef DUFWI_CP_L2_256
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
#endif
}
__device__ __forceinline__ void cp4(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kPipe = 4;       // rows of loads in flight per lane (power of two)
constexpr int kPipeWarps = 4;  // warps per CTA (shared-memory ring per lane)

// Per-lane ring of kPipe row slots, structure-of-arrays so every access is
// bank-conflict free: u[t-1] row x+1 (+ strip edges), u[t-2] row x, E row x.
struct FwdRing {
  float4 u1[kPipe][kPipeWarps * 32];
  float4 u2[kPipe][kPipeWarps * 32];
  double2 e[kPipe][2][kPipeWarps * 32];
  float2 edge[kPipe][kPipeWarps * 32];
};

template <int MODE>
__global__ void __launch_bounds__(kPipeWarps * 32)
    fwd_vec_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int TX,
                   const float* __restrict__ u1, const float* u2, float* uo,
                   float* __restrict__ rec_t, float* __restrict__ strip_t, int has1, int has2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdRing& ring = *reinterpret_cast<FwdRing*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nz = g.nz, nx = g.nx;
  const int z0 = blockIdx.x * 128;
  const int z4 = z0 + 4 * lane;
  const bool act = z4 < nz;
  const int x0 = (blockIdx.y * kPipeWarps + warp) * TX;
  if (x0 >= nx) return;  // warp-uniform
  const int x1 = min(nx, x0 + TX);
  const int lu = blockIdx.z;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)nx * nz;
  const float* f1 = u1 + (size_t)lu * N2;
  const float* f2 = u2 + (size_t)lu * N2;
  float* fo = uo + (size_t)lu * N2;
  const double* Ed = m.Ed + (size_t)b * N2;
  const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
  const int tk = (txz >= z4 && txz < z4 + 4) ? txz - z4 : -1;
  const double pulse_t = __ldg(g.pulse + t);
  bool lane_damped = false;
  if (T.px && act) {
#pragma unroll
    for (int k = 0; k < 4; ++k) lane_damped |= __ldg(T.pz + min(z4 + k, nz - 1)) != 0.0;
  }
  const bool edge_l = lane == 0 && z0 > 0, edge_r = lane == 31 && z0 + 128 < nz;
  const int zc = act ? z4 : 0;

  // issue the copies of "row r": u[t-1] row r+1 (+ edges), u[t-2] row r, E row r.
  // 32-bit row offsets from per-lane base pointers keep the address math short.
  const float* b1 = f1 + zc;
  const float* b2 = f2 + zc;
  const double* be = Ed + zc;
  const float* bl = f1 + (edge_l ? z0 - 1 : 0);
  const float* br = f1 + (edge_r ? z0 + 128 : 0);
  const bool has2a = has2 && act;
  auto issue = [&](int r) {
    const int sl = r & (kPipe - 1);
    const bool okn = r + 1 < nx;
    const int ou = okn ? (r + 1) * nz : 0;
    const int orr = r * nz;  // r < x1 <= nx
    const bool ok1 = has1 && okn;
    cp16(&ring.u1[sl][tid], b1 + ou, ok1 && act);
    cp16(&ring.u2[sl][tid], b2 + orr, has2a);
    cp16(&ring.e[sl][0][tid], be + orr, act);
    cp16(&ring.e[sl][1][tid], be + orr + 2, act);
    float* ed = reinterpret_cast<float*>(&ring.edge[sl][tid]);
    cp4(ed, bl + ou, ok1 && edge_l);
    cp4(ed + 1, br + ou, ok1 && edge_r);
  };

  auto ld_row = [&](int x, float& el, float& er) -> float4 {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    el = er = 0.f;
    if (has1 && x >= 0 && x < nx) {
      const float* p = f1 + (size_t)x * nz;
      if (act) r = __ldg(reinterpret_cast<const float4*>(p + z4));
      if (edge_l) el = __ldg(p + z0 - 1);
      if (edge_r) er = __ldg(p + z0 + 128);
    }
    return r;
  };
  float elm, erm, elc, erc;
  Row4 um = to_d(ld_row(x0 - 1, elm, erm));
  Row4 uc = to_d(ld_row(x0, elc, erc));
  (void)elm;
  (void)erm;
#pragma unroll
  for (int k = 0; k < kPipe - 1; ++k) {
    if (x0 + k < x1) issue(x0 + k);
    cp_commit();
  }

  for (int x = x0; x < x1; ++x) {
    if (x + kPipe - 1 < x1) issue(x + kPipe - 1);
    cp_commit();
    cp_wait<kPipe - 1>();  // the group of row x has landed
    const int sl = x & (kPipe - 1);
    const Row4 up = to_d(ring.u1[sl][tid]);
    const Row4 w2 = to_d(ring.u2[sl][tid]);
    const double2 e0 = ring.e[sl][0][tid], e1 = ring.e[sl][1][tid];
    const float2 edn = ring.edge[sl][tid];
    const double ed[4] = {e0.x, e0.y, e1.x, e1.y};
    double zl = __shfl_up_sync(0xffffffffu, uc.v[3], 1);
    double zr = __shfl_down_sync(0xffffffffu, uc.v[0], 1);
    if (lane == 0) zl = (double)elc;
    if (lane == 31) zr = (double)erc;
    double A[4], B[4];
    ab4(T, x, z4, nz, lane_damped, A, B);
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double zm = k == 0 ? zl : uc.v[k - 1];
      const double zp = k == 3 ? zr : uc.v[k + 1];
      const double lap = (((-4.0 * uc.v[k] + um.v[k]) + up.v[k]) + zm) + zp;
      v[k] = A[k] * uc.v[k] + B[k] * w2.v[k] + ed[k] * lap;
    }
    if (x == txx && tk >= 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k == tk) v[k] += pulse_t;
    }
    if (act) {
      const size_t row = (size_t)x * nz;
      *reinterpret_cast<float4*>(fo + row + z4) =
          make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
      if (__ldg(g.row_flag + x)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int slot = __ldg(g.node_slot + row + z4 + k);
          if (slot >= 0) rec_t[(size_t)lu * g.M + slot] = (float)v[k];
        }
      }
      if (MODE == 2) {
        float* st = strip_t + (size_t)lu * g.SL;
        const bool xr = x == g.x_lo - 1 || x == g.x_hi + 1;
        const bool xin = x >= g.x_lo && x <= g.x_hi;
        if (xr || xin) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int z = z4 + k;
            if (xr && z >= g.z_lo && z <= g.z_hi)
              st[(x == g.x_lo - 1 ? 0 : g.Lz) + z - g.z_lo] = (float)v[k];
            if (xin && (z == g.z_lo - 1 || z == g.z_hi + 1))
              st[2 * g.Lz + (z == g.z_lo - 1 ? 0 : g.Lx) + x - g.x_lo] = (float)v[k];
          }
        }
      }
    }
    um = uc;
    uc = up;
    elc = edn.x;
    erc = edn.y;
  }
  cp_wait<0>();
}

}  // namespace dufwi

namespace dufwi {

// ---------------------------------------------------------------------------
// Vectorised adjoint (constant density, nz % 4 == 0), split in two kernels per
// step: adjlam_vec (lam[t]) then img_vec (imaging + u[t-2] reconstruction).
// A warp owns a 128-wide z strip x kVecAdjTX rows.
constexpr int kVecAdjWarps = 4;
constexpr int kVecAdjTX = 8;


// ---------------------------------------------------------------------------
// Split vectorised adjoint (constant density, nz % 4 == 0), kernel 1 of 2:
// lam[t] = A lam[t+1] + L^T(E lam[t+1]) + B lam[t+2] (+ merged residual at the
// receiver nodes), in place over lam[t+2], one shot per warp.  DRAM: 12 B per
// cell update (E is shared by the phantom's shots through L2).
// Pipelined variant of the lam update: the rows of lam[t+1] (+ E, + strip
// edges) and lam[t+2] stream through a per-lane cp.async ring of kPipe rows,
// as in fwd_vec_kernel, so each warp keeps kPipe-1 rows of loads in flight.
struct AdjRing {
  float4 l1[kPipe][kPipeWarps * 32];      // lam[t+1] row r+1
  double2 e[kPipe][2][kPipeWarps * 32];   // E row r+1
  float4 l2[kPipe][kPipeWarps * 32];      // lam[t+2] row r
  float2 edl[kPipe][kPipeWarps * 32];     // lam[t+1] row r+1 at z0-1 / z0+128
  double2 ede[kPipe][kPipeWarps * 32];    // E row r+1 at z0-1 / z0+128
};

__device__ __forceinline__ void cp8(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(ok ? 8 : 0)
               : "memory");
}

__global__ void __launch_bounds__(kPipeWarps * 32)
    adjlam_pipe_kernel(Geo g, Model m, ABTables T, int t, int unit_begin, int TX,
                       const float* __restrict__ l1, float* l2o, const double* __restrict__ rres_t,
                       int has1, int has2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AdjRing& ring = *reinterpret_cast<AdjRing*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nz = g.nz, nx = g.nx;
  const int z0 = blockIdx.x * 128;
  const int z4 = z0 + 4 * lane;
  const bool act = z4 < nz;
  const int x0 = (blockIdx.y * kPipeWarps + warp) * TX;
  if (x0 >= nx) return;  // warp-uniform
  const int x1 = min(nx, x0 + TX);
  const int lu = blockIdx.z;
  const int b = (unit_begin + lu) / g.S;
  const size_t N2 = (size_t)nx * nz;
  const float* L1 = l1 + (size_t)lu * N2;
  float* L2 = l2o + (size_t)lu * N2;
  const double* Ed = m.Ed + (size_t)b * N2;
  bool lane_damped = false;
  if (T.px && act) {
#pragma unroll
    for (int k = 0; k < 4; ++k) lane_damped |= __ldg(T.pz + min(z4 + k, nz - 1)) != 0.0;
  }
  const bool edge_l = lane == 0 && z0 > 0, edge_r = lane == 31 && z0 + 128 < nz;
  const int zc = act ? z4 : 0;
  const int zl = edge_l ? z0 - 1 : 0, zr = edge_r ? z0 + 128 : 0;
  const bool has1a = has1 && act, has2a = has2 && act;

  // copies of "row r": lam1 / E row r+1 (+ edges), lam2 row r
  auto issue = [&](int r) {
    const int sl = r & (kPipe - 1);
    const bool okn = r + 1 < nx;
    const int on = okn ? (r + 1) * nz : 0;
    const int orr = r * nz;
    cp16(&ring.l1[sl][tid], L1 + on + zc, has1a && okn);
    cp16(&ring.e[sl][0][tid], Ed + on + zc, act && okn);
    cp16(&ring.e[sl][1][tid], Ed + on + zc + 2, act && okn);
    cp16(&ring.l2[sl][tid], L2 + orr + zc, has2a);
    float* el = reinterpret_cast<float*>(&ring.edl[sl][tid]);
    double* ee = reinterpret_cast<double*>(&ring.ede[sl][tid]);
    cp4(el, L1 + on + zl, has1 && okn && edge_l);
    cp4(el + 1, L1 + on + zr, has1 && okn && edge_r);
    cp8(ee, Ed + on + zl, okn && edge_l);
    cp8(ee + 1, Ed + on + zr, okn && edge_r);
  };
  // E*lam1 of row x (4 own cells, strip edges) and raw lam1, loaded directly
  struct ERow {
    double e[4], l[4], el, er;
  };
  auto ld = [&](int x) -> ERow {
    ERow r;
#pragma unroll
    for (int k = 0; k < 4; ++k) r.e[k] = r.l[k] = 0.0;
    r.el = r.er = 0.0;
    if (has1 && x >= 0 && x < nx) {
      const size_t row = (size_t)x * nz;
      if (act) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(L1 + row + z4));
        const double2 a = __ldg(reinterpret_cast<const double2*>(Ed + row + z4));
        const double2 c = __ldg(reinterpret_cast<const double2*>(Ed + row + z4 + 2));
        r.l[0] = f.x; r.l[1] = f.y; r.l[2] = f.z; r.l[3] = f.w;
        r.e[0] = a.x * r.l[0]; r.e[1] = a.y * r.l[1]; r.e[2] = c.x * r.l[2]; r.e[3] = c.y * r.l[3];
      }
      if (edge_l) r.el = __ldg(Ed + row + z0 - 1) * (double)__ldg(L1 + row + z0 - 1);
      if (edge_r) r.er = __ldg(Ed + row + z0 + 128) * (double)__ldg(L1 + row + z0 + 128);
    }
    return r;
  };
  ERow rm = ld(x0 - 1), rc = ld(x0);
#pragma unroll
  for (int k = 0; k < kPipe - 1; ++k) {
    if (x0 + k < x1) issue(x0 + k);
    cp_commit();
  }
  for (int x = x0; x < x1; ++x) {
    if (x + kPipe - 1 < x1) issue(x + kPipe - 1);
    cp_commit();
    cp_wait<kPipe - 1>();  // the group of row x has landed
    const int sl = x & (kPipe - 1);
    // row x+1 from the ring
    ERow rp;
    {
      const float4 f = ring.l1[sl][tid];
      const double2 a = ring.e[sl][0][tid], c = ring.e[sl][1][tid];
      rp.l[0] = f.x; rp.l[1] = f.y; rp.l[2] = f.z; rp.l[3] = f.w;
      rp.e[0] = a.x * rp.l[0]; rp.e[1] = a.y * rp.l[1]; rp.e[2] = c.x * rp.l[2]; rp.e[3] = c.y * rp.l[3];
      const float2 fl = ring.edl[sl][tid];
      const double2 el = ring.ede[sl][tid];
      rp.el = el.x * (double)fl.x;
      rp.er = el.y * (double)fl.y;
    }
    const Row4 w2 = to_d(ring.l2[sl][tid]);
    double zm0 = __shfl_up_sync(0xffffffffu, rc.e[3], 1);
    double zp3 = __shfl_down_sync(0xffffffffu, rc.e[0], 1);
    if (lane == 0) zm0 = rc.el;
    if (lane == 31) zp3 = rc.er;
    double A[4], B[4];
    ab4(T, x, z4, nz, lane_damped, A, B);
    double lam[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double zm = k == 0 ? zm0 : rc.e[k - 1];
      const double zp = k == 3 ? zp3 : rc.e[k + 1];
      const double adj = (((-4.0 * rc.e[k] + rm.e[k]) + rp.e[k]) + zm) + zp;
      lam[k] = (A[k] * rc.l[k] + adj) + B[k] * w2.v[k];
    }
    if (act) {
      const size_t row = (size_t)x * nz;
      if (__ldg(g.row_flag + x)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int slot = __ldg(g.node_slot + row + z4 + k);
          if (slot >= 0) lam[k] += __ldg(rres_t + (size_t)lu * g.M + slot);
        }
      }
      *reinterpret_cast<float4*>(L2 + row + z4) =
          make_float4((float)lam[0], (float)lam[1], (float)lam[2], (float)lam[3]);
    }
    rm = rc;
    rc = rp;
  }
  cp_wait<0>();
}

// Split vectorised adjoint, kernel 2 of 2: imaging sum_t L(u[t-1]) lam[t] over
// the group's shots (per-warp shared tile, one read-modify-write of
// acc_part[group] per step) and, MODE 2, the reconstruction
// u[t-2] = 2 u[t-1] + E L u[t-1] + s[t] d_tx - u[t] in place over u[t] on the
// undamped box, with the ring neighbours taken from strips[t-1].
// DRAM per cell update: MODE 2 read u[t-1], u[t], lam[t], write u[t-2] = 16 B;
// MODE 1 read u[t-1] (history), lam[t] = 8 B.
template <int MODE>
__global__ void __launch_bounds__(kVecAdjWarps * 32)
    img_vec_kernel(Geo g, Model m, int t, int unit_begin, int U, int gs,
                   const float* __restrict__ lam_t, const float* __restrict__ F, float* ut,
                   const float* __restrict__ utm1, const float* __restrict__ strip_tm1,
                   double* __restrict__ acc_part, int do_recon) {
  __shared__ double acc_s[kVecAdjWarps][kVecAdjTX][128];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nz = g.nz, nx = g.nx;
  const int z0 = blockIdx.x * 128;
  const int z4 = z0 + 4 * lane;
  const bool act = z4 < nz;
  int x0 = (blockIdx.y * kVecAdjWarps + warp) * kVecAdjTX;
  int x1 = min(nx, x0 + kVecAdjTX);
  if (MODE == 2) {  // imaging and reconstruction live on the undamped box only
    x0 = max(x0, g.x_lo);
    x1 = min(x1, g.x_hi + 1);
  }
  if (x0 >= x1) return;
  const ShotGroup sg = shot_group(g, blockIdx.z, unit_begin, U, gs);
  if (sg.n == 0) return;
  const size_t N2 = (size_t)nx * nz;
  const double* Ed = m.Ed + (size_t)sg.b * N2;
  const double pulse_t = __ldg(g.pulse + t);
  const bool edge_l = lane == 0 && z0 > 0, edge_r = lane == 31 && z0 + 128 < nz;
  double(&acc)[kVecAdjTX][128] = acc_s[warp];
  const int xb = (blockIdx.y * kVecAdjWarps + warp) * kVecAdjTX;
#pragma unroll
  for (int r = 0; r < kVecAdjTX; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[r][4 * lane + k] = 0.0;
  // which of my cells are in the box (MODE 2) / on a ring column
  unsigned inbox = 0u;
  int ringk[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int z = z4 + k;
    if (MODE == 1 || (act && z >= g.z_lo && z <= g.z_hi)) inbox |= 1u << k;
    // ring columns inside the grid only (no PML: the ring lies outside, = 0)
    ringk[k] = (MODE == 2 && act && z == g.z_lo - 1) ? 2 * g.Lz
             : (MODE == 2 && act && z == g.z_hi + 1) ? 2 * g.Lz + g.Lx : -1;
  }
  const int ring_l = (MODE == 2 && z0 - 1 == g.z_lo - 1) ? 2 * g.Lz : -1;
  const int ring_r = (MODE == 2 && z0 + 128 == g.z_hi + 1) ? 2 * g.Lz + g.Lx : -1;
  const bool in_l = MODE == 1 || (z0 - 1 >= g.z_lo && z0 - 1 <= g.z_hi);
  const bool in_r = MODE == 1 || (z0 + 128 >= g.z_lo && z0 + 128 <= g.z_hi);

  struct URow {
    double v[4], el, er;
  };
  for (int k0 = 0; k0 < sg.n; ++k0) {
    const int lu = sg.lu0 + k0;
    const size_t fo = (size_t)lu * N2;
    const int s = (unit_begin + lu) % g.S;
    const int txx = __ldg(g.tx + 2 * s), txz = __ldg(g.tx + 2 * s + 1);
    const int tk = (txz >= z4 && txz < z4 + 4) ? txz - z4 : -1;
    const float* UB = MODE == 1 ? F + fo : utm1 + fo;
    const float* st = MODE == 2 ? strip_tm1 + (size_t)lu * g.SL : nullptr;
    // u[t-1] of row x as the reconstruction sees it
    auto ld = [&](int x) -> URow {
      URow r;
#pragma unroll
      for (int k = 0; k < 4; ++k) r.v[k] = 0.0;
      r.el = r.er = 0.0;
      if (x < 0 || x >= nx) return r;
      const size_t row = (size_t)x * nz;
      const bool xbox = MODE == 1 || (x >= g.x_lo && x <= g.x_hi);
      if (xbox) {
        if (act) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(UB + row + z4));
          r.v[0] = f.x; r.v[1] = f.y; r.v[2] = f.z; r.v[3] = f.w;
        }
        if (edge_l) r.el = in_l ? (double)__ldg(UB + row + z0 - 1)
                                : (ring_l >= 0 ? (double)__ldg(st + ring_l + x - g.x_lo) : 0.0);
        if (edge_r) r.er = in_r ? (double)__ldg(UB + row + z0 + 128)
                                : (ring_r >= 0 ? (double)__ldg(st + ring_r + x - g.x_lo) : 0.0);
        if (MODE == 2) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (ringk[k] >= 0) r.v[k] = (double)__ldg(st + ringk[k] + x - g.x_lo);
            else if (!(inbox & (1u << k))) r.v[k] = 0.0;
          }
        }
      } else if (MODE == 2) {  // ring row above/below the box
        const float* sr = st + (x == g.x_lo - 1 ? 0 : g.Lz);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (inbox & (1u << k)) r.v[k] = (double)__ldg(sr + z4 + k - g.z_lo);
        if (edge_l && in_l) r.el = (double)__ldg(sr + z0 - 1 - g.z_lo);
        if (edge_r && in_r) r.er = (double)__ldg(sr + z0 + 128 - g.z_lo);
      }
      return r;
    };
    URow rm = ld(x0 - 1), rc = ld(x0), rn = ld(x0 + 1);
    for (int x = x0; x < x1; ++x) {
      const URow rp = rn;
      const size_t row = (size_t)x * nz;
      const float4 lf = act ? __ldg(reinterpret_cast<const float4*>(lam_t + fo + row + z4))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 uf = make_float4(0.f, 0.f, 0.f, 0.f);
      if (MODE == 2 && do_recon && act) uf = *reinterpret_cast<const float4*>(ut + fo + row + z4);
      double2 e0 = make_double2(0, 0), e1 = make_double2(0, 0);
      if (MODE == 2 && do_recon && act) {
        e0 = __ldg(reinterpret_cast<const double2*>(Ed + row + z4));
        e1 = __ldg(reinterpret_cast<const double2*>(Ed + row + z4 + 2));
      }
      if (x + 1 < x1) rn = ld(x + 2);
      double zl = __shfl_up_sync(0xffffffffu, rc.v[3], 1);
      double zr = __shfl_down_sync(0xffffffffu, rc.v[0], 1);
      if (lane == 0) zl = rc.el;
      if (lane == 31) zr = rc.er;
      const Row4 lam = to_d(lf);
      const double ed[4] = {e0.x, e0.y, e1.x, e1.y};
      const Row4 uv = to_d(uf);
      float o[4] = {uf.x, uf.y, uf.z, uf.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double zm = k == 0 ? zl : rc.v[k - 1];
        const double zp = k == 3 ? zr : rc.v[k + 1];
        const double lapu = (((-4.0 * rc.v[k] + rm.v[k]) + rp.v[k]) + zm) + zp;
        if (inbox & (1u << k)) {
          acc[x - xb][4 * lane + k] += lapu * lam.v[k];
          if (MODE == 2 && do_recon) {
            double prev = 2.0 * rc.v[k] + ed[k] * lapu - uv.v[k];
            if (x == txx && k == tk) prev += pulse_t;
            o[k] = (float)prev;
          }
        }
      }
      if (MODE == 2 && do_recon && act)
        *reinterpret_cast<float4*>(ut + fo + row + z4) = make_float4(o[0], o[1], o[2], o[3]);
      rm = rc;
      rc = rp;
    }
  }
  if (act) {
    double* dst = acc_part + (size_t)blockIdx.z * N2;
    for (int x = x0; x < x1; ++x)
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[(size_t)x * nz + z4 + k] += acc[x - xb][4 * lane + k];
  }
}



}  // namespace dufwi
