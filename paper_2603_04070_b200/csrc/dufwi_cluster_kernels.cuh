// Cluster engine: one kernel launch per sweep, one thread-block cluster per unit.
//
// For grids whose per-unit state fits the cluster's shared memory (configs
// 0/1: 160^2; config 2: 296^2) the whole time loop runs inside one launch.
// The unit's grid is cut into `cs` slabs of `rows` x-rows, one per CTA of the
// cluster.  Each CTA keeps its slab of every live field (u[t-1], u[t-2] for the
// forward; lam[t+1], lam[t+2], u[t], u[t-1] for the adjoint) plus one halo row
// on each side in shared memory.  After a CTA updates a boundary row it pushes
// the new values straight into the neighbour CTA's halo row through
// distributed shared memory (st.shared::cluster); one cluster barrier per time
// step orders those pushes against the next step's reads.  HBM then only sees
// the receiver samples, the 1-cell ring strips and the final two states — the
// "temporal blocking in the extreme" of SURVEY §7.1-5.
//
// Numerics are the stepwise engine's: f32 storage, f64 per-cell arithmetic in
// the reference's operation order.
#pragma once

#include <cooperative_groups.h>

#include "dufwi_common.cuh"

namespace dufwi {

namespace cg = cooperative_groups;

struct ClusterCfg {
  int cs = 0;        // CTAs per cluster (slabs per unit)
  int rows = 0;      // x-rows per slab
  int threads = 0;   // threads per CTA
  size_t smem_fwd = 0, smem_adj = 0;
};

constexpr int kClusterThreads = 512;

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// shared-memory carve-up (all offsets 16-byte aligned)
struct SmemPlan {
  size_t fA, fB, fC, fD;   // field buffers, (rows+2) x nz floats each
  size_t ed;               // (rows+2) x nz doubles (E/dx^2, halo rows included)
  size_t acc;              // rows x nz doubles (adjoint imaging accumulator)
  size_t px, pz;           // rows / nz doubles
  size_t total;
};

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

__host__ __device__ inline SmemPlan smem_plan(int rows, int nz, bool adjoint) {
  SmemPlan p{};
  const size_t fb = al16((size_t)(rows + 2) * nz * sizeof(float));
  size_t o = 0;
  p.fA = o; o += fb;
  p.fB = o; o += fb;
  if (adjoint) { p.fC = o; o += fb; p.fD = o; o += fb; } else { p.fC = p.fD = 0; }
  p.ed = o; o += al16((size_t)(rows + 2) * nz * sizeof(double));
  if (adjoint) { p.acc = o; o += al16((size_t)rows * nz * sizeof(double)); } else { p.acc = 0; }
  p.px = o; o += al16((size_t)rows * sizeof(double));
  p.pz = o; o += al16((size_t)nz * sizeof(double));
  p.total = o;
  return p;
}

// Slab geometry of this CTA.
struct Slab {
  int rank, cs, rows, r0, nr;  // rows [r0, r0+nr)
};

__device__ __forceinline__ Slab my_slab(int cs, int rows, int nx) {
  Slab s;
  s.cs = cs;
  s.rows = rows;
  s.rank = (int)cg::this_cluster().block_rank();
  s.r0 = s.rank * rows;
  s.nr = max(0, min(nx, s.r0 + rows) - s.r0);
  return s;
}

// Push a freshly computed boundary value of local slab row xr (1-based) into
// the neighbouring CTAs' halo rows of the same buffer.
__device__ __forceinline__ void push_halo(float* buf, const Slab& sl, int xr, int z, int nz,
                                          int nx, float v) {
  if (xr == 1 && sl.rank > 0) {
    float* dst = cg::this_cluster().map_shared_rank(buf, sl.rank - 1);
    dst[(size_t)(sl.rows + 1) * nz + z] = v;
  }
  if (xr == sl.nr && sl.rank + 1 < sl.cs && (sl.rank + 1) * sl.rows < nx) {
    float* dst = cg::this_cluster().map_shared_rank(buf, sl.rank + 1);
    dst[z] = v;
  }
}

// ---------------------------------------------------------------------------
// forward sweep (MODE 0 none / 1 full history / 2 strips)
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kClusterThreads, 1)
    cluster_fwd_kernel(Geo g, Model m, int cs, int rows, int unit_begin, int U,
                       float* __restrict__ rec, float* __restrict__ hist,
                       float* __restrict__ strips, float* __restrict__ ubuf) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Slab sl = my_slab(cs, rows, g.nx);
  const int nz = g.nz;
  const SmemPlan sp = smem_plan(rows, nz, false);
  float* P[2] = {reinterpret_cast<float*>(smem + sp.fA), reinterpret_cast<float*>(smem + sp.fB)};
  double* eds = reinterpret_cast<double*>(smem + sp.ed);
  double* pxs = reinterpret_cast<double*>(smem + sp.px);
  double* pzs = reinterpret_cast<double*>(smem + sp.pz);

  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * nz;
  const size_t pb = (size_t)b * N2;
  const int txx = g.tx[2 * s], txz = g.tx[2 * s + 1];
  const int tid = threadIdx.x, T = blockDim.x;
  const int halo_n = (rows + 2) * nz;
  const int ncell = sl.nr * nz;

  for (int i = tid; i < halo_n; i += T) { P[0][i] = 0.f; P[1][i] = 0.f; }
  for (int i = tid; i < ncell; i += T) eds[nz + i] = m.Ed[pb + (size_t)sl.r0 * nz + i];
  for (int i = tid; i < sl.nr; i += T) pxs[i] = g.px ? g.px[sl.r0 + i] : 0.0;
  for (int i = tid; i < nz; i += T) pzs[i] = g.pz ? g.pz[i] : 0.0;
  cluster_barrier();

  for (int t = 0; t < g.nt; ++t) {
    const float* u1 = P[(t + 1) & 1];
    float* u2 = P[t & 1];
    const double pulse_t = g.pulse[t];
    float* rec_t = rec + ((size_t)t * U + lu) * g.M;
    for (int i = tid; i < ncell; i += T) {
      const int xr = i / nz + 1;
      const int z = i - (xr - 1) * nz;
      const int x = sl.r0 + xr - 1;
      const int k = xr * nz + z;
      const double uc = u1[k];
      const double xm = u1[k - nz], xp = u1[k + nz];
      const double zm = z > 0 ? (double)u1[k - 1] : 0.0;
      const double zp = z < nz - 1 ? (double)u1[k + 1] : 0.0;
      double lap;
      if (RHO) {
        const RhoW w = rho_weights(m.rho + pb, m.q + pb, g.nx, nz, x, z);
        lap = (((-w.W * uc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp;
      } else {
        lap = (((-4.0 * uc + xm) + xp) + zm) + zp;
      }
      double A, Bc;
      const double D = g.px ? fmax(pxs[xr - 1], pzs[z]) : g.d2d[(size_t)x * nz + z];
      ab_coeffs(D, g.dt, A, Bc);
      double v = A * uc + Bc * (double)u2[k] + eds[k] * lap;
      if (x == txx && z == txz) v += pulse_t;
      const float vf = (float)v;
      u2[k] = vf;
      push_halo(u2, sl, xr, z, nz, g.nx, vf);
      if (g.row_flag[x]) {
        const int slot = g.node_slot[(size_t)x * nz + z];
        if (slot >= 0) rec_t[slot] = vf;
      }
      if (MODE == 1) hist[((size_t)t * U + lu) * N2 + (size_t)x * nz + z] = vf;
      if (MODE == 2) {
        float* st = strips + ((size_t)t * U + lu) * g.SL;
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
    cluster_barrier();
  }
  if (MODE != 1) {
    // final two states for the adjoint's reconstruction, in the stepwise
    // engine's ping-pong layout: ubuf[t & 1][lu] holds u[t].
    for (int k2 = 0; k2 < 2; ++k2) {
      float* dst = ubuf + ((size_t)k2 * U + lu) * N2 + (size_t)sl.r0 * nz;
      const float* src = P[k2] + nz;
      for (int i = tid; i < ncell; i += T) dst[i] = src[i];
    }
  }
}

// ---------------------------------------------------------------------------
// adjoint sweep (MODE 1 full history / 2 strip reconstruction).  Writes the
// unit's imaging sum over time into acc_unit[lu][cell] (f64).
template <bool RHO, int MODE>
__global__ void __launch_bounds__(kClusterThreads, 1)
    cluster_adj_kernel(Geo g, Model m, int cs, int rows, int unit_begin, int U,
                       const double* __restrict__ rres, const float* __restrict__ hist,
                       const float* __restrict__ strips, const float* __restrict__ ubuf,
                       double* __restrict__ acc_unit, int acc_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Slab sl = my_slab(cs, rows, g.nx);
  const int nz = g.nz;
  const SmemPlan sp = smem_plan(rows, nz, true);
  float* Lb[2] = {reinterpret_cast<float*>(smem + sp.fA), reinterpret_cast<float*>(smem + sp.fB)};
  float* Ub[2] = {reinterpret_cast<float*>(smem + sp.fC), reinterpret_cast<float*>(smem + sp.fD)};
  double* eds = reinterpret_cast<double*>(smem + sp.ed);
  double* acc = reinterpret_cast<double*>(smem + sp.acc);
  double* pxs = reinterpret_cast<double*>(smem + sp.px);
  double* pzs = reinterpret_cast<double*>(smem + sp.pz);

  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * nz;
  const size_t pb = (size_t)b * N2;
  const int txx = g.tx[2 * s], txz = g.tx[2 * s + 1];
  const int tid = threadIdx.x, T = blockDim.x;
  const int halo_n = (rows + 2) * nz;
  const int ncell = sl.nr * nz;

  for (int i = tid; i < halo_n; i += T) {
    Lb[0][i] = 0.f;
    Lb[1][i] = 0.f;
    const int x = sl.r0 - 1 + i / nz;  // global row of this smem row
    const bool in = x >= 0 && x < g.nx && (i / nz) <= sl.nr + 1;
    double e = 0.0;
    if (in) e = m.Ed[pb + (size_t)x * nz + (i % nz)];
    eds[i] = e;
    if (MODE == 2) {
      Ub[0][i] = in ? ubuf[((size_t)0 * U + lu) * N2 + (size_t)x * nz + (i % nz)] : 0.f;
      Ub[1][i] = in ? ubuf[((size_t)1 * U + lu) * N2 + (size_t)x * nz + (i % nz)] : 0.f;
    }
  }
  for (int i = tid; i < ncell; i += T) acc[i] = 0.0;
  for (int i = tid; i < sl.nr; i += T) pxs[i] = g.px ? g.px[sl.r0 + i] : 0.0;
  for (int i = tid; i < nz; i += T) pzs[i] = g.pz ? g.pz[i] : 0.0;
  cluster_barrier();

  for (int t = g.nt - 1; t >= 0; --t) {
    const float* l1 = Lb[(t + 1) & 1];
    float* l2 = Lb[t & 1];
    float* ut = Ub[t & 1];          // u[t]   -> u[t-2] in place
    const float* um = Ub[(t + 1) & 1];  // u[t-1]
    const double* rr = rres + ((size_t)t * U + lu) * g.M;
    const float* st = MODE == 2 && t >= 1 ? strips + ((size_t)(t - 1) * U + lu) * g.SL : nullptr;
    const float* F = MODE == 1 && t >= 1 ? hist + ((size_t)(t - 1) * U + lu) * N2 : nullptr;
    const double pulse_t = g.pulse[t];
    for (int i = tid; i < ncell; i += T) {
      const int xr = i / nz + 1;
      const int z = i - (xr - 1) * nz;
      const int x = sl.r0 + xr - 1;
      const int k = xr * nz + z;
      const bool okzm = z > 0, okzp = z < nz - 1;
      double A, Bc;
      const double D = g.px ? fmax(pxs[xr - 1], pzs[z]) : g.d2d[(size_t)x * nz + z];
      ab_coeffs(D, g.dt, A, Bc);
      // lam[t] = A lam1 + L^T(E lam1) + B lam2  (+ residual)
      const double lc = l1[k];
      const double ec = eds[k];
      double adj;
      RhoW w{1.0, 1.0, 1.0, 1.0, 4.0};
      if (RHO) {
        const double* rho = m.rho + pb;
        const double* q = m.q + pb;
        const size_t c = (size_t)x * nz + z;
        w = rho_weights(rho, q, g.nx, nz, x, z);
        adj = -w.W * ec * lc;
        if (x > 0) adj += rho_in_weight(rho, q, c, c - nz) * eds[k - nz] * (double)l1[k - nz];
        if (x < g.nx - 1) adj += rho_in_weight(rho, q, c, c + nz) * eds[k + nz] * (double)l1[k + nz];
        if (okzm) adj += rho_in_weight(rho, q, c, c - 1) * eds[k - 1] * (double)l1[k - 1];
        if (okzp) adj += rho_in_weight(rho, q, c, c + 1) * eds[k + 1] * (double)l1[k + 1];
      } else {
        adj = -4.0 * ec * lc;
        adj += eds[k - nz] * (double)l1[k - nz];
        adj += eds[k + nz] * (double)l1[k + nz];
        if (okzm) adj += eds[k - 1] * (double)l1[k - 1];
        if (okzp) adj += eds[k + 1] * (double)l1[k + 1];
      }
      double lam = A * lc + adj + Bc * (double)l2[k];
      if (g.row_flag[x]) {
        const int slot = g.node_slot[(size_t)x * nz + z];
        if (slot >= 0) lam += rr[slot];
      }
      const float lf = (float)lam;
      l2[k] = lf;
      push_halo(l2, sl, xr, z, nz, g.nx, lf);
      if (t >= 1) {
        if (MODE == 1) {
          const size_t c = (size_t)x * nz + z;
          const double fc = F[c];
          const double xm = x > 0 ? (double)F[c - nz] : 0.0;
          const double xp = x < g.nx - 1 ? (double)F[c + nz] : 0.0;
          const double zm = okzm ? (double)F[c - 1] : 0.0;
          const double zp = okzp ? (double)F[c + 1] : 0.0;
          const double lapu = RHO ? ((((-w.W * fc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp)
                                  : ((((-4.0 * fc + xm) + xp) + zm) + zp);
          acc[i] += lapu * lam;
        } else if (x >= g.x_lo && x <= g.x_hi && z >= g.z_lo && z <= g.z_hi) {
          const double fc = um[k];
          const double xm = x > g.x_lo ? (double)um[k - nz] : (x > 0 ? (double)st[z - g.z_lo] : 0.0);
          const double xp = x < g.x_hi ? (double)um[k + nz]
                                       : (x < g.nx - 1 ? (double)st[g.Lz + z - g.z_lo] : 0.0);
          const double zm = z > g.z_lo ? (double)um[k - 1]
                                       : (z > 0 ? (double)st[2 * g.Lz + x - g.x_lo] : 0.0);
          const double zp = z < g.z_hi ? (double)um[k + 1]
                                       : (z < nz - 1 ? (double)st[2 * g.Lz + g.Lx + x - g.x_lo] : 0.0);
          const double lapu = RHO ? ((((-w.W * fc + w.xm * xm) + w.xp * xp) + w.zm * zm) + w.zp * zp)
                                  : ((((-4.0 * fc + xm) + xp) + zm) + zp);
          acc[i] += lapu * lam;
          if (t >= 2) {
            double prev = 2.0 * fc + ec * lapu - (double)ut[k];
            if (x == txx && z == txz) prev += pulse_t;
            const float pf = (float)prev;
            ut[k] = pf;
            push_halo(ut, sl, xr, z, nz, g.nx, pf);
          }
        }
      }
    }
    cluster_barrier();
  }
  double* dst = acc_unit + (size_t)(lu + acc_off) * N2 + (size_t)sl.r0 * nz;
  for (int i = tid; i < ncell; i += T) dst[i] = acc[i];
}

// ------------------------------------------------------------------ host side
template <class K>
inline bool cluster_fits(K kernel, int cs, size_t smem) {
  if (smem > 227 * 1024) return false;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return false;
  if (cs > 8 && cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

template <bool RHO>
inline bool cluster_config_t(const Geo& g, ClusterCfg* out) {
  // Prefer 16-CTA clusters (more SMs per unit, shortest per-step critical path),
  // fall back to smaller clusters only if shared memory demands it.
  for (int cs : {16, 8, 4}) {
    const int rows = (g.nx + cs - 1) / cs;
    if (rows < 2) continue;
    const size_t sf = smem_plan(rows, g.nz, false).total;
    const size_t sa = smem_plan(rows, g.nz, true).total;
    if (sa > 220 * 1024) continue;
    if (!cluster_fits(cluster_fwd_kernel<RHO, 0>, cs, sf)) continue;
    if (!cluster_fits(cluster_adj_kernel<RHO, 2>, cs, sa)) continue;
    cluster_fits(cluster_fwd_kernel<RHO, 1>, cs, sf);
    cluster_fits(cluster_fwd_kernel<RHO, 2>, cs, sf);
    cluster_fits(cluster_adj_kernel<RHO, 1>, cs, sa);
    out->cs = cs;
    out->rows = rows;
    out->threads = kClusterThreads;
    out->smem_fwd = sf;
    out->smem_adj = sa;
    return true;
  }
  return false;
}

inline bool cluster_config(const Geo& g, bool rho, ClusterCfg* out) {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return false; }
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess || major < 10) {
    cudaGetLastError();
    return false;
  }
  return rho ? cluster_config_t<true>(g, out) : cluster_config_t<false>(g, out);
}

template <class K, class... Args>
inline cudaError_t launch_cluster(K kernel, const ClusterCfg& c, int U, size_t smem,
                                  cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(U * c.cs);
  cfg.blockDim = dim3(c.threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

inline int cluster_forward(const Geo& g, const Model& m, const ClusterCfg& c, bool rho, int mode,
                           int unit_begin, int U, float* rec, float* hist, float* strips,
                           float* ubuf, cudaStream_t st) {
  cudaError_t e;
#define DUFWI_CF(R, M)                                                                      \
  e = launch_cluster(cluster_fwd_kernel<R, M>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,    \
                     unit_begin, U, rec, hist, strips, ubuf)
  if (rho) {
    if (mode == 0) DUFWI_CF(true, 0); else if (mode == 1) DUFWI_CF(true, 1); else DUFWI_CF(true, 2);
  } else {
    if (mode == 0) DUFWI_CF(false, 0); else if (mode == 1) DUFWI_CF(false, 1); else DUFWI_CF(false, 2);
  }
#undef DUFWI_CF
  return (int)e;
}

inline int cluster_adjoint(const Geo& g, const Model& m, const ClusterCfg& c, bool rho, int mode,
                           int unit_begin, int U, const double* rres, const float* hist,
                           const float* strips, const float* ubuf, double* acc_part, int acc_off,
                           cudaStream_t st) {
  cudaError_t e;
#define DUFWI_CA(R, M)                                                                      \
  e = launch_cluster(cluster_adj_kernel<R, M>, c, U, c.smem_adj, st, g, m, c.cs, c.rows,    \
                     unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off)
  if (rho) {
    if (mode == 1) DUFWI_CA(true, 1); else DUFWI_CA(true, 2);
  } else {
    if (mode == 1) DUFWI_CA(false, 1); else DUFWI_CA(false, 2);
  }
#undef DUFWI_CA
  return (int)e;
}

}  // namespace dufwi
