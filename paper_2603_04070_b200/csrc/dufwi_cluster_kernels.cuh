// Cluster engine: one kernel launch per sweep, one thread-block cluster per unit.
//
// For grids whose per-unit state fits a cluster (configs 0/1: 160^2) the whole
// time loop of a sweep runs inside one launch ("temporal blocking in the
// extreme").  The unit's grid is cut into `cs` slabs of `rows`
// x-rows, one per CTA.  Inside a CTA thread (seg, z) owns column z of rows
// [seg*RPT, seg*RPT+RPT): its cells' state (u[t-1], u[t-2] forward; lam[t+1],
// lam[t+2], u[t], u[t-1] adjoint), E/dx^2 and the imaging accumulators live in
// f64 REGISTERS for the whole sweep.  Per time step a thread
//   * reads z-neighbours from a double-buffered shared-memory exchange row,
//   * takes x-neighbours from its own registers, from the exchange rows of the
//     adjacent segment, or from the halo rows of the buffer,
//   * writes its new value into the exchange buffer; threads owning the slab's
//     first/last row also push it into the neighbouring CTA's halo row with
//     st.async (DSMEM), completing bytes on that CTA's mbarrier.
// A step then costs one __syncthreads and one mbarrier phase wait — no
// cluster-wide barrier, no GPU-scope fence, no L1 invalidation.  HBM only sees
// receiver samples, the 1-cell ring strips and the final two states.
//
// Numerics: f64 state and arithmetic in the reference's operation order; the
// exchange rows are f64 when they fit shared memory (T = double), making the
// sweep a plain float64 computation; receiver samples, strips and the final
// states are stored f32 (the ChannelData/workspace format).
#pragma once

#include <cooperative_groups.h>

#include "dufwi_common.cuh"

namespace dufwi {

namespace cg = cooperative_groups;
#ifdef DUFWI_EXP_TIMING
__device__ unsigned long long g_dbg[256];
#endif

struct ClusterCfg {
  int cs = 0;       // CTAs per cluster (slabs per unit)
  int rows = 0;     // x-rows per slab
  int rpt = 0;      // rows per thread (template instance)
  int nseg = 0;     // thread segments per column
  int threads = 0;  // threads per CTA = nz * nseg
  int dbl = 0;      // exchange rows in f64 (1) or f32 (0)
  int maxrec = 0;   // receiver cells per CTA (upper bound) staged in shared memory
  int maxring = 0;  // ring-strip cells per CTA (upper bound) staged in shared memory
  size_t smem_fwd = 0, smem_adj = 0;
};

// Receiver samples / ring strips / residuals move between HBM and the step loop
// through shared-memory stages of kStage steps: written (forward) or read
// (adjoint) with one coalesced pass per kStage steps instead of scattered
// global accesses inside every step.
constexpr int kStage = 16;

constexpr int kClusterMaxThreads = 512;  // 128 registers per thread available

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; "
      "@!p bra WAIT_%=; }" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void push_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void push_async(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
// Predicated push: keeps the value in a register (no run-time register indexing).
__device__ __forceinline__ void push_if(uint32_t on, uint32_t raddr, double v, uint32_t rbar) {
  asm volatile(
      "{ .reg .pred q; setp.ne.u32 q, %3, 0; "
      "@q st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2]; }" ::"r"(raddr),
      "l"(__double_as_longlong(v)), "r"(rbar), "r"(on)
      : "memory");
}
__device__ __forceinline__ void push_if(uint32_t on, uint32_t raddr, float v, uint32_t rbar) {
  asm volatile(
      "{ .reg .pred q; setp.ne.u32 q, %3, 0; "
      "@q st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2]; }" ::"r"(raddr),
      "r"(__float_as_uint(v)), "r"(rbar), "r"(on)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// One thread moves a whole exchange row into a neighbour CTA's halo row and
// completes the bytes on that CTA's mbarrier (async proxy).
__device__ __forceinline__ void push_row(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                         uint32_t bar_cluster) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_addr(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ------------------------------------------------------------ smem layout
// [nbufs exchange buffers of (rows+2) x (nz+2) T] [rows x nz double2 (A, B)] [2 mbarriers]
// Exchange row stride: nz + 2 pad columns, rounded so every row starts on a
// 16-byte boundary (bulk DSMEM copies move whole rows).
template <class T>
__host__ __device__ inline int xstride(int nz) {
  const int q = 16 / (int)sizeof(T);
  return (nz + 2 + q - 1) / q * q;
}
template <class T>
__host__ __device__ inline size_t xbuf_elems(int rows, int nz) {
  return (size_t)(rows + 2) * xstride<T>(nz);
}
template <class T>
__host__ __device__ inline size_t ab_offset(int rows, int nz, int nbufs) {
  return ((size_t)nbufs * xbuf_elems<T>(rows, nz) * sizeof(T) + 15) & ~(size_t)15;
}
template <class T>
__host__ __device__ inline size_t bar_offset(int rows, int nz, int nbufs) {
  return ab_offset<T>(rows, nz, nbufs) + (size_t)rows * nz * sizeof(double2);
}
// IO stage after the mbarriers: [n_rec, n_ring, pad] [rec_g[maxrec]] [ring_g[maxring]]
// [double stage_rec[kStage][maxrec]] [float stage_ring[kStage][maxring]]
struct IoStage {
  int* counts;
  int* rec_g;
  int* ring_g;
  double* srec;
  float* sring;
  int maxrec, maxring;
};

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

template <class T>
__host__ __device__ inline size_t io_offset(int rows, int nz, int nbufs) {
  return al16(bar_offset<T>(rows, nz, nbufs) + 2 * sizeof(uint64_t));
}

__host__ __device__ inline size_t io_bytes(int maxrec, int maxring) {
  return 16 + al16((size_t)maxrec * 4) + al16((size_t)maxring * 4) +
         al16((size_t)kStage * maxrec * 8) + al16((size_t)kStage * maxring * 4);
}

template <class T>
__host__ __device__ inline size_t cluster_smem_bytes(int rows, int nz, int nbufs, int maxrec,
                                                     int maxring) {
  return io_offset<T>(rows, nz, nbufs) + io_bytes(maxrec, maxring);
}

__device__ __forceinline__ IoStage io_stage(unsigned char* base, int maxrec, int maxring) {
  IoStage io;
  io.counts = reinterpret_cast<int*>(base);
  size_t o = 16;
  io.rec_g = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxrec * 4);
  io.ring_g = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxring * 4);
  io.srec = reinterpret_cast<double*>(base + o);
  o += al16((size_t)kStage * maxrec * 8);
  io.sring = reinterpret_cast<float*>(base + o);
  io.maxrec = maxrec;
  io.maxring = maxring;
  return io;
}

// Per-thread static description of its cells.
struct CellCtx {
  int rank, cs, rows, nr, r0;  // slab of this CTA: global rows [r0, r0+nr)
  int seg, z, lrow0;           // thread: column z, local rows lrow0 .. lrow0+RPT-1
  int W;                       // exchange row stride (>= nz + 2, 16-byte rows)
  int seg_last;                // segment owning the slab's last row
  bool has_up, has_dn;         // CTA rank-1 / rank+1 exist with rows
};

__device__ __forceinline__ CellCtx make_ctx(int cs, int rows, int nx, int nz, int rpt, int W) {
  CellCtx c;
  c.rank = (int)cg::this_cluster().block_rank();
  c.cs = cs;
  c.rows = rows;
  c.r0 = c.rank * rows;
  c.nr = max(0, min(nx, c.r0 + rows) - c.r0);
  c.seg = threadIdx.x / nz;
  c.z = threadIdx.x - c.seg * nz;
  c.lrow0 = c.seg * rpt;
  c.W = W;
  c.seg_last = c.nr > 0 ? (c.nr - 1) / rpt : 0;
  c.has_up = c.rank > 0 && c.nr > 0;
  c.has_dn = c.nr > 0 && c.rank + 1 < cs && (c.rank + 1) * rows < nx;
  return c;
}

// Ring-strip slot of cell (x, z) (layout of the stepwise engine), or -1.
__device__ __forceinline__ int ring_index(const Geo& g, int x, int z) {
  if (z >= g.z_lo && z <= g.z_hi) {
    if (x == g.x_lo - 1) return z - g.z_lo;
    if (x == g.x_hi + 1) return g.Lz + z - g.z_lo;
  }
  if (x >= g.x_lo && x <= g.x_hi) {
    if (z == g.z_lo - 1) return 2 * g.Lz + x - g.x_lo;
    if (z == g.z_hi + 1) return 2 * g.Lz + g.Lx + x - g.x_lo;
  }
  return -1;
}

__device__ __forceinline__ bool in_box(const Geo& g, int x, int z) {
  return x >= g.x_lo && x <= g.x_hi && z >= g.z_lo && z <= g.z_hi;
}

// Static per-cell data loaded once per sweep.
template <int RPT>
struct CellStatic {
  double ed[RPT];
  int rl[RPT];  // receiver cell: local index into the IO stage, else -1
  int gl[RPT];  // ring cell: local index into the IO stage, else -1
  unsigned active, src, interior;
  bool pushes_up, pushes_dn;  // owns the slab's first / last row
  unsigned dn_mask;           // bit j set: register j holds the slab's last row (pushes_dn)
  bool special;               // any receiver / ring / source / push / history cell
  bool undamped;              // every cell has D == 0: (A, B) = (2, -1), no table reads
  const double2* ab;          // shared (A, B) table, row stride nz
};

template <int RPT>
__device__ __forceinline__ void load_static(const Geo& g, const Model& m, const CellCtx& c,
                                            size_t pb, int txx, int txz, double2* ab_table,
                                            const IoStage& io, CellStatic<RPT>& st) {
  st.active = st.src = st.interior = 0u;
  st.ab = ab_table;
  st.pushes_up = c.has_up && c.lrow0 == 0;
  st.pushes_dn = false;
  st.dn_mask = 0u;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = c.lrow0 + j;
    st.ed[j] = 0.0;
    st.rl[j] = -1;
    st.gl[j] = -1;
    if (lr < c.nr) {
      const int x = c.r0 + lr;
      st.active |= 1u << j;
      st.ed[j] = m.Ed[pb + (size_t)x * g.nz + c.z];
      double A, B;
      ab_coeffs(damping_at(g, x, c.z), g.dt, A, B);
      ab_table[(size_t)lr * g.nz + c.z] = make_double2(A, B);
      const int slot = g.row_flag[x] ? g.node_slot[(size_t)x * g.nz + c.z] : -1;
      if (slot >= 0) {
        st.rl[j] = atomicAdd(&io.counts[0], 1);  // storage slot only: order does not matter
        io.rec_g[st.rl[j]] = slot;
      }
      const int ring = ring_index(g, x, c.z);
      if (ring >= 0 && io.maxring > 0) {
        st.gl[j] = atomicAdd(&io.counts[1], 1);
        io.ring_g[st.gl[j]] = ring;
      }
      if (x == txx && c.z == txz) st.src |= 1u << j;
      if (in_box(g, x, c.z)) st.interior |= 1u << j;
      if (lr == c.nr - 1 && c.has_dn) {
        st.pushes_dn = true;
        st.dn_mask = 1u << j;
      }
    }
  }
  st.undamped = true;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (c.lrow0 + j < c.nr && damping_at(g, c.r0 + c.lrow0 + j, c.z) != 0.0) st.undamped = false;
  bool any = st.src != 0u;
#pragma unroll
  for (int j = 0; j < RPT; ++j) any = any || st.rl[j] >= 0 || st.gl[j] >= 0;
  st.special = any;
}

// x-neighbours of cell j of a thread column: register when the neighbour is the
// thread's own cell, else the exchange buffer row (adjacent segment or halo).
// Row index in the buffer is lr + 1 (row 0 = top halo).
template <int RPT, class T>
__device__ __forceinline__ void x_neighbours(const CellCtx& c, const double (&v)[RPT],
                                             const T* X, double (&xm)[RPT], double (&xp)[RPT]) {
  const int W = c.W, z = c.z;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = min(c.lrow0 + j, c.rows - 1);
    xm[j] = j > 0 ? v[j - 1] : (double)X[(size_t)lr * W + z + 1];
    const bool own_next = j < RPT - 1 && c.lrow0 + j + 1 < c.nr;
    xp[j] = own_next ? v[j + 1] : (double)X[(size_t)(lr + 2) * W + z + 1];
  }
}

// Bulk halo exchange: the threads owning the slab's first (last) row sync on a
// named barrier, then one of them copies the whole row into the halo row of
// CTA rank-1 (rank+1).  Needs nz % 32 == 0 so a row's threads are whole warps.
template <class T>
__device__ __forceinline__ void push_rows(const CellCtx& c, int nz, T* Xw, uint32_t bar_w) {
  const uint32_t bytes = (uint32_t)(c.W * sizeof(T));
  if (c.has_up && c.seg == 0) {
    named_sync(1, nz);
    if (threadIdx.x == 0)
      push_row(mapa_rank(smem_addr(Xw + (size_t)(c.rows + 1) * c.W), c.rank - 1), Xw + (size_t)c.W,
               bytes, mapa_rank(bar_w, c.rank - 1));
  }
  if (c.has_dn && c.seg == c.seg_last) {
    named_sync(2, nz);
    if (threadIdx.x == c.seg_last * nz)
      push_row(mapa_rank(smem_addr(Xw), c.rank + 1), Xw + (size_t)c.nr * c.W, bytes,
               mapa_rank(bar_w, c.rank + 1));
  }
}

// ---------------------------------------------------------------------------
// forward step i (time t = i).  u1 = u[t-1] (read), u2 = u[t-2] -> u[t].
// Reads exchange buffer Xr (step i-1), writes Xw (step i) and pushes the slab's
// boundary rows into the neighbours' Xw halo rows (mbarrier `bar_w` remote).
template <int RPT, class T, int MODE>
__device__ __forceinline__ void fwd_step(const Geo& g, const CellCtx& c, const CellStatic<RPT>& s,
                                         double (&u1)[RPT], double (&u2)[RPT], int t, int U,
                                         int lu, const T* Xr, T* Xw, uint32_t bar_r,
                                         uint32_t bar_w, uint32_t tx_bytes, double pulse_t,
                                         const IoStage& io, float* __restrict__ hist, size_t N2,
                                         bool bulk) {
  const int W = c.W, z = c.z;
#ifdef DUFWI_EXP_TIMING
  const bool tm = blockIdx.x == 5 && (threadIdx.x & 31) == 0;
  long long T0 = clock64();
#endif
#ifndef DUFWI_EXP_NOSYNC
  __syncthreads();  // exchange rows of step i-1 complete; Xw free for reuse
#endif
#ifdef DUFWI_EXP_TIMING
  long long T1 = clock64();
#endif
#ifndef DUFWI_EXP_NOWAIT
  if (t >= 1 && (c.has_up || c.has_dn)) mbar_wait(bar_r, ((t - 1) >> 1) & 1);
#endif
#ifdef DUFWI_EXP_TIMING
  long long T2 = clock64();
#endif
  if (threadIdx.x == 0 && (c.has_up || c.has_dn)) mbar_expect_tx(bar_w, tx_bytes);
  double xm[RPT], xp[RPT], zm[RPT], zp[RPT], v[RPT];
#ifdef DUFWI_EXP_NOLDS
#pragma unroll
  for (int j = 0; j < RPT; ++j) { xm[j] = xp[j] = zm[j] = zp[j] = u1[j] * 0.25; }
#else
  x_neighbours<RPT, T>(c, u1, Xr, xm, xp);
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = min(c.lrow0 + j, c.rows - 1);
    zm[j] = (double)Xr[(size_t)(lr + 1) * W + z];
    zp[j] = (double)Xr[(size_t)(lr + 1) * W + z + 2];
  }
#endif
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const double lap = (((-4.0 * u1[j] + xm[j]) + xp[j]) + zm[j]) + zp[j];
    const double2 ab = s.undamped ? make_double2(2.0, -1.0) : s.ab[(size_t)min(c.lrow0 + j, c.rows - 1) * g.nz + z];
#ifdef DUFWI_EXP_NOCOMPUTE
    v[j] = u1[j] + zm[j];
#else
    v[j] = ab.x * u1[j] + ab.y * u2[j] + s.ed[j] * lap;
#endif
    if (s.src & (1u << j)) v[j] += pulse_t;
  }
  // common path: state and exchange row (inactive rows only exist in the last segment)
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!(s.active & (1u << j))) continue;
    u2[j] = v[j];
    Xw[(size_t)(c.lrow0 + j + 1) * W + z + 1] = (T)v[j];
  }
#ifdef DUFWI_EXP_TIMING
  long long T3 = clock64();
  if (tm) {
    const int w = threadIdx.x >> 5;
    atomicAdd(&g_dbg[w * 4 + 0], (unsigned long long)(T1 - T0));
    atomicAdd(&g_dbg[w * 4 + 1], (unsigned long long)(T2 - T1));
    atomicAdd(&g_dbg[w * 4 + 2], (unsigned long long)(T3 - T2));
  }
#endif
  // halo rows to the neighbouring CTAs
  if (bulk) {
    push_rows<T>(c, g.nz, Xw, bar_w);
  } else {
    if (s.pushes_up)  // my first row -> bottom halo of rank-1
      push_async(mapa_rank(smem_addr(Xw + (size_t)(c.rows + 1) * W + z + 1), c.rank - 1), (T)v[0],
                 mapa_rank(bar_w, c.rank - 1));
    if (s.pushes_dn) {  // my last row -> top halo of rank+1
      const uint32_t ra = mapa_rank(smem_addr(Xw + z + 1), c.rank + 1);
      const uint32_t rb = mapa_rank(bar_w, c.rank + 1);
      // explicit predicate per register so v[] is never indexed at run time
#pragma unroll
      for (int j = 0; j < RPT; ++j) push_if((s.dn_mask >> j) & 1u, ra, (T)v[j], rb);
    }
  }
  if (!s.special) return;
  // rare path: receivers, history / ring strips
  const int k = t % kStage;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!(s.active & (1u << j))) continue;
    const float vf = (float)v[j];
    if (s.rl[j] >= 0) io.srec[k * io.maxrec + s.rl[j]] = (double)vf;
    if (MODE == 1) hist[((size_t)t * U + lu) * N2 + (size_t)(c.r0 + c.lrow0 + j) * g.nz + z] = vf;
    if (MODE == 2 && s.gl[j] >= 0) io.sring[k * io.maxring + s.gl[j]] = vf;
  }
#ifdef DUFWI_EXP_TIMING
  if (tm) atomicAdd(&g_dbg[(threadIdx.x >> 5) * 4 + 3], (unsigned long long)(clock64() - T3));
#endif
}

// Write the staged receiver samples / ring strips of steps [t0, t0+nk) to HBM.
template <int MODE>
__device__ __forceinline__ void flush_stage(const Geo& g, const IoStage& io, int t0, int nk, int U,
                                            int lu, float* __restrict__ rec,
                                            float* __restrict__ strips) {
  __syncthreads();
  const int nrec = io.counts[0], nring = io.counts[1];
  for (int idx = threadIdx.x; idx < nk * nrec; idx += blockDim.x) {
    const int k = idx / nrec, i = idx - k * nrec;
    rec[((size_t)(t0 + k) * U + lu) * g.M + io.rec_g[i]] = (float)io.srec[k * io.maxrec + i];
  }
  if (MODE == 2) {
    for (int idx = threadIdx.x; idx < nk * nring; idx += blockDim.x) {
      const int k = idx / nring, i = idx - k * nring;
      strips[((size_t)(t0 + k) * U + lu) * g.SL + io.ring_g[i]] = io.sring[k * io.maxring + i];
    }
  }
}

template <int RPT, class T, int MODE>
__global__ void __launch_bounds__(kClusterMaxThreads, 1)
    cluster_fwd_kernel(Geo g, Model m, int cs, int rows, int maxrec, int maxring,
                       int unit_begin, int U, float* __restrict__ rec, float* __restrict__ hist,
                       float* __restrict__ strips, float* __restrict__ ubuf) {
  extern __shared__ __align__(16) unsigned char smem[];
  const CellCtx c = make_ctx(cs, rows, g.nx, g.nz, RPT, xstride<T>(g.nz));
  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t pb = (size_t)b * N2;
  const size_t xe = xbuf_elems<T>(rows, g.nz);
  T* X[2] = {reinterpret_cast<T*>(smem), reinterpret_cast<T*>(smem) + xe};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_offset<T>(rows, g.nz, 2));
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  for (size_t i = threadIdx.x; i < 2 * xe; i += blockDim.x) X[0][i] = T(0);
  const IoStage io = io_stage(smem + io_offset<T>(rows, g.nz, 2), maxrec, maxring);
  if (threadIdx.x == 0) {
    mbar_init(bar[0], 1);
    mbar_init(bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    io.counts[0] = io.counts[1] = 0;
  }
  __syncthreads();
  CellStatic<RPT> st;
  load_static<RPT>(g, m, c, pb, g.tx[2 * s], g.tx[2 * s + 1],
                   reinterpret_cast<double2*>(smem + ab_offset<T>(rows, g.nz, 2)), io, st);
  if (MODE == 1) st.special = true;  // every cell goes to the history
  const bool bulk = false;  // measured slower than per-thread st.async (named-barrier + bulk-copy latency)
  const uint32_t tx_bytes =
      (uint32_t)((c.has_up ? 1 : 0) + (c.has_dn ? 1 : 0)) * (bulk ? c.W : g.nz) * sizeof(T);
  double ua[RPT], ub[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) ua[j] = ub[j] = 0.0;
  const bool owns_src = st.src != 0u;
  double p_next = owns_src ? g.pulse[0] : 0.0;
  cluster_sync_all();  // barriers initialised and buffers zeroed cluster-wide

  // step t writes X[t & 1] / bar[t & 1]; ub receives u[t] at even t, ua at odd t
  int t = 0;
  for (; t + 1 < g.nt; t += 2) {
    double p = p_next;
    if (owns_src) p_next = g.pulse[t + 1];
    fwd_step<RPT, T, MODE>(g, c, st, ua, ub, t, U, lu, X[1], X[0], bar[1], bar[0], tx_bytes, p,
                           io, hist, N2, bulk);
    p = p_next;
    if (owns_src && t + 2 < g.nt) p_next = g.pulse[t + 2];
    fwd_step<RPT, T, MODE>(g, c, st, ub, ua, t + 1, U, lu, X[0], X[1], bar[0], bar[1], tx_bytes, p,
                           io, hist, N2, bulk);
    if ((t + 2) % kStage == 0) flush_stage<MODE>(g, io, t + 2 - kStage, kStage, U, lu, rec, strips);
  }
  if (t < g.nt)
    fwd_step<RPT, T, MODE>(g, c, st, ua, ub, t, U, lu, X[1], X[0], bar[1], bar[0], tx_bytes,
                           p_next, io, hist, N2, bulk);
  if (g.nt % kStage) {
    const int t0 = g.nt - g.nt % kStage;
    flush_stage<MODE>(g, io, t0, g.nt - t0, U, lu, rec, strips);
  }
  // drain the last step's incoming pushes before any CTA of the cluster exits
  if (c.has_up || c.has_dn) mbar_wait(bar[(g.nt - 1) & 1], ((g.nt - 1) >> 1) & 1);
  cluster_sync_all();

  if (MODE != 1) {
    // final two states in the stepwise-engine layout: ubuf[t & 1][lu] holds u[t]
    const bool last_odd = ((g.nt - 1) & 1) != 0;
    float* d_last = ubuf + ((size_t)((g.nt - 1) & 1) * U + lu) * N2;
    float* d_prev = ubuf + ((size_t)((g.nt - 2) & 1) * U + lu) * N2;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (!(st.active & (1u << j))) continue;
      const size_t cell = (size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z;
      d_last[cell] = (float)(last_odd ? ua[j] : ub[j]);
      d_prev[cell] = (float)(last_odd ? ub[j] : ua[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// adjoint step i (time t = nt-1-i).  l1 = lam[t+1], l2 = lam[t+2] -> lam[t];
// ua = u[t] -> u[t-2] (reconstruction, MODE 2), ub = u[t-1].
// XL: exchange of E*lam, XU: exchange of u (MODE 2).  Buffers/bars indexed by i.
template <int RPT, class T, int MODE>
__device__ __forceinline__ void adj_step(const Geo& g, const CellCtx& c, const CellStatic<RPT>& s,
                                         double (&l1)[RPT], double (&l2)[RPT], double (&ua)[RPT],
                                         double (&ub)[RPT], double (&acc)[RPT], int i, int U,
                                         int lu, const T* XLr, T* XLw, const T* XUr, T* XUw,
                                         uint32_t bar_r, uint32_t bar_w, uint32_t tx_bytes,
                                         double pulse_t, const IoStage& io,
                                         const float* __restrict__ hist, size_t N2, bool bulk) {
  const int W = c.W, z = c.z;
  const int t = g.nt - 1 - i;
  __syncthreads();
  // residuals / ring values of this step from the shared-memory stage
  double rr[RPT];
  float ring_v[RPT];
  const int k = i % kStage;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    rr[j] = s.rl[j] >= 0 ? io.srec[k * io.maxrec + s.rl[j]] : 0.0;
    ring_v[j] = (MODE == 2 && s.gl[j] >= 0) ? io.sring[k * io.maxring + s.gl[j]] : 0.f;
  }
  if (i >= 1 && (c.has_up || c.has_dn)) mbar_wait(bar_r, ((i - 1) >> 1) & 1);
  if (threadIdx.x == 0 && (c.has_up || c.has_dn)) mbar_expect_tx(bar_w, tx_bytes);

  // lam[t] = A lam1 + L^T(E lam1) + B lam2 (+ residual), reference order
  double el[RPT], xm[RPT], xp[RPT], lam[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) el[j] = s.ed[j] * l1[j];
  x_neighbours<RPT, T>(c, el, XLr, xm, xp);
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = min(c.lrow0 + j, c.rows - 1);
    const size_t o = (size_t)(lr + 1) * W + z + 1;
    const double adj = (((-4.0 * el[j] + xm[j]) + xp[j]) + (double)XLr[o - 1]) + (double)XLr[o + 1];
    const double2 ab = s.undamped ? make_double2(2.0, -1.0) : s.ab[(size_t)lr * g.nz + z];
    lam[j] = ab.x * l1[j] + adj + ab.y * l2[j] + rr[j];
  }
  // imaging with L(u[t-1]) and reconstruction of u[t-2]
  double lapu[RPT];
  if (MODE == 2) {
    double fxm[RPT], fxp[RPT];
    x_neighbours<RPT, T>(c, ub, XUr, fxm, fxp);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int lr = min(c.lrow0 + j, c.rows - 1);
      const size_t o = (size_t)(lr + 1) * W + z + 1;
      lapu[j] = (((-4.0 * ub[j] + fxm[j]) + fxp[j]) + (double)XUr[o - 1]) + (double)XUr[o + 1];
    }
  } else {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      lapu[j] = 0.0;
      if (t >= 1 && (s.active & (1u << j))) {
        const float* F = hist + ((size_t)(t - 1) * U + lu) * N2;
        const int x = c.r0 + c.lrow0 + j;
        const size_t cell = (size_t)x * g.nz + z;
        const double fxm = x > 0 ? (double)F[cell - g.nz] : 0.0;
        const double fxp = x < g.nx - 1 ? (double)F[cell + g.nz] : 0.0;
        const double fzm = z > 0 ? (double)F[cell - 1] : 0.0;
        const double fzp = z < g.nz - 1 ? (double)F[cell + 1] : 0.0;
        lapu[j] = (((-4.0 * (double)F[cell] + fxm) + fxp) + fzm) + fzp;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!(s.active & (1u << j))) continue;
    const int lr = c.lrow0 + j;
    const size_t o = (size_t)(lr + 1) * W + z + 1;
    l2[j] = lam[j];
    const T elw = (T)(s.ed[j] * lam[j]);
    XLw[o] = elw;
    if (t >= 1) {
      if (MODE == 1) {
        acc[j] += lapu[j] * lam[j];
      } else if (s.interior & (1u << j)) {
        acc[j] += lapu[j] * lam[j];
        if (t >= 2) {
          double prev = 2.0 * ub[j] + s.ed[j] * lapu[j] - ua[j];
          if (s.src & (1u << j)) prev += pulse_t;
          ua[j] = prev;
        }
      } else if (s.gl[j] >= 0 && t >= 2) {
        ua[j] = (double)ring_v[j];  // ring cell: the saved strip stands in for the reconstruction
      }
    }
    if (MODE == 2) XUw[o] = (T)ua[j];
  }
  // halo rows to the neighbouring CTAs
  if (bulk) {
    push_rows<T>(c, g.nz, XLw, bar_w);
    if (MODE == 2) push_rows<T>(c, g.nz, XUw, bar_w);
    return;
  }
  if (s.pushes_up) {
    const uint32_t rb = mapa_rank(bar_w, c.rank - 1);
    const size_t ho = (size_t)(c.rows + 1) * W + z + 1;
    push_async(mapa_rank(smem_addr(XLw + ho), c.rank - 1), (T)(s.ed[0] * l2[0]), rb);
    if (MODE == 2) push_async(mapa_rank(smem_addr(XUw + ho), c.rank - 1), (T)ua[0], rb);
  }
  if (s.pushes_dn) {
    const uint32_t rb = mapa_rank(bar_w, c.rank + 1);
    const uint32_t ral = mapa_rank(smem_addr(XLw + z + 1), c.rank + 1);
    const uint32_t rau = mapa_rank(smem_addr(XUw + z + 1), c.rank + 1);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const uint32_t on = (s.dn_mask >> j) & 1u;
      push_if(on, ral, (T)(s.ed[j] * l2[j]), rb);
      if (MODE == 2) push_if(on, rau, (T)ua[j], rb);
    }
  }
}

// Load residuals of steps [i0, i0+kStage) (t = nt-1-i) and the ring strips they
// reconstruct from (t-2) into the shared-memory stage, one coalesced pass.
template <int MODE>
__device__ __forceinline__ void prefetch_stage(const Geo& g, const IoStage& io, int i0, int U,
                                               int lu, const double* __restrict__ rres,
                                               const float* __restrict__ strips) {
  __syncthreads();  // the previous block's readers are done with the stage
  const int nk = min(kStage, g.nt - i0);
  const int nrec = io.counts[0], nring = io.counts[1];
  for (int idx = threadIdx.x; idx < nk * nrec; idx += blockDim.x) {
    const int k = idx / nrec, r = idx - k * nrec;
    const int t = g.nt - 1 - (i0 + k);
    io.srec[k * io.maxrec + r] = rres[((size_t)t * U + lu) * g.M + io.rec_g[r]];
  }
  if (MODE == 2) {
    for (int idx = threadIdx.x; idx < nk * nring; idx += blockDim.x) {
      const int k = idx / nring, r = idx - k * nring;
      const int t = g.nt - 1 - (i0 + k);
      io.sring[k * io.maxring + r] = t >= 2 ? strips[((size_t)(t - 2) * U + lu) * g.SL + io.ring_g[r]] : 0.f;
    }
  }
}

template <int RPT, class T, int MODE>
__global__ void __launch_bounds__(kClusterMaxThreads, 1)
    cluster_adj_kernel(Geo g, Model m, int cs, int rows, int maxrec, int maxring,
                       int unit_begin, int U,
                       const double* __restrict__ rres, const float* __restrict__ hist,
                       const float* __restrict__ strips, const float* __restrict__ ubuf,
                       double* __restrict__ acc_part, int acc_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  const CellCtx c = make_ctx(cs, rows, g.nx, g.nz, RPT, xstride<T>(g.nz));
  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t pb = (size_t)b * N2;
  const int W = c.W;
  const size_t xe = xbuf_elems<T>(rows, g.nz);
  T* base = reinterpret_cast<T*>(smem);
  T* XL[2] = {base, base + xe};
  T* XU[2] = {base + 2 * xe, base + 3 * xe};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_offset<T>(rows, g.nz, 4));
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  for (size_t k = threadIdx.x; k < 4 * xe; k += blockDim.x) base[k] = T(0);
  const IoStage io = io_stage(smem + io_offset<T>(rows, g.nz, 4), maxrec, maxring);
  if (threadIdx.x == 0) {
    mbar_init(bar[0], 1);
    mbar_init(bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    io.counts[0] = io.counts[1] = 0;
  }
  __syncthreads();
  CellStatic<RPT> st;
  load_static<RPT>(g, m, c, pb, g.tx[2 * s], g.tx[2 * s + 1],
                   reinterpret_cast<double2*>(smem + ab_offset<T>(rows, g.nz, 4)), io, st);
  const int per = MODE == 2 ? 2 : 1;
  const bool bulk = false;  // measured slower than per-thread st.async (named-barrier + bulk-copy latency)
  const uint32_t tx_bytes =
      (uint32_t)(per * ((c.has_up ? 1 : 0) + (c.has_dn ? 1 : 0)) * (bulk ? c.W : g.nz) * sizeof(T));
  const int nt = g.nt;
  const float* u_last = ubuf + ((size_t)((nt - 1) & 1) * U + lu) * N2;
  const float* u_prev = ubuf + ((size_t)((nt - 2) & 1) * U + lu) * N2;
  __syncthreads();  // zero fill done before the u[nt-2] exchange rows are written
  // step i = 0 reads XU[1] = u[nt-2] (own rows and both halo rows from global)
  if (MODE == 2 && c.nr > 0) {
    for (int k = threadIdx.x; k < (c.nr + 2) * g.nz; k += blockDim.x) {
      const int r = k / g.nz, zz = k - r * g.nz;
      const int x = c.r0 - 1 + r;
      if (x >= 0 && x < g.nx) XU[1][(size_t)r * W + zz + 1] = (T)u_prev[(size_t)x * g.nz + zz];
    }
  }
  double la[RPT], lb[RPT], ua[RPT], ub[RPT], acc[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    la[j] = lb[j] = acc[j] = ua[j] = ub[j] = 0.0;
    if (MODE == 2 && (st.active & (1u << j))) {
      const size_t cell = (size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z;
      ua[j] = u_last[cell];
      ub[j] = u_prev[cell];
    }
  }
  const bool owns_src = st.src != 0u;
  cluster_sync_all();

  // step i writes XL[i&1], XU[i&1], bar[i&1]; reads XL[(i+1)&1], XU[(i+1)&1], bar[(i+1)&1]
  int i = 0;
  for (; i + 1 < nt; i += 2) {
    if (i % kStage == 0) prefetch_stage<MODE>(g, io, i, U, lu, rres, strips);
    const double p0 = owns_src ? g.pulse[nt - 1 - i] : 0.0;
    adj_step<RPT, T, MODE>(g, c, st, la, lb, ua, ub, acc, i, U, lu, XL[1], XL[0], XU[1], XU[0],
                           bar[1], bar[0], tx_bytes, p0, io, hist, N2, bulk);
    const double p1 = owns_src ? g.pulse[nt - 2 - i] : 0.0;
    adj_step<RPT, T, MODE>(g, c, st, lb, la, ub, ua, acc, i + 1, U, lu, XL[0], XL[1], XU[0], XU[1],
                           bar[0], bar[1], tx_bytes, p1, io, hist, N2, bulk);
  }
  if (i < nt) {
    if (i % kStage == 0) prefetch_stage<MODE>(g, io, i, U, lu, rres, strips);
    adj_step<RPT, T, MODE>(g, c, st, la, lb, ua, ub, acc, i, U, lu, XL[1], XL[0], XU[1], XU[0],
                           bar[1], bar[0], tx_bytes, owns_src ? g.pulse[0] : 0.0, io, hist, N2, bulk);
  }
  if (c.has_up || c.has_dn) mbar_wait(bar[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
  cluster_sync_all();
  double* dst = acc_part + (size_t)(lu + acc_off) * N2;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (st.active & (1u << j)) dst[(size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z] = acc[j];
}

// ------------------------------------------------------------------ host side
template <class K>
inline int max_active_clusters(K kernel, int cs, int threads, size_t smem) {
  if (smem > 227 * 1024 || threads > kClusterMaxThreads) return 0;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      (cs > 8 && cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
    cudaGetLastError();
    return 0;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) { cudaGetLastError(); return 0; }
  if ((long)fa.numRegs * threads > 65536) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(threads);
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
    return 0;
  }
  return n;
}

template <int RPT, class T>
inline bool try_cluster_cfg(const Geo& g, int cs, ClusterCfg* out) {
  const int rows = (g.nx + cs - 1) / cs;
  if (rows < 2) return false;
  const int nseg = (rows + RPT - 1) / RPT;
  const int threads = g.nz * nseg;
  if (threads > kClusterMaxThreads) return false;
  const int maxrec = std::min(g.M, rows * g.nz);
  const int maxring = g.SL > 0 ? std::min(g.SL, 2 * rows + 2 * g.nz) : 0;
  const size_t sf = cluster_smem_bytes<T>(rows, g.nz, 2, maxrec, maxring);
  const size_t sa = cluster_smem_bytes<T>(rows, g.nz, 4, maxrec, maxring);
  if (max_active_clusters(cluster_fwd_kernel<RPT, T, 0>, cs, threads, sf) <= 0) return false;
  if (max_active_clusters(cluster_fwd_kernel<RPT, T, 1>, cs, threads, sf) <= 0) return false;
  if (max_active_clusters(cluster_fwd_kernel<RPT, T, 2>, cs, threads, sf) <= 0) return false;
  if (max_active_clusters(cluster_adj_kernel<RPT, T, 1>, cs, threads, sa) <= 0) return false;
  if (max_active_clusters(cluster_adj_kernel<RPT, T, 2>, cs, threads, sa) <= 0) return false;
  out->cs = cs;
  out->rows = rows;
  out->rpt = RPT;
  out->nseg = nseg;
  out->threads = threads;
  out->dbl = sizeof(T) == 8;
  out->smem_fwd = sf;
  out->smem_adj = sa;
  out->maxrec = maxrec;
  out->maxring = maxring;
  return true;
}

inline bool cluster_config(const Geo& g, bool rho, ClusterCfg* out) {
  if (rho) return false;  // density runs on the stepwise engine
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      major < 10) {
    cudaGetLastError();
    return false;
  }
  for (int cs : {16, 8}) {
#ifndef DUFWI_EXCHANGE_F32
    if (try_cluster_cfg<4, double>(g, cs, out)) return true;
    if (try_cluster_cfg<2, double>(g, cs, out)) return true;
#endif
    if (try_cluster_cfg<4, float>(g, cs, out)) return true;
    if (try_cluster_cfg<2, float>(g, cs, out)) return true;
  }
  return false;
}

template <class K, class... Args>
inline cudaError_t launch_cluster(K kernel, const ClusterCfg& c, int U, size_t smem,
                                  cudaStream_t st, Args... args) {
  // the dynamic shared-memory limit is per kernel, not per plan: plans with
  // different receiver / ring counts need their own size set before launching
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
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

template <int RPT, class T>
inline cudaError_t cluster_forward_t(const Geo& g, const Model& m, const ClusterCfg& c, int mode,
                                     int unit_begin, int U, float* rec, float* hist, float* strips,
                                     float* ubuf, cudaStream_t st) {
  if (mode == 0)
    return launch_cluster(cluster_fwd_kernel<RPT, T, 0>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,
                          c.maxrec, c.maxring, unit_begin, U, rec, hist, strips, ubuf);
  if (mode == 1)
    return launch_cluster(cluster_fwd_kernel<RPT, T, 1>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,
                          c.maxrec, c.maxring, unit_begin, U, rec, hist, strips, ubuf);
  return launch_cluster(cluster_fwd_kernel<RPT, T, 2>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,
                        c.maxrec, c.maxring, unit_begin, U, rec, hist, strips, ubuf);
}

template <int RPT, class T>
inline cudaError_t cluster_adjoint_t(const Geo& g, const Model& m, const ClusterCfg& c, int mode,
                                     int unit_begin, int U, const double* rres, const float* hist,
                                     const float* strips, const float* ubuf, double* acc_part,
                                     int acc_off, cudaStream_t st) {
  if (mode == 1)
    return launch_cluster(cluster_adj_kernel<RPT, T, 1>, c, U, c.smem_adj, st, g, m, c.cs, c.rows,
                          c.maxrec, c.maxring, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off);
  return launch_cluster(cluster_adj_kernel<RPT, T, 2>, c, U, c.smem_adj, st, g, m, c.cs, c.rows,
                        c.maxrec, c.maxring, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off);
}

inline int cluster_forward(const Geo& g, const Model& m, const ClusterCfg& c, bool /*rho*/,
                           int mode, int unit_begin, int U, float* rec, float* hist,
                           float* strips, float* ubuf, cudaStream_t st) {
  cudaError_t e;
  if (c.rpt == 4 && c.dbl) e = cluster_forward_t<4, double>(g, m, c, mode, unit_begin, U, rec, hist, strips, ubuf, st);
  else if (c.rpt == 2 && c.dbl) e = cluster_forward_t<2, double>(g, m, c, mode, unit_begin, U, rec, hist, strips, ubuf, st);
  else if (c.rpt == 4) e = cluster_forward_t<4, float>(g, m, c, mode, unit_begin, U, rec, hist, strips, ubuf, st);
  else e = cluster_forward_t<2, float>(g, m, c, mode, unit_begin, U, rec, hist, strips, ubuf, st);
  return (int)e;
}

inline int cluster_adjoint(const Geo& g, const Model& m, const ClusterCfg& c, bool /*rho*/,
                           int mode, int unit_begin, int U, const double* rres, const float* hist,
                           const float* strips, const float* ubuf, double* acc_part, int acc_off,
                           cudaStream_t st) {
  cudaError_t e;
  if (c.rpt == 4 && c.dbl) e = cluster_adjoint_t<4, double>(g, m, c, mode, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off, st);
  else if (c.rpt == 2 && c.dbl) e = cluster_adjoint_t<2, double>(g, m, c, mode, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off, st);
  else if (c.rpt == 4) e = cluster_adjoint_t<4, float>(g, m, c, mode, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off, st);
  else e = cluster_adjoint_t<2, float>(g, m, c, mode, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off, st);
  return (int)e;
}

}  // namespace dufwi
