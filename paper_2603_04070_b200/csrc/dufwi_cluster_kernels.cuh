// Cluster engine: one kernel launch per sweep, one thread-block cluster per unit.
//
// For grids whose per-unit state fits a cluster (configs 0/1: 160^2) the whole
// time loop of a sweep runs inside one launch ("temporal blocking in the
// extreme").  The unit's grid is cut into `cs` slabs of `rows`
// x-rows, one per CTA.  Inside a CTA thread (seg, z) owns column z of rows
// [seg*RPT, seg*RPT+RPT): its cells' state (u[t-1], u[t-2] forward; lam[t+1],
// lam[t+2], u[t], u[t-1] adjoint), E/dx^2 and the imaging accumulators live in
// f64 REGISTERS for the whole sweep.  Per time step a thread
//   * reads z-neighbours from a double-buffered shared-memory exchange buffer,
//   * takes x-neighbours from its own registers, from the exchange cells of the
//     adjacent segment, or from the halo rows of the buffer,
//   * writes its new values into the exchange buffer; threads owning the slab's
//     first/last row also push it into the neighbouring CTA's halo row with
//     st.async (DSMEM), completing bytes on that CTA's mbarrier.
// Columns are permuted so that the few holding damped, receiver, ring or
// source cells share warps; every other warp runs a branch-free fast step
// (A = 2, B = -1, no IO), chosen once per sweep and uniform per warp.
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

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dufwi_common.cuh"

namespace dufwi {

namespace cg = cooperative_groups;
#ifdef DUFWI_EXP_TIMING
#ifndef DUFWI_DBG_RANK
#define DUFWI_DBG_RANK 4
#endif
// per-warp step timing of CTA ranks 0 and DUFWI_DBG_RANK of cluster 0: [sweep][cta][warp < 32][sync, body, path, -]
__device__ unsigned long long g_dbg[2 * 2 * 32 * 4];
__device__ __forceinline__ void dbg_step(int sweep, long long T0, long long T1, int path) {
  if ((blockIdx.x == 0 || blockIdx.x == DUFWI_DBG_RANK) && (threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    unsigned long long* d = g_dbg + ((sweep * 2 + (blockIdx.x ? 1 : 0)) * 32 + w) * 4;
    atomicAdd(d + 0, (unsigned long long)(T1 - T0));
    atomicAdd(d + 1, (unsigned long long)(clock64() - T1));
    atomicAdd(d + 2, (unsigned long long)path);
  }
}
// slot 3: cycles in the step's __syncthreads (low 32 bits) and in its halo wait (high 32 bits)
__device__ long long g_dbg_tb, g_dbg_tm;  // unused placeholders keep the symbol table stable
__device__ __forceinline__ void dbg_sync(int sweep, long long T0, long long Tb, long long Tm) {
  if ((blockIdx.x == 0 || blockIdx.x == DUFWI_DBG_RANK) && (threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    unsigned long long* d = g_dbg + ((sweep * 2 + (blockIdx.x ? 1 : 0)) * 32 + w) * 4;
    atomicAdd(d + 3, (unsigned long long)(Tb - T0) + ((unsigned long long)(Tm - Tb) << 32));
  }
}
#endif

struct ClusterCfg {
  int cs = 0;       // CTAs per cluster (slabs per unit)
  int rows = 0;     // x-rows per slab
  int rpt = 0;      // rows per thread (template instance)
  int nseg = 0;     // thread segments per column
  int threads = 0;  // threads per CTA = nz * nseg
  int dbl = 0;      // exchange rows in f64 (1) or f32 (0)
  int maxrec = 0;   // receiver stage entries per CTA: RPT per thread holding receivers
  int maxring = 0;  // ring-strip cells per CTA (upper bound) staged in shared memory
  int maxc = 0;     // clusters co-resident on the device (one wave)
  int per_sm = 1;   // CTAs of the sweep kernels that fit one SM (registers / shared memory)
  size_t smem_fwd = 0, smem_adj = 0;
  size_t smem_lap = 0;     // adjoint over the L(u) history (DUFWI_STORE_LAP)
};

// Receiver samples / ring strips / residuals move between HBM and the step loop
// through shared-memory stages of kStage steps: written (forward) or read
// (adjoint) with one coalesced pass per kStage steps instead of scattered
// global accesses inside every step.
#ifndef DUFWI_KSTAGE
#define DUFWI_KSTAGE 32
#endif
constexpr int kStage = DUFWI_KSTAGE;

// Threads per CTA the sweep kernels are compiled for: the register budget per
// thread (65536 / threads) must hold RPT rows of f64 state (6 per row in the
// adjoint) without spilling.
// (<= 5 rows: up to 20 warps, e.g. config 1's 4 x 4 adjoint shape at 96 registers)
__host__ __device__ constexpr int cluster_max_threads(int rpt) {
  return rpt >= 7 ? 384 : rpt >= 6 ? 512 : 640;
}
// registers per thread for that budget (one CTA per SM, multiples of 8; a warp's
// registers come from one SM sub-partition, 16384 each, so 15 warps cap at 128)
__host__ __device__ constexpr int cluster_max_regs(int rpt) {
  return (65536 / cluster_max_threads(rpt)) / 8 * 8;
}

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
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ------------------------------------------------------------ smem layout
// [nbufs exchange buffers] [nz x nseg*RPT float2 (A, B)] [2 mbarriers] [IO stage]
// An exchange buffer is column-major: cell (buffer row r, column z) at
// (z + 1) * RS + r, r = local row + 1 (r = 0 / rows + 1: never written, zero),
// z = -1 / nz: zero pad columns.  RS >= nseg * RPT + 2 is odd, so 32 lanes on
// consecutive columns hit 32 distinct banks, and a thread's own rows sit at
// compile-time offsets from one base address.  The halo rows pushed by the
// neighbouring CTAs are ROW-major side rows after the column-major part (top
// halo at xmain + z, bottom halo at xmain + nzp + z): a warp's st.async then
// covers 128 contiguous bytes of the neighbour's shared memory instead of 32
// scattered words.
__host__ __device__ inline int xcol_stride(int rows, int rpt) {
  const int nseg = (rows + rpt - 1) / rpt;
  return (nseg * rpt + 2) | 1;
}
__host__ __device__ inline size_t xbuf_main(int rows, int rpt, int nz) {
  return (((size_t)(nz + 2) * xcol_stride(rows, rpt)) + 3) & ~(size_t)3;
}
__host__ __device__ inline int xhalo_pitch(int nz) { return (nz + 3) & ~3; }
__host__ __device__ inline size_t xbuf_elems(int rows, int rpt, int nz) {
  return xbuf_main(rows, rpt, nz) + 2 * (size_t)xhalo_pitch(nz);
}
template <class T>
__host__ __device__ inline size_t ab_offset(int rows, int rpt, int nz, int nbufs) {
  return ((size_t)nbufs * xbuf_elems(rows, rpt, nz) * sizeof(T) + 15) & ~(size_t)15;
}
// (A, B) table: column-major like the buffers, >= nseg * RPT row slots per
// column, odd so 16-byte accesses of consecutive columns are conflict-free
__host__ __device__ inline int ab_col_stride(int rows, int rpt) {
  return ((rows + rpt - 1) / rpt * rpt) | 1;
}
template <class T>
__host__ __device__ inline size_t bar_offset(int rows, int rpt, int nz, int nbufs) {
  return ab_offset<T>(rows, rpt, nz, nbufs) + (size_t)ab_col_stride(rows, rpt) * nz * sizeof(pair_t<T>);
}
// IO stage after the mbarriers: [n_rec, n_ring, pad] [rec_g[maxrec]] [ring_g[maxring]]
// [rec_b[maxrec]] [ring_b[maxring]] [float stage_rec[kStage][maxrec]]
// [float stage_ring[kStage][maxring]].  *_g: HBM slot, *_b: exchange-buffer index.
template <class T>
struct IoStage {
  int* counts;
  int* rec_g;
  int* ring_g;
  int* rec_b;
  int* ring_b;
  T* srec;
  float* sring;
  T* spulse;  // pulse samples of the stage's steps (adjoint)
  int maxrec, maxring;
};

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

template <class T>
__host__ __device__ inline size_t io_offset(int rows, int rpt, int nz, int nbufs) {
  return al16(bar_offset<T>(rows, rpt, nz, nbufs) + 2 * sizeof(uint64_t));
}

template <class T>
__host__ __device__ inline size_t io_bytes(int maxrec, int maxring) {
  return 16 + 2 * al16((size_t)maxrec * 4) + 2 * al16((size_t)maxring * 4) +
         al16((size_t)kStage * maxrec * sizeof(T)) + al16((size_t)kStage * maxring * 4) +
         al16((size_t)kStage * sizeof(T));
}

template <class T>
__host__ __device__ inline size_t cluster_smem_bytes(int rows, int rpt, int nz, int nbufs,
                                                     int maxrec, int maxring) {
  return io_offset<T>(rows, rpt, nz, nbufs) + io_bytes<T>(maxrec, maxring);
}

template <class T>
__device__ __forceinline__ IoStage<T> io_stage(unsigned char* base, int maxrec, int maxring) {
  IoStage<T> io;
  io.counts = reinterpret_cast<int*>(base);
  size_t o = 16;
  io.rec_g = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxrec * 4);
  io.ring_g = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxring * 4);
  io.rec_b = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxrec * 4);
  io.ring_b = reinterpret_cast<int*>(base + o);
  o += al16((size_t)maxring * 4);
  io.srec = reinterpret_cast<T*>(base + o);
  o += al16((size_t)kStage * maxrec * sizeof(T));
  io.sring = reinterpret_cast<float*>(base + o);
  o += al16((size_t)kStage * maxring * 4);
  io.spulse = reinterpret_cast<T*>(base + o);
  io.maxrec = maxrec;
  io.maxring = maxring;
  return io;
}

// ------------------------------------------------------------ per-thread state
struct CellCtx {
  int rank, cs, rows, nr, r0;  // slab of this CTA: global rows [r0, r0+nr)
  int seg, zi, z, lrow0;       // thread: column z (= order[zi]), local rows lrow0 ..
  int RS;                      // exchange column stride
  int xo;                      // buffer offset of the thread's first cell
  uint32_t off_up, off_dn;     // byte offsets of this column's halo cells in a buffer
  int o_xm, o_xp;              // buffer offsets of the x neighbours of the thread's first / last row
  bool has_up, has_dn;         // CTA rank-1 / rank+1 exist with rows
  uint32_t lbase, rup, rdn;    // shared-window base: own, rank-1, rank+1
};

__device__ __forceinline__ CellCtx make_ctx(int cs, int rows, int nx, int nz, int rpt,
                                            const void* smem) {
  CellCtx c;
  c.rank = (int)cg::this_cluster().block_rank();
  c.cs = cs;
  c.rows = rows;
  c.r0 = c.rank * rows;
  c.nr = max(0, min(nx, c.r0 + rows) - c.r0);
  c.seg = threadIdx.x / nz;
  c.zi = threadIdx.x - c.seg * nz;
  c.z = c.zi;
  c.lrow0 = c.seg * rpt;
  c.RS = xcol_stride(rows, rpt);
  c.xo = 0;
  c.has_up = c.rank > 0 && c.nr > 0;
  c.has_dn = c.nr > 0 && c.rank + 1 < cs && (c.rank + 1) * rows < nx;
  c.lbase = smem_addr(smem);
  c.rup = c.has_up ? mapa_rank(c.lbase, c.rank - 1) : 0u;
  c.rdn = c.has_dn ? mapa_rank(c.lbase, c.rank + 1) : 0u;
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

// Column order of the slab, in three classes so that warps are uniform:
// columns with no cell in the undamped box (PML, incl. ring columns) first,
// then columns holding any damped, receiver, ring or source cell, then plain
// columns (every warp of those runs the fast step).  Sets c.z / c.xo.
//
// Warp placement: a CTA of W warps puts warp w on scheduler (SMSP) w % 4, so
// with W % 4 != 0 some SMSPs issue for more warps than others (config 1:
// 10 warps = 3 + 3 + 2 + 2), and the step ends when the busiest SMSP is done.
// The heavy virtual warps — those holding PML or special columns, which run
// the slower paths — are placed on the SMSPs with the fewest warps, the plain
// ones fill the rest (measured per warp with DUFWI_EXP_TIMING: the io and PML
// warps on a 3-warp SMSP set the step time).  Needs nz % 32 == 0 so that a
// warp's lanes stay within one row segment.
// scratch: 2 * nz + 64 + W ints of shared memory (the exchange buffers,
// before they are zeroed).
#ifndef DUFWI_PLACE_FWD
#define DUFWI_PLACE_FWD 1
#endif
#ifndef DUFWI_PLACE_ADJ
#define DUFWI_PLACE_ADJ 0
#endif
template <class T>
__device__ __forceinline__ void order_columns(const Geo& g, CellCtx& c, int txx, int txz,
                                              int* scratch, int rpt, int mode) {
  const int nz = g.nz;
  int* cls = scratch;
  int* order = scratch + nz;
  int* wmap = scratch + 2 * nz;  // physical warp -> virtual warp
  const int W = blockDim.x >> 5;
  // mode 0: identity, 1: heavy warps on the SMSPs with fewest warps, 2: one heavy per SMSP
  const bool place = mode != 0 && (blockDim.x & 31) == 0 && (nz & 31) == 0 && W <= 64;
  for (int z = threadIdx.x; z < nz; z += blockDim.x) {
    int plain = 1, boxed = 0;
    for (int lr = 0; lr < c.nr; ++lr) {
      const int x = c.r0 + lr;
      const bool inb = in_box(g, x, z);
      boxed |= inb;
      if (damping_at(g, x, z) != 0.0 || !inb || (x == txx && z == txz) ||
          (g.row_flag[x] && g.node_slot[(size_t)x * nz + z] >= 0) || ring_index(g, x, z) >= 0)
        plain = 0;
    }
    cls[z] = plain ? 2 : boxed ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0, nheavy = 0;
    for (int q = 0; q < 3; ++q)
      for (int z = 0; z < nz; ++z)
        if (cls[z] == q) {
          order[k++] = z;
          nheavy += q < 2;
        }
    if (place) {
      // physical warps, SMSPs with fewer warps first; virtual warps, heavy first
      const int bps = nz >> 5, hb = (nheavy + 31) >> 5;
      int cnt[4] = {0, 0, 0, 0};
      for (int w = 0; w < W; ++w) ++cnt[w & 3];
      int n = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int v = 0; v < W; ++v)
          if (((v % bps) < hb) == (pass == 0)) wmap[64 + n++] = v;  // staged virtual order
      int i = 0;
      if (mode == 2) {
        for (int w = 0; w < W; ++w) wmap[w] = wmap[64 + w];  // round robin over SMSPs
      } else {
        for (int m = 1; m <= 64 && i < W; ++m)  // SMSPs holding m warps, in SMSP order
          for (int s = 0; s < 4; ++s)
            if (cnt[s] == m)
              for (int w = s; w < W; w += 4) wmap[w] = wmap[64 + i++];
      }
    }
  }
  __syncthreads();
  if (place) {
    const int vt = wmap[threadIdx.x >> 5] * 32 + (threadIdx.x & 31);
    c.seg = vt / nz;
    c.zi = vt - c.seg * nz;
    c.lrow0 = c.seg * rpt;
  }
  c.z = order[c.zi];
  c.xo = (c.z + 1) * c.RS + c.lrow0 + 1;
  {
    const int xm = (int)xbuf_main(c.rows, rpt, nz), hp = xhalo_pitch(nz);
    c.off_dn = (uint32_t)(xm + c.z) * (uint32_t)sizeof(T);       // top halo row of rank+1
    c.off_up = (uint32_t)(xm + hp + c.z) * (uint32_t)sizeof(T);  // bottom halo row of rank-1
    // x neighbours across the slab's edges come from the side rows, inside the
    // slab from the adjacent segment's cell (a missing neighbour: a zero cell)
    // (o_xp: of the thread's last ACTIVE row — the slab's last row may sit
    // anywhere in a partial last segment)
    const bool holds_last = c.lrow0 < c.nr && c.lrow0 + rpt >= c.nr;
    c.o_xm = (c.lrow0 == 0 && c.has_up) ? xm + c.z : c.xo - 1;
    c.o_xp = !holds_last ? c.xo + rpt : c.has_dn ? xm + hp + c.z : c.xo + (c.nr - c.lrow0);
  }
  __syncthreads();  // scratch is reused as exchange buffer afterwards
}

// Static per-cell data loaded once per sweep.
template <int RPT, class T>
struct CellStatic {
  T ed[RPT];
  // receiver / ring rows (bit j = row j) and their first IO-stage index.  A
  // thread holding receivers owns RPT consecutive receiver entries (row j at
  // base + j; slot -1 where row j has none), ring row j's entry is
  // gbase + popc(gmask below j)
  unsigned rmask, gmask;
  int rbase, gbase;
  uint32_t gsa;  // shared address of the thread's first ring stage entry (slot 0)
  unsigned active, src, interior;
  bool pushes_up, pushes_dn;  // owns the slab's first / last row
  unsigned dn_mask;           // bit j set: register j holds the slab's last row (pushes_dn)
  bool special;               // any receiver / ring / source cell
  bool undamped;              // every cell has D == 0: (A, B) = (2, -1), no table reads
  bool fast;                  // whole warp: full, undamped, interior, not special
  bool plainio;               // whole warp: full, undamped, interior (receivers / source allowed)
  bool full;                  // whole warp: every row slot active
  bool unif;                  // whole warp: full, and one (A, B) per thread for all its rows
  bool pml;                   // whole warp: full, and no cell in the undamped box
  bool idle;                  // whole warp: no active row (the bulk-copy issuer's warp)
  const pair_t<T>* ab;          // this thread's (A, B) column: ab[j] for row j
};

template <int RPT, class T>
__device__ __forceinline__ void load_static(const Geo& g, const Model& m, const CellCtx& c,
                                            size_t pb, int txx, int txz, pair_t<T>* ab_table,
                                            const IoStage<T>& io, bool allow_fast,
                                            CellStatic<RPT, T>& st) {
  st.active = st.src = st.interior = 0u;
  st.ab = ab_table + (size_t)c.z * ab_col_stride(c.rows, RPT) + c.lrow0;
  st.pushes_up = c.has_up && c.lrow0 == 0;
  st.pushes_dn = false;
  st.dn_mask = 0u;
  st.rmask = st.gmask = 0u;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = c.lrow0 + j;
    st.ed[j] = T(0);
    if (lr < c.nr) {
      const int x = c.r0 + lr;
      st.active |= 1u << j;
      st.ed[j] = (T)m.Ed[pb + (size_t)x * g.nz + c.z];
      const_cast<pair_t<T>*>(st.ab)[j] = ab_pair<T>(damping_at(g, x, c.z), g.dt);
      if (g.row_flag[x] && g.node_slot[(size_t)x * g.nz + c.z] >= 0) st.rmask |= 1u << j;
      if (io.maxring > 0 && ring_index(g, x, c.z) >= 0) st.gmask |= 1u << j;
      if (x == txx && c.z == txz) st.src |= 1u << j;
      if (in_box(g, x, c.z)) st.interior |= 1u << j;
      if (lr == c.nr - 1 && c.has_dn) {
        st.pushes_dn = true;
        st.dn_mask = 1u << j;
      }
    }
  }
  // IO-stage entries (storage slots only: their order does not matter)
  st.rbase = st.rmask ? atomicAdd(&io.counts[0], RPT) : 0;
  st.gbase = st.gmask ? atomicAdd(&io.counts[1], __popc(st.gmask)) : 0;
  st.gsa = smem_addr(io.sring + st.gbase);
  if (st.rmask)
    for (int j = 0; j < RPT; ++j) {
      const int x = c.r0 + c.lrow0 + j;
      io.rec_g[st.rbase + j] = (st.rmask & (1u << j)) ? g.node_slot[(size_t)x * g.nz + c.z] : -1;
      io.rec_b[st.rbase + j] = c.xo + j;
    }
  for (int j = 0, n = 0; j < RPT; ++j)
    if (st.gmask & (1u << j)) {
      io.ring_g[st.gbase + n] = ring_index(g, c.r0 + c.lrow0 + j, c.z);
      io.ring_b[st.gbase + n] = c.xo + j;
      ++n;
    }
  st.undamped = true;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (c.lrow0 + j < c.nr && damping_at(g, c.r0 + c.lrow0 + j, c.z) != 0.0) st.undamped = false;
  const bool any = st.src != 0u || st.rmask != 0u || st.gmask != 0u;
  st.special = any;
  const unsigned full = (1u << RPT) - 1u;
  const bool f = allow_fast && st.active == full && st.interior == full && st.undamped && !any;
  // warp-uniform path choice
  st.fast = __all_sync(__activemask(), f);
  st.plainio = __all_sync(__activemask(), allow_fast && st.active == full &&
                                              st.interior == full && st.undamped);
  st.full = __all_sync(__activemask(), st.active == full);
  bool same = true;  // one damping value (hence one (A, B)) down the thread's column
#pragma unroll
  for (int j = 1; j < RPT; ++j)
    if (c.lrow0 + j < c.nr &&
        damping_at(g, c.r0 + c.lrow0 + j, c.z) != damping_at(g, c.r0 + c.lrow0, c.z))
      same = false;
  st.unif = __all_sync(__activemask(), st.active == full && same);
  st.pml = __all_sync(__activemask(), st.active == full && st.interior == 0u);
  st.idle = __all_sync(__activemask(), st.active == 0u);
}

// Exchange-row pushes to the neighbouring CTAs (DSMEM st.async completing on
// their mbarrier): the slab's first row -> bottom halo of rank-1, last row ->
// top halo of rank+1.  A CTA's shared memory is one contiguous range of the
// cluster window, so remote addresses are the mapped base plus the offset.
// xb: byte offset of the written buffer from the CTA's shared-memory base
// (uniform), bb: same for the mbarrier completing the step.
template <int RPT, class T>
__device__ __forceinline__ void push_edges(const CellCtx& c, const CellStatic<RPT, T>& s, uint32_t xb,
                                           uint32_t bb, const T (&v)[RPT], bool full) {
  if (s.pushes_up) push_async(c.rup + xb + c.off_up, (T)v[0], c.rup + bb);
  if (s.pushes_dn) {
    const uint32_t ra = c.rdn + xb + c.off_dn;
    const uint32_t rb = c.rdn + bb;
    if (full) {  // every slot active: the slab's last row is register RPT-1
      push_async(ra, (T)v[RPT - 1], rb);
    } else {
      // explicit predicate per register so v[] is never indexed at run time
#pragma unroll
      for (int j = 0; j < RPT; ++j) push_if((s.dn_mask >> j) & 1u, ra, (T)v[j], rb);
    }
  }
}

// ---------------------------------------------------------------------------
// Step synchronisation: the CTA's exchange cells of step i-1 are complete and
// the buffer written at step i is free again (__syncthreads); the neighbours'
// halo rows of step i-1 have landed (mbarrier phase of bar_r); bar_w is armed
// for the bytes the neighbours push during step i.
__device__ __forceinline__ void step_sync(const CellCtx& c, int i, uint32_t bar_r, uint32_t bar_w,
                                          uint32_t tx_bytes, int sweep = 0) {
#ifdef DUFWI_EXP_TIMING
  const long long T0 = clock64();
#endif
  __syncthreads();
#ifdef DUFWI_EXP_TIMING
  const long long Tb = clock64();
#endif
  if (i >= 1 && (c.has_up || c.has_dn)) mbar_wait(bar_r, ((i - 1) >> 1) & 1);
#ifdef DUFWI_EXP_TIMING
  dbg_sync(sweep, T0, Tb, clock64());
#endif
  if (threadIdx.x == 0 && (c.has_up || c.has_dn)) mbar_expect_tx(bar_w, tx_bytes);
}

// Buffers of a step: the one read (r) and the one written (w), as pointers and
// as byte offsets from the shared-memory base (for the DSMEM pushes).
template <class T>
struct StepBufs {
  const T* r;
  T* w;
  uint32_t wb, bar_r, bar_w, bar_wb;
};

// ---- L(u) history transport (DUFWI_STORE_LAP; the adjoint kernel is below)
constexpr int kLapDepth = 4;  // adjoint ring slots

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// The CTA's rows inside the undamped box: [b0, b0 + nb) (nb <= 0: none).
struct BoxRows {
  int b0, nb;
};
__device__ __forceinline__ BoxRows box_rows(const Geo& g, const CellCtx& c) {
  BoxRows r;
  r.b0 = max(c.r0, g.x_lo);
  r.nb = min(c.r0 + c.nr - 1, g.x_hi) - r.b0 + 1;
  return r;
}

// Adjoint ring: kLapDepth mbarriers (32 B) then kLapDepth slots of rows x nz floats.
template <class T>
__host__ __device__ inline size_t lap_ring_offset(int rows, int rpt, int nz, int maxrec) {
  return al16(io_offset<T>(rows, rpt, nz, 2) + io_bytes<T>(maxrec, 0));
}
template <class T>
__host__ __device__ inline size_t cluster_lap_smem_bytes(int rows, int rpt, int nz, int maxrec) {
  return lap_ring_offset<T>(rows, rpt, nz, maxrec) + 32 + (size_t)kLapDepth * rows * nz * 4;
}

// Adjoint, thread 0: bulk load of step j's operand L(u[t-1]) (t = nt-1-j) into
// ring slot j % depth, completing on that slot's mbarrier.
__device__ __forceinline__ void lap_load(const Geo& g, const BoxRows& br, int rows, int j,
                                         uint32_t ring_sa, uint32_t ringbar, const float* hbox,
                                         size_t hstep) {
  if (br.nb > 0 && j <= g.nt - 2) {
    const int sl = j % kLapDepth;
    const uint32_t bytes = (uint32_t)(br.nb * g.nz) * 4u;
    const uint32_t bar = ringbar + 8u * (uint32_t)sl;
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring_sa + (uint32_t)(sl * rows * g.nz) * 4u, hbox + (size_t)(g.nt - 2 - j) * hstep,
             bytes, bar);
  }
}

// The thread that issues the adjoint's bulk loads.  Issuing them costs the
// thread a few hundred cycles per step (per-warp clock64 timing): in a warp
// that pushes a halo row that delays the push, and the neighbouring CTAs wait
// for it.  The job goes to the first thread of a middle segment: its warp
// pushes no halo row, so its late start delays no neighbour, and inside the
// CTA it is hidden behind the halo wait.
// (the adjoint over the L(u) history; adjoint 0.721 -> 0.697 ms on config 1)
__device__ __forceinline__ bool bulk_issuer_mid(const CellCtx& c, int nz, int rows, int rpt) {
  const int nseg = (rows + rpt - 1) / rpt;
  return c.seg * nz + c.zi == (nseg >= 3 ? (nseg / 2) * nz : 0);
}

// Edge rows first: a thread computes its first and last row before the others
// and pushes them to the neighbouring CTAs at once, so the DSMEM transfer of
// the halo rows overlaps the rest of the step body instead of following it.  A
// thread still reads its halo inputs before it pushes (the edge rows are the
// only ones that read them), which is what orders the neighbour's next
// overwrite of that halo row after this read.  Full slabs only.
#ifndef DUFWI_EDGE_FIRST
#define DUFWI_EDGE_FIRST 1
#endif
constexpr bool kEdgeFirst = DUFWI_EDGE_FIRST != 0;
__host__ __device__ constexpr int edge_order(int i, int rpt) {
  return i == 0 ? 0 : i == 1 ? rpt - 1 : i - 1;
}

// One forward step of a thread's cells (u1 = u[t-1] -> u2 := u[t]).  FULL:
// every row slot active (no per-row predicates); PLAIN: undamped cells of the
// box (A = 2, B = -1); IO: a PLAIN thread may hold the source (receivers are
// gathered separately).  All warp-uniform, chosen once per sweep.
// Receiver / ring samples are gathered from the exchange buffer by io_gather.
template <int RPT, class T, int MODE, bool FULL, bool PLAIN, bool UNIF, bool IO>
__device__ __forceinline__ void fwd_body(const Geo& g, const CellCtx& c, const CellStatic<RPT, T>& s,
                                         T (&u1)[RPT], T (&u2)[RPT], int t, int U,
                                         int lu, const StepBufs<T>& B, T pulse_t,
                                         float* __restrict__ hist, size_t N2) {
  const T* pc = B.r + c.xo;
  const T* pm = pc - c.RS;
  const T* pp = pc + c.RS;
  T v[RPT];
  const pair_t<T> ab0 = (!PLAIN && UNIF) ? s.ab[0] : free_pair<T>();
  // MODE 3: the step's L(u[t-1]) (5-point sum, f32) of the box cells straight
  // to history slot t-1 (`hist`: the thread's first cell there): a warp's
  // st.global covers one 128-byte row piece, nothing waits on it
  float* hl = hist;
  constexpr bool EARLY = FULL && kEdgeFirst;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int j = EARLY ? edge_order(i, RPT) : i;
    const T xm = j > 0 ? u1[j - 1] : (T)B.r[c.o_xm];
    const bool own_next = j + 1 < RPT && (FULL || c.lrow0 + j + 1 < c.nr);
    const T xp = own_next ? u1[j + 1]
                          : ((FULL ? j == RPT - 1 : c.lrow0 + j + 1 >= c.nr) ? (T)B.r[c.o_xp] : (T)pc[j + 1]);
    const T lap = lap_s(u1[j], xm, xp, (T)pm[j], (T)pp[j]);
    if (MODE == 3 && t >= 1 && (PLAIN || ((s.interior >> j) & 1u))) hl[j * g.nz] = (float)lap;
    if (PLAIN) {
      v[j] = step_free(u1[j], u2[j], s.ed[j], lap);
    } else {
      const pair_t<T> ab = UNIF ? ab0 : s.ab[j];
      v[j] = step_ab(ab, u1[j], u2[j], s.ed[j], lap);
    }
    if ((!PLAIN || IO) && (s.src & (1u << j))) v[j] = add_s(v[j], pulse_t);
    if (EARLY && i == (RPT > 1 ? 1 : 0)) push_edges<RPT, T>(c, s, B.wb, B.bar_wb, v, FULL);
  }
  T* q = B.w + c.xo;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!FULL && !(s.active & (1u << j))) continue;
    u2[j] = v[j];
    q[j] = (T)v[j];
    if (MODE == 1) hist[((size_t)t * U + lu) * N2 + (size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z] = (float)v[j];
  }
  if (!EARLY) push_edges<RPT, T>(c, s, B.wb, B.bar_wb, v, FULL);
}

// Receiver samples / ring cells of step t, read back from the exchange buffer
// written at step t (complete after the following __syncthreads) into stage
// slot t % kStage: one cell per thread, no per-row branches in the step bodies.
//
// gather_rank(): the order in which threads take the cells — warps on the SM
// sub-partitions that hold fewer warps first (a CTA of W warps puts warp w on
// SMSP w % 4, so with W % 4 != 0 the SMSPs >= W % 4 hold one warp less and
// finish their step bodies earlier).
__device__ __forceinline__ int gather_rank() {
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = W & 3;
  if (r == 0 || (blockDim.x & 31)) return threadIdx.x;
  const int nl = W / 4 * (4 - r);  // warps on the lighter SMSPs
  const bool light = (w & 3) >= r;
  const int idx = light ? (w >> 2) * (4 - r) + (w & 3) - r : (w >> 2) * r + (w & 3);
  return (light ? idx : nl + idx) * 32 + lane;
}

template <class T, int MODE>
__device__ __forceinline__ void io_gather(const IoStage<T>& io, int nrec, int nio, const T* X, int t,
                                          int rank) {
  const int k = t % kStage;
  for (int i = rank; i < nio; i += blockDim.x) {
    if (i < nrec) {
      io.srec[k * io.maxrec + i] = (T)(float)X[io.rec_b[i]];
    } else if (MODE == 2) {
      const int r = i - nrec;
      io.sring[k * io.maxring + r] = (float)X[io.ring_b[r]];
    }
  }
}

// Write the staged receiver samples / ring strips of steps [t0, t0+nk) to HBM.
template <class T, int MODE>
__device__ __forceinline__ void flush_stage(const Geo& g, const IoStage<T>& io, int t0, int nk, int U,
                                            int lu, float* __restrict__ rec,
                                            float* __restrict__ strips) {
  __syncthreads();
  const int nrec = io.counts[0], nring = io.counts[1];
  for (int idx = threadIdx.x; idx < nk * nrec; idx += blockDim.x) {
    const int k = idx / nrec, i = idx - k * nrec;
    const int slot = io.rec_g[i];
    if (slot >= 0) rec[((size_t)(t0 + k) * U + lu) * g.M + slot] = (float)io.srec[k * io.maxrec + i];
  }
  if (MODE == 2) {
    for (int idx = threadIdx.x; idx < nk * nring; idx += blockDim.x) {
      const int k = idx / nring, i = idx - k * nring;
      strips[((size_t)(t0 + k) * U + lu) * g.SL + io.ring_g[i]] = io.sring[k * io.maxring + i];
    }
  }
}

template <int RPT, class T, int MODE>
__device__ __forceinline__ void fwd_step(const Geo& g, const CellCtx& c, const CellStatic<RPT, T>& s,
                                         T (&u1)[RPT], T (&u2)[RPT], int t, int U,
                                         int lu, const StepBufs<T>& B, uint32_t tx_bytes,
                                         T pulse_t, const IoStage<T>& io, int nrec, int nio,
                                         float* __restrict__ rec, float* __restrict__ strips,
                                         float* __restrict__ hist, size_t N2, int grank) {
#ifdef DUFWI_EXP_TIMING
  const long long T0 = clock64();
#endif
  step_sync(c, t, B.bar_r, B.bar_w, tx_bytes);
  if (t >= 1) {
    io_gather<T, MODE>(io, nrec, nio, B.r, t - 1, grank);
    if (t % kStage == 0) flush_stage<T, MODE>(g, io, t - kStage, kStage, U, lu, rec, strips);
  }
#ifdef DUFWI_EXP_TIMING
  const long long T1 = clock64();
#endif
  if (s.idle) {
  } else if (s.fast)
    fwd_body<RPT, T, MODE, true, true, false, false>(g, c, s, u1, u2, t, U, lu, B, pulse_t, hist, N2);
  else if (s.plainio)
    fwd_body<RPT, T, MODE, true, true, false, true>(g, c, s, u1, u2, t, U, lu, B, pulse_t, hist, N2);
  else if (MODE != 3 && s.unif)  // (0.663 -> 0.636 ms with the strips store; the L(u)-storing
                                 // forward, at its 80-register cap, loses 3% with it)
    fwd_body<RPT, T, MODE, true, false, true, true>(g, c, s, u1, u2, t, U, lu, B, pulse_t, hist, N2);
  else if (s.full)
    fwd_body<RPT, T, MODE, true, false, false, true>(g, c, s, u1, u2, t, U, lu, B, pulse_t, hist, N2);
  else
    fwd_body<RPT, T, MODE, false, false, false, true>(g, c, s, u1, u2, t, U, lu, B, pulse_t, hist, N2);
#ifdef DUFWI_EXP_TIMING
  dbg_step(0, T0, T1, s.fast ? 0 : s.plainio ? 5 : s.full ? 1 : 2);
#endif
}

template <int RPT, class T, int MODE>
__global__ void __maxnreg__(cluster_max_regs(RPT))
    cluster_fwd_kernel(Geo g, Model m, int cs, int rows, int maxrec, int maxring,
                       int unit_begin, int U, float* __restrict__ rec, float* __restrict__ hist,
                       float* __restrict__ strips, float* __restrict__ ubuf) {
  extern __shared__ __align__(16) unsigned char smem[];
  CellCtx c = make_ctx(cs, rows, g.nx, g.nz, RPT, smem);
  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const int txx = g.tx[2 * s], txz = g.tx[2 * s + 1];
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t pb = (size_t)b * N2;
  const size_t xe = xbuf_elems(rows, RPT, g.nz);
  T* X[2] = {reinterpret_cast<T*>(smem), reinterpret_cast<T*>(smem) + xe};
  const uint32_t bar_off = (uint32_t)bar_offset<T>(rows, RPT, g.nz, 2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  order_columns<T>(g, c, txx, txz, reinterpret_cast<int*>(smem), RPT, DUFWI_PLACE_FWD);
  for (size_t i = threadIdx.x; i < 2 * xe; i += blockDim.x) X[0][i] = T(0);
  const IoStage<T> io = io_stage<T>(smem + io_offset<T>(rows, RPT, g.nz, 2), maxrec, maxring);
  if (threadIdx.x == 0) {
    mbar_init(bar[0], 1);
    mbar_init(bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    io.counts[0] = io.counts[1] = 0;
  }
  __syncthreads();
  CellStatic<RPT, T> st;
  load_static<RPT, T>(g, m, c, pb, txx, txz,
                   reinterpret_cast<pair_t<T>*>(smem + ab_offset<T>(rows, RPT, g.nz, 2)),
                   io,
                   true, st);  // (FULL too: the history store is in every step variant)
  const uint32_t tx_bytes =
      (uint32_t)((c.has_up ? 1 : 0) + (c.has_dn ? 1 : 0)) * g.nz * sizeof(T);
  T ua[RPT], ub[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) ua[j] = ub[j] = T(0);
  const bool owns_src = st.src != 0u;
  T p_next = owns_src ? (T)g.pulse[0] : T(0);
  cluster_sync_all();  // barriers initialised, buffers zeroed, IO lists complete cluster-wide
  const int nrec = io.counts[0];
  const int nio = nrec + (MODE == 2 ? io.counts[1] : 0);
  const int grank = gather_rank();

  // step t writes X[t & 1] / bar[t & 1]; ub receives u[t] at even t, ua at odd t
  const uint32_t xb1 = (uint32_t)(xe * sizeof(T));
  const StepBufs<T> B0{X[1], X[0], 0u, bar[1], bar[0], bar_off};
  const StepBufs<T> B1{X[0], X[1], xb1, bar[0], bar[1], bar_off + 8u};
  // MODE 3: the thread's first cell in history slot 0 (slots hold whole [x][z]
  // maps per unit; only the undamped box is written and read)
  const size_t hstep = (size_t)U * N2;
  float* hcell = MODE == 3 ? hist + (size_t)lu * N2 + (size_t)(c.r0 + c.lrow0) * g.nz + c.z : hist;
  // step t stores L(u[t-1]) to slot t-1 (t >= 1; never dereferenced at t = 0)
#define DUFWI_HS(t) (MODE == 3 ? hcell + ((ptrdiff_t)(t) - 1) * (ptrdiff_t)hstep : hist)
  int t = 0;
  for (; t + 1 < g.nt; t += 2) {
    T p = p_next;
    if (owns_src) p_next = (T)g.pulse[t + 1];
    fwd_step<RPT, T, MODE>(g, c, st, ua, ub, t, U, lu, B0, tx_bytes, p, io, nrec, nio, rec,
                           strips, DUFWI_HS(t), N2, grank);
    p = p_next;
    if (owns_src && t + 2 < g.nt) p_next = (T)g.pulse[t + 2];
    fwd_step<RPT, T, MODE>(g, c, st, ub, ua, t + 1, U, lu, B1, tx_bytes, p, io, nrec, nio, rec,
                           strips, DUFWI_HS(t + 1), N2, grank);
  }
  if (t < g.nt)
    fwd_step<RPT, T, MODE>(g, c, st, ua, ub, t, U, lu, B0, tx_bytes, p_next, io, nrec, nio, rec,
                           strips, DUFWI_HS(t), N2, grank);
#undef DUFWI_HS
  // the last step's samples, then the partial stage
  __syncthreads();
  io_gather<T, MODE>(io, nrec, nio, X[(g.nt - 1) & 1], g.nt - 1, gather_rank());
  {
    const int t0 = (g.nt - 1) / kStage * kStage;
    flush_stage<T, MODE>(g, io, t0, g.nt - t0, U, lu, rec, strips);
  }
  // drain the last step's incoming pushes before any CTA of the cluster exits
  if (c.has_up || c.has_dn) mbar_wait(bar[(g.nt - 1) & 1], ((g.nt - 1) >> 1) & 1);
  cluster_sync_all();

  if (MODE == 0 || MODE == 2) {
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

// The imaging sums run in f32 over blocks of kAccBlock steps and are folded
// into f64 totals between blocks: a block's partial sum carries ~sqrt(16) f32
// roundings, the sum over the sweep's thousands of (cancelling) terms none.
constexpr int kAccBlock = 16;
static_assert(kAccBlock % 2 == 0, "flushed between step pairs");
template <int RPT>
__device__ __forceinline__ void acc_flush(double (&)[RPT], double (&)[RPT]) {}  // f64 sums: nothing to fold
template <int RPT>
__device__ __forceinline__ void acc_flush(float (&acc)[RPT], double (&accd)[RPT]) {
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    accd[j] += (double)acc[j];
    acc[j] = 0.f;
  }
}

// ---------------------------------------------------------------------------
// adjoint step i (time t = nt-1-i).  l1 = lam[t+1], l2 = lam[t+2] -> lam[t];
// ua = u[t] -> u[t-2] (reconstruction, MODE 2), ub = u[t-1].
// Buffers: XL exchange of E*lam, XU exchange of u (MODE 2), indexed by i.
// T2: t >= 2 (every step but the last two: imaging and reconstruction run).
template <class T>
struct AdjBufs {
  const T* lr;
  T* lw;
  const T* ur;
  T* uw;
  uint32_t lwb, uwb, bar_r, bar_w, bar_wb;
};

// NOIMG (MODE 2): no cell of the thread lies in the undamped box, so there is
// no imaging and no reconstruction; only ring cells carry u (from the strips).
template <int RPT, class T, int MODE, bool FULL, bool PLAIN, bool UNIF, bool IO, bool NOIMG,
          bool T2>
__device__ __forceinline__ void adj_body(const Geo& g, const CellCtx& c, const CellStatic<RPT, T>& s,
                                         T (&l1)[RPT], T (&l2)[RPT], T (&ua)[RPT],
                                         T (&ub)[RPT], T (&acc)[RPT], int i, int U,
                                         int lu, const AdjBufs<T>& B, const IoStage<T>& io,
                                         const float* __restrict__ hist, size_t N2) {
  const int RS = c.RS, z = c.z;
  const int t = g.nt - 1 - i;
  const int k = i % kStage;
  // lam[t] = A lam1 + L^T(E lam1) + B lam2 (+ residual at receivers)
  T el[RPT], lam[RPT];
  const pair_t<T> ab0 = (!PLAIN && UNIF) ? s.ab[0] : free_pair<T>();
#pragma unroll
  for (int j = 0; j < RPT; ++j) el[j] = mul_s(s.ed[j], l1[j]);
  {
    const T* pc = B.lr + c.xo;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const T xm = j > 0 ? el[j - 1] : (T)B.lr[c.o_xm];
      const bool own_next = j + 1 < RPT && (FULL || c.lrow0 + j + 1 < c.nr);
      const T xp = own_next ? el[j + 1]
                          : ((FULL ? j == RPT - 1 : c.lrow0 + j + 1 >= c.nr) ? (T)B.lr[c.o_xp] : (T)pc[j + 1]);
      const T adj = lap_s(el[j], xm, xp, (T)pc[j - RS], (T)pc[j + RS]);
      if (PLAIN) {
        lam[j] = adjs_free(l1[j], l2[j], adj);
      } else {
        const pair_t<T> ab = UNIF ? ab0 : s.ab[j];
        lam[j] = adjs_ab(ab, l1[j], l2[j], adj);
      }
    }
  }
  if ((!PLAIN || IO) && !NOIMG && s.rmask) {
    // one entry per row (0 where the row has no receiver: adding it is exact)
    const T* r = io.srec + (size_t)k * io.maxrec + s.rbase;
#pragma unroll
    for (int j = 0; j < RPT; ++j) lam[j] = add_s(lam[j], r[j]);
  }
  // imaging with L(u[t-1]) and reconstruction of u[t-2]
  const bool img = T2 || t >= 1;
  T lapu[RPT];
  if (MODE == 2 && !NOIMG) {
    const T* pc = B.ur + c.xo;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const T xm = j > 0 ? ub[j - 1] : (T)B.ur[c.o_xm];
      const bool own_next = j + 1 < RPT && (FULL || c.lrow0 + j + 1 < c.nr);
      const T xp = own_next ? ub[j + 1]
                          : ((FULL ? j == RPT - 1 : c.lrow0 + j + 1 >= c.nr) ? (T)B.ur[c.o_xp] : (T)pc[j + 1]);
      lapu[j] = lap_s(ub[j], xm, xp, (T)pc[j - RS], (T)pc[j + RS]);
    }
  } else if (MODE == 1) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      lapu[j] = T(0);
      if (img && (FULL || (s.active & (1u << j)))) {
        const float* F = hist + ((size_t)(t - 1) * U + lu) * N2;
        const int x = c.r0 + c.lrow0 + j;
        const size_t cell = (size_t)x * g.nz + z;
        const T fxm = x > 0 ? (T)F[cell - g.nz] : T(0);
        const T fxp = x < g.nx - 1 ? (T)F[cell + g.nz] : T(0);
        const T fzm = z > 0 ? (T)F[cell - 1] : T(0);
        const T fzp = z < g.nz - 1 ? (T)F[cell + 1] : T(0);
        lapu[j] = lap_s((T)F[cell], fxm, fxp, fzm, fzp);
      }
    }
  }
  T* ql = B.lw + c.xo;
  T* qu = B.uw + c.xo;
  T elw[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    elw[j] = mul_s(s.ed[j], lam[j]);
    if (!FULL && !(s.active & (1u << j))) continue;
    l2[j] = lam[j];
    ql[j] = (T)elw[j];
    if (MODE == 2 && NOIMG) {
      if (s.gmask & (1u << j)) {
        if (T2 || t >= 2)
          ua[j] = (T)lds_f32(s.gsa + 4u * (uint32_t)(k * io.maxring + __popc(s.gmask & ((1u << j) - 1u))));
        qu[j] = (T)ua[j];
      }
      continue;
    }
    if (img) {
      if (MODE == 1) {
        acc[j] = fma_s(lapu[j], lam[j], acc[j]);
      } else if (PLAIN || (s.interior & (1u << j))) {
        acc[j] = fma_s(lapu[j], lam[j], acc[j]);
        if (T2 || t >= 2) {
          T prev = recon_s(ub[j], ua[j], s.ed[j], lapu[j]);
          // source sample s[t] from the shared-memory stage (a global load here
          // would sit on the step's critical path)
          if ((!PLAIN || IO) && (s.src & (1u << j))) prev = add_s(prev, io.spulse[k]);
          ua[j] = prev;
        }
      } else if ((s.gmask & (1u << j)) && (T2 || t >= 2)) {
        // ring cell: the saved strip stands in for the reconstruction
        ua[j] = (T)lds_f32(s.gsa + 4u * (uint32_t)(k * io.maxring + __popc(s.gmask & ((1u << j) - 1u))));
      }
    }
    if (MODE == 2) qu[j] = (T)ua[j];
  }
  push_edges<RPT, T>(c, s, B.lwb, B.bar_wb, elw, FULL);
  if (MODE == 2) push_edges<RPT, T>(c, s, B.uwb, B.bar_wb, ua, FULL);
}

// Load residuals of steps [i0, i0+kStage) (t = nt-1-i) and the ring strips they
// reconstruct from (t-2) into the shared-memory stage, one coalesced pass.
template <class T, int MODE>
__device__ __forceinline__ void prefetch_stage(const Geo& g, const IoStage<T>& io, int i0, int U,
                                               int lu, const double* __restrict__ rres,
                                               const float* __restrict__ strips) {
  __syncthreads();  // the previous block's readers are done with the stage
  const int nk = min(kStage, g.nt - i0);
  const int nrec = io.counts[0], nring = io.counts[1];
  for (int idx = threadIdx.x; idx < nk * nrec; idx += blockDim.x) {
    const int k = idx / nrec, r = idx - k * nrec;
    const int t = g.nt - 1 - (i0 + k);
    const int slot = io.rec_g[r];
    io.srec[k * io.maxrec + r] = slot >= 0 ? (T)rres[((size_t)t * U + lu) * g.M + slot] : T(0);
  }
  if (MODE == 2) {
    for (int idx = threadIdx.x; idx < nk * nring; idx += blockDim.x) {
      const int k = idx / nring, r = idx - k * nring;
      const int t = g.nt - 1 - (i0 + k);
      io.sring[k * io.maxring + r] = t >= 2 ? strips[((size_t)(t - 2) * U + lu) * g.SL + io.ring_g[r]] : 0.f;
    }
    // (a strided loop: a small grid's CTA can have fewer threads than kStage)
    for (int k = threadIdx.x; k < nk; k += blockDim.x) io.spulse[k] = (T)g.pulse[g.nt - 1 - (i0 + k)];
  }
}

template <int RPT, class T, int MODE, bool T2>
__device__ __forceinline__ void adj_step(const Geo& g, const CellCtx& c, const CellStatic<RPT, T>& s,
                                         T (&l1)[RPT], T (&l2)[RPT], T (&ua)[RPT],
                                         T (&ub)[RPT], T (&acc)[RPT], int i, int U,
                                         int lu, const AdjBufs<T>& B, uint32_t tx_bytes,
                                         const IoStage<T>& io,
                                         const float* __restrict__ hist, size_t N2) {
#ifdef DUFWI_EXP_TIMING
  const long long T0 = clock64();
#endif
  step_sync(c, i, B.bar_r, B.bar_w, tx_bytes, 1);
#ifdef DUFWI_EXP_TIMING
  const long long T1 = clock64();
#endif
#define DUFWI_ADJ_BODY(FULL, PLAIN, UNIF, IO, NOIMG)                                           \
  adj_body<RPT, T, MODE, FULL, PLAIN, UNIF, IO, NOIMG, T2>(g, c, s, l1, l2, ua, ub, acc, i, U, lu, \
                                                           B, io, hist, N2)
#ifdef DUFWI_EXP_NOIO
  if (MODE == 2 && (s.fast || s.plainio))
    DUFWI_ADJ_BODY(true, true, false, false, false);
#else
  if (MODE == 2 && s.fast)
    DUFWI_ADJ_BODY(true, true, false, false, false);
#endif
  else if (MODE == 2 && s.plainio)
    DUFWI_ADJ_BODY(true, true, false, true, false);
  else if (MODE == 2 && s.pml && s.unif)
    DUFWI_ADJ_BODY(true, false, true, true, true);
  else if (MODE == 2 && s.pml)
    DUFWI_ADJ_BODY(true, false, false, true, true);
  else if (s.unif)
    DUFWI_ADJ_BODY(true, false, true, true, false);
  else if (s.full)
    DUFWI_ADJ_BODY(true, false, false, true, false);
  else
    DUFWI_ADJ_BODY(false, false, false, true, false);
#undef DUFWI_ADJ_BODY
#ifdef DUFWI_EXP_TIMING
  dbg_step(1, T0, T1, (MODE == 2 && s.fast) ? 0 : (MODE == 2 && s.plainio) ? 5 : (MODE == 2 && s.pml) ? 4 : s.unif ? 3 : s.full ? 1 : 2);
#endif
}

template <int RPT, class T, int MODE>
__global__ void __maxnreg__(cluster_max_regs(RPT))
    cluster_adj_kernel(Geo g, Model m, int cs, int rows, int maxrec, int maxring,
                       int unit_begin, int U,
                       const double* __restrict__ rres, const float* __restrict__ hist,
                       const float* __restrict__ strips, const float* __restrict__ ubuf,
                       double* __restrict__ acc_part, int acc_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  CellCtx c = make_ctx(cs, rows, g.nx, g.nz, RPT, smem);
  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const int txx = g.tx[2 * s], txz = g.tx[2 * s + 1];
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t pb = (size_t)b * N2;
  const int RS = c.RS;
  const size_t xe = xbuf_elems(rows, RPT, g.nz);
  T* base = reinterpret_cast<T*>(smem);
  T* XL[2] = {base, base + xe};
  T* XU[2] = {base + 2 * xe, base + 3 * xe};
  const uint32_t bar_off = (uint32_t)bar_offset<T>(rows, RPT, g.nz, 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  order_columns<T>(g, c, txx, txz, reinterpret_cast<int*>(smem), RPT, DUFWI_PLACE_ADJ);
  for (size_t k = threadIdx.x; k < 4 * xe; k += blockDim.x) base[k] = T(0);
  const IoStage<T> io = io_stage<T>(smem + io_offset<T>(rows, RPT, g.nz, 4), maxrec, maxring);
  if (threadIdx.x == 0) {
    mbar_init(bar[0], 1);
    mbar_init(bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    io.counts[0] = io.counts[1] = 0;
  }
  __syncthreads();
  CellStatic<RPT, T> st;
  load_static<RPT, T>(g, m, c, pb, txx, txz,
                   reinterpret_cast<pair_t<T>*>(smem + ab_offset<T>(rows, RPT, g.nz, 4)),
                   io,
                   MODE == 2, st);
  const int per = MODE == 2 ? 2 : 1;
  const uint32_t tx_bytes =
      (uint32_t)(per * ((c.has_up ? 1 : 0) + (c.has_dn ? 1 : 0)) * g.nz * sizeof(T));
  const int nt = g.nt;
  const float* u_last = ubuf + ((size_t)((nt - 1) & 1) * U + lu) * N2;
  const float* u_prev = ubuf + ((size_t)((nt - 2) & 1) * U + lu) * N2;
  __syncthreads();  // zero fill done before the u[nt-2] exchange rows are written
  // step i = 0 reads XU[1] = u[nt-2] (own rows and both halo rows from global)
  if (MODE == 2 && c.nr > 0) {
    for (int k = threadIdx.x; k < (c.nr + 2) * g.nz; k += blockDim.x) {
      const int r = k / g.nz, zz = k - r * g.nz;
      const int x = c.r0 - 1 + r;
      // own rows: column-major cell r; the halo rows: the row-major side rows
      const size_t xm = xbuf_main(rows, RPT, g.nz);
      const size_t cell = r == 0 ? xm + zz
                          : r == c.nr + 1 ? xm + xhalo_pitch(g.nz) + zz
                                          : (size_t)(zz + 1) * RS + r;
      if (x >= 0 && x < g.nx) XU[1][cell] = (T)u_prev[(size_t)x * g.nz + zz];
    }
  }
  T la[RPT], lb[RPT], ua[RPT], ub[RPT], acc[RPT];
  double accd[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    la[j] = lb[j] = acc[j] = ua[j] = ub[j] = T(0);
    accd[j] = 0.0;
    if (MODE == 2 && (st.active & (1u << j))) {
      const size_t cell = (size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z;
      ua[j] = u_last[cell];
      ub[j] = u_prev[cell];
    }
  }
  cluster_sync_all();

  // step i writes XL[i&1], XU[i&1], bar[i&1]; reads XL[(i+1)&1], XU[(i+1)&1], bar[(i+1)&1]
  const uint32_t xsz = (uint32_t)(xe * sizeof(T));
  const AdjBufs<T> B0{XL[1], XL[0], XU[1], XU[0], 0u, 2 * xsz, bar[1], bar[0], bar_off};
  const AdjBufs<T> B1{XL[0], XL[1], XU[0], XU[1], xsz, 3 * xsz, bar[0], bar[1], bar_off + 8u};
  // steps with t >= 2 (i <= nt - 3) in pairs, then the tail
  int i = 0;
  for (; i + 1 < nt - 2; i += 2) {
    if (i % kAccBlock == 0) acc_flush<RPT>(acc, accd);
    if (i % kStage == 0) prefetch_stage<T, MODE>(g, io, i, U, lu, rres, strips);
    adj_step<RPT, T, MODE, true>(g, c, st, la, lb, ua, ub, acc, i, U, lu, B0, tx_bytes, io, hist,
                                 N2);
    adj_step<RPT, T, MODE, true>(g, c, st, lb, la, ub, ua, acc, i + 1, U, lu, B1, tx_bytes, io,
                                 hist, N2);
  }
  for (; i < nt; ++i) {
    if (i % kStage == 0) prefetch_stage<T, MODE>(g, io, i, U, lu, rres, strips);
    if (i & 1)
      adj_step<RPT, T, MODE, false>(g, c, st, lb, la, ub, ua, acc, i, U, lu, B1, tx_bytes, io, hist,
                                    N2);
    else
      adj_step<RPT, T, MODE, false>(g, c, st, la, lb, ua, ub, acc, i, U, lu, B0, tx_bytes, io, hist,
                                    N2);
  }
  if (c.has_up || c.has_dn) mbar_wait(bar[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
  cluster_sync_all();
  double* dst = acc_part + (size_t)(lu + acc_off) * N2;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (st.active & (1u << j))
      dst[(size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z] = accd[j] + (double)acc[j];
}

// ---------------------------------------------------------------------------
// L(u) history (DUFWI_STORE_LAP).  The forward stores L(u[t-1]) of every
// undamped-box cell and step (f32, 4 B per cell update: the masked gradient
// only needs the box, like the strips store), so the reverse sweep carries only
// lam: per step the lam update with its E*lam exchange, the residual at
// receivers, and acc += L(u[t-1]) * lam.  No u state, no backward
// reconstruction, no second exchange buffer or push.
//
// The forward writes its box cells' L(u) with plain st.global from the step
// body: fire-and-forget, a warp covers 128 contiguous bytes of a row.  (Staging
// the rows in shared memory and writing them with cp.async.bulk from a 21st
// warp cost a fence.proxy.async per thread and step and an 80-register cap:
// 0.682 against 0.637 ms on config 1.)  The adjoint cannot afford the latency
// of per-thread loads (operand loaded one step ahead into registers: 0.81 ms,
// in the same step: 0.93 ms, against 0.67 ms): it prefetches a CTA's box rows
// of a step as ONE contiguous cp.async.bulk (global -> shared, the rows of a
// slab are contiguous in the [x][z] layout) kLapDepth steps ahead, completing
// on a per-slot mbarrier, issued by one thread.
template <int RPT, class T, bool FULL, bool PLAIN, bool UNIF, bool IO, bool IMG>
__device__ __forceinline__ void adjlap_body(const CellCtx& c, const CellStatic<RPT, T>& s,
                                            T (&l1)[RPT], T (&l2)[RPT],
                                            T (&acc)[RPT], int i, const AdjBufs<T>& B,
                                            const IoStage<T>& io, const float* lr, int nz) {
  const int RS = c.RS;
  const int k = i % kStage;
  T el[RPT], lam[RPT];
  const pair_t<T> ab0 = (!PLAIN && UNIF) ? s.ab[0] : free_pair<T>();
#pragma unroll
  for (int j = 0; j < RPT; ++j) el[j] = mul_s(s.ed[j], l1[j]);
  const T* pc = B.lr + c.xo;
  constexpr bool EARLY = FULL && kEdgeFirst;
  const bool rx = (!PLAIN || IO) && s.rmask;  // one stage entry per row (0: no receiver)
  const T* r = io.srec + (size_t)k * io.maxrec + s.rbase;
  T elw[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int j = EARLY ? edge_order(i, RPT) : i;
    const T xm = j > 0 ? el[j - 1] : (T)B.lr[c.o_xm];
    const bool own_next = j + 1 < RPT && (FULL || c.lrow0 + j + 1 < c.nr);
    const T xp = own_next ? el[j + 1]
                          : ((FULL ? j == RPT - 1 : c.lrow0 + j + 1 >= c.nr) ? (T)B.lr[c.o_xp] : (T)pc[j + 1]);
    const T adj = lap_s(el[j], xm, xp, (T)pc[j - RS], (T)pc[j + RS]);
    if (PLAIN) {
      lam[j] = adjs_free(l1[j], l2[j], adj);
    } else {
      const pair_t<T> ab = UNIF ? ab0 : s.ab[j];
      lam[j] = adjs_ab(ab, l1[j], l2[j], adj);
    }
    if (rx) lam[j] = add_s(lam[j], r[j]);
    elw[j] = mul_s(s.ed[j], lam[j]);
    if (EARLY && i == (RPT > 1 ? 1 : 0)) push_edges<RPT, T>(c, s, B.lwb, B.bar_wb, elw, FULL);
  }
  T* ql = B.lw + c.xo;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!FULL && !(s.active & (1u << j))) continue;
    l2[j] = lam[j];
    ql[j] = (T)elw[j];
    if (IMG && (PLAIN || ((s.interior >> j) & 1u)))
      acc[j] = fma_s((T)lr[j * nz], lam[j], acc[j]);
  }
  if (!EARLY) push_edges<RPT, T>(c, s, B.lwb, B.bar_wb, elw, FULL);
}

template <int RPT, class T, bool IMG>
__device__ __forceinline__ void adjlap_step(const Geo& g, const CellCtx& c,
                                            const CellStatic<RPT, T>& s, T (&l1)[RPT],
                                            T (&l2)[RPT], T (&acc)[RPT], int i,
                                            const AdjBufs<T>& B, uint32_t tx_bytes,
                                            const IoStage<T>& io, const BoxRows& br, int rows,
                                            const float* ring, uint32_t ring_sa, uint32_t ringbar,
                                            const float* hbox, size_t hstep, int lofs,
                                            bool issuer) {
#ifdef DUFWI_EXP_TIMING
  const long long T0 = clock64();
#endif
  step_sync(c, i, B.bar_r, B.bar_w, tx_bytes, 1);
  // every thread is past step i-1: its ring slot is free for step i-1+depth
  if (issuer && i >= 1) lap_load(g, br, rows, i - 1 + kLapDepth, ring_sa, ringbar, hbox, hstep);
  const int sl = i % kLapDepth;
  if (IMG && br.nb > 0 && !s.idle) mbar_wait(ringbar + 8u * (uint32_t)sl, (uint32_t)(i / kLapDepth) & 1u);
#ifdef DUFWI_EXP_TIMING
  const long long T1 = clock64();
#endif
  const float* lr = ring + (size_t)sl * rows * g.nz + lofs;
  if (s.idle) {
  } else if (s.fast)
    adjlap_body<RPT, T, true, true, false, false, IMG>(c, s, l1, l2, acc, i, B, io, lr, g.nz);
  else if (s.plainio)
    adjlap_body<RPT, T, true, true, false, true, IMG>(c, s, l1, l2, acc, i, B, io, lr, g.nz);
  else if (s.unif)
    adjlap_body<RPT, T, true, false, true, true, IMG>(c, s, l1, l2, acc, i, B, io, lr, g.nz);
  else if (s.full)
    adjlap_body<RPT, T, true, false, false, true, IMG>(c, s, l1, l2, acc, i, B, io, lr, g.nz);
  else
    adjlap_body<RPT, T, false, false, false, true, IMG>(c, s, l1, l2, acc, i, B, io, lr, g.nz);
#ifdef DUFWI_EXP_TIMING
  dbg_step(1, T0, T1, s.fast ? 0 : s.plainio ? 5 : s.unif ? 3 : s.full ? 1 : 2);
#endif
}

template <int RPT, class T>
__global__ void __maxnreg__(cluster_max_regs(RPT))
    cluster_adjlap_kernel(Geo g, Model m, int cs, int rows, int maxrec, int unit_begin, int U,
                          const double* __restrict__ rres, const float* __restrict__ hlap,
                          double* __restrict__ acc_part, int acc_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  CellCtx c = make_ctx(cs, rows, g.nx, g.nz, RPT, smem);
  const int lu = blockIdx.x / cs;
  const int u = unit_begin + lu;
  const int b = u / g.S;
  const int s = u - b * g.S;
  const int txx = g.tx[2 * s], txz = g.tx[2 * s + 1];
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t pb = (size_t)b * N2;
  const size_t xe = xbuf_elems(rows, RPT, g.nz);
  T* XL[2] = {reinterpret_cast<T*>(smem), reinterpret_cast<T*>(smem) + xe};
  const uint32_t bar_off = (uint32_t)bar_offset<T>(rows, RPT, g.nz, 2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  const uint32_t bar[2] = {smem_addr(&bars[0]), smem_addr(&bars[1])};
  order_columns<T>(g, c, txx, txz, reinterpret_cast<int*>(smem), RPT, DUFWI_PLACE_ADJ);
  for (size_t k = threadIdx.x; k < 2 * xe; k += blockDim.x) XL[0][k] = T(0);
  const IoStage<T> io = io_stage<T>(smem + io_offset<T>(rows, RPT, g.nz, 2), maxrec, 0);
  unsigned char* rbase = smem + lap_ring_offset<T>(rows, RPT, g.nz, maxrec);
  const uint32_t ringbar = smem_addr(rbase);
  const float* ring = reinterpret_cast<const float*>(rbase + 32);
  const uint32_t ring_sa = smem_addr(ring);
  const BoxRows br = box_rows(g, c);
  const size_t hstep = (size_t)U * N2;
  const float* hbox = hlap + (size_t)lu * N2 + (size_t)max(br.b0, 0) * g.nz;
  if (threadIdx.x == 0) {
    mbar_init(bar[0], 1);
    mbar_init(bar[1], 1);
    for (int d = 0; d < kLapDepth; ++d) mbar_init(ringbar + 8u * d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    io.counts[0] = io.counts[1] = 0;
    for (int d = 0; d < kLapDepth; ++d) lap_load(g, br, rows, d, ring_sa, ringbar, hbox, hstep);
  }
  __syncthreads();
  CellStatic<RPT, T> st;
  load_static<RPT, T>(g, m, c, pb, txx, txz,
                   reinterpret_cast<pair_t<T>*>(smem + ab_offset<T>(rows, RPT, g.nz, 2)), io, true,
                   st);
  const uint32_t tx_bytes = (uint32_t)(((c.has_up ? 1 : 0) + (c.has_dn ? 1 : 0)) * g.nz * sizeof(T));
  const int nt = g.nt;
  // the thread's first cell in a ring slot (slots hold the box rows from b0)
  const int lofs = (c.r0 + c.lrow0 - br.b0) * g.nz + c.z;
  const bool issuer = bulk_issuer_mid(c, g.nz, rows, RPT);
  T la[RPT], lb[RPT], acc[RPT];
  double accd[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    la[j] = lb[j] = acc[j] = T(0);
    accd[j] = 0.0;
  }
  cluster_sync_all();

  const uint32_t xsz = (uint32_t)(xe * sizeof(T));
  const AdjBufs<T> B0{XL[1], XL[0], nullptr, nullptr, 0u, 0u, bar[1], bar[0], bar_off};
  const AdjBufs<T> B1{XL[0], XL[1], nullptr, nullptr, xsz, 0u, bar[0], bar[1], bar_off + 8u};
#define DUFWI_ADJLAP(IMG, L1, L2, BB, I)                                                          \
  adjlap_step<RPT, T, IMG>(g, c, st, L1, L2, acc, I, BB, tx_bytes, io, br, rows, ring, ring_sa,   \
                           ringbar, hbox, hstep, lofs, issuer)
  int i = 0;
  for (; i + 1 < nt - 1; i += 2) {  // steps with t >= 1: imaging
    if (i % kAccBlock == 0) acc_flush<RPT>(acc, accd);
    if (i % kStage == 0) prefetch_stage<T, 1>(g, io, i, U, lu, rres, nullptr);
    DUFWI_ADJLAP(true, la, lb, B0, i);
    DUFWI_ADJLAP(true, lb, la, B1, i + 1);
  }
  for (; i < nt; ++i) {
    if (i % kStage == 0) prefetch_stage<T, 1>(g, io, i, U, lu, rres, nullptr);
    const bool img = nt - 1 - i >= 1;
    if (i & 1) {
      if (img) DUFWI_ADJLAP(true, lb, la, B1, i); else DUFWI_ADJLAP(false, lb, la, B1, i);
    } else {
      if (img) DUFWI_ADJLAP(true, la, lb, B0, i); else DUFWI_ADJLAP(false, la, lb, B0, i);
    }
  }
#undef DUFWI_ADJLAP
  if (c.has_up || c.has_dn) mbar_wait(bar[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
  cluster_sync_all();
  double* dst = acc_part + (size_t)(lu + acc_off) * N2;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (st.active & (1u << j))
      dst[(size_t)(c.r0 + c.lrow0 + j) * g.nz + c.z] = accd[j] + (double)acc[j];
}

// ------------------------------------------------------------------ host side
template <class K>
inline int max_active_clusters(K kernel, int cs, int threads, size_t smem) {
  if (smem > 227 * 1024) return 0;
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

// Largest number of ring-strip cells (ring_index >= 0, inside the grid) in any
// slab of `rows` rows: two ring columns per box row plus the ring rows.
inline int max_ring_cells(const Geo& g, int rows) {
  const int zc = (g.z_lo - 1 >= 0 ? 1 : 0) + (g.z_hi + 1 < g.nz ? 1 : 0);
  int best = 0;
  for (int r0 = 0; r0 < g.nx; r0 += rows) {
    const int r1 = std::min(g.nx, r0 + rows);  // [r0, r1)
    const int box = std::max(0, std::min(r1, g.x_hi + 1) - std::max(r0, g.x_lo));
    int n = zc * box;
    if (g.x_lo - 1 >= r0 && g.x_lo - 1 < r1) n += g.Lz;
    if (g.x_hi + 1 >= r0 && g.x_hi + 1 < r1 && g.x_hi + 1 < g.nx) n += g.Lz;
    best = std::max(best, n);
  }
  return best;
}

// Receiver stage entries of the fullest slab: RPT per (column, segment) that
// holds a receiver node (`rxn`: distinct receiver nodes, host copy).
inline int max_rec_entries(const Geo& g, int rows, int rpt, const std::vector<int2>& rxn) {
  int best = 0;
  std::vector<char> seen;
  for (int r0 = 0; r0 < g.nx; r0 += rows) {
    const int nseg = (rows + rpt - 1) / rpt;
    seen.assign((size_t)nseg * g.nz, 0);
    int n = 0;
    for (const int2& p : rxn)
      if (p.x >= r0 && p.x < r0 + rows) {
        char& f = seen[(size_t)((p.x - r0) / rpt) * g.nz + p.y];
        if (!f) { f = 1; ++n; }
      }
    best = std::max(best, n * rpt);
  }
  return best;
}

template <int RPT, class T>
inline bool try_cluster_cfg(const Geo& g, int cs, const std::vector<int2>& rxn, ClusterCfg* out) {
  const int rows = (g.nx + cs - 1) / cs;
  if (rows < 2) return false;
  const int nseg = (rows + RPT - 1) / RPT;
  const int threads = g.nz * nseg;
  if (threads > cluster_max_threads(RPT)) return false;
  const int maxrec = max_rec_entries(g, rows, RPT, rxn);
  const int maxring = g.SL > 0 ? max_ring_cells(g, rows) : 0;
  const size_t sf = cluster_smem_bytes<T>(rows, RPT, g.nz, 2, maxrec, maxring);
  const size_t sa = cluster_smem_bytes<T>(rows, RPT, g.nz, 4, maxrec, maxring);
  // clusters co-resident on the device: the least over the sweep kernels
  const size_t sl = cluster_lap_smem_bytes<T>(rows, RPT, g.nz, maxrec);
  int n = max_active_clusters(cluster_fwd_kernel<RPT, T, 0>, cs, threads, sf);
  n = std::min(n, max_active_clusters(cluster_fwd_kernel<RPT, T, 1>, cs, threads, sf));
  n = std::min(n, max_active_clusters(cluster_fwd_kernel<RPT, T, 2>, cs, threads, sf));
  n = std::min(n, max_active_clusters(cluster_fwd_kernel<RPT, T, 3>, cs, threads, sf));
  n = std::min(n, max_active_clusters(cluster_adj_kernel<RPT, T, 1>, cs, threads, sa));
  n = std::min(n, max_active_clusters(cluster_adj_kernel<RPT, T, 2>, cs, threads, sa));
  n = std::min(n, max_active_clusters(cluster_adjlap_kernel<RPT, T>, cs, threads, sl));
  if (n <= 0) return false;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cluster_adj_kernel<RPT, T, 2>, threads,
                                                    sa) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  out->per_sm = std::max(1, per_sm);
  out->cs = cs;
  out->rows = rows;
  out->rpt = RPT;
  out->nseg = nseg;
  out->threads = threads;
  out->dbl = sizeof(T) == 8;
  out->smem_fwd = sf;
  out->smem_adj = sa;
  out->smem_lap = sl;
  out->maxrec = maxrec;
  out->maxring = maxring;
  out->maxc = n;
  return true;
}

// Rows per thread are a template parameter (register-resident state); the
// instances below cover up to 8 rows per thread with f64 exchange rows and
// 2 / 4 with the f32 fallback (large nz, where f64 rows exceed shared memory).
template <class T>
inline bool try_cluster_rpt(const Geo& g, int cs, int rpt, const std::vector<int2>& rxn,
                            ClusterCfg* out) {
  switch (rpt) {
    case 2: return try_cluster_cfg<2, T>(g, cs, rxn, out);
    case 4: return try_cluster_cfg<4, T>(g, cs, rxn, out);
    case 8: return try_cluster_cfg<8, T>(g, cs, rxn, out);
    // (f64 arithmetic, the precise variant: 2 / 4 / 8 rows per thread only)
    case 5: return sizeof(T) == 4 && try_cluster_cfg<5, float>(g, cs, rxn, out);
    case 6: return sizeof(T) == 4 && try_cluster_cfg<6, float>(g, cs, rxn, out);
    case 7: return sizeof(T) == 4 && try_cluster_cfg<7, float>(g, cs, rxn, out);
    default: return false;
  }
}

// Every launch shape that fits: cluster sizes 16 .. 2, each with the fewest
// rows per thread that fit the thread budget and any larger count that splits
// the slab exactly.  DUFWI_CLUSTER_CS / DUFWI_CLUSTER_RPT pin them (experiments).
inline bool cluster_candidates(const Geo& g, bool rho, bool f64, const std::vector<int2>& rxn,
                               std::vector<ClusterCfg>& out) {
  out.clear();
  if (rho) return false;  // density runs on the stepwise engine
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      major < 10) {
    cudaGetLastError();
    return false;
  }
  int only_cs = 0, only_rpt = 0;
  if (const char* e = getenv("DUFWI_CLUSTER_CS")) only_cs = atoi(e);
  if (const char* e = getenv("DUFWI_CLUSTER_RPT")) only_rpt = atoi(e);
  const int opts[6] = {2, 4, 5, 6, 7, 8};
  for (int cs = 16; cs >= 2; --cs) {
    if (only_cs && cs != only_cs) continue;
    const int rows = (g.nx + cs - 1) / cs;
    if (rows < 2 || g.nz < 1) continue;
    bool first = true;
    for (int r : opts) {
      const int nseg = (rows + r - 1) / r;
      if (g.nz * nseg > cluster_max_threads(r)) continue;
      const bool take = only_rpt ? r == only_rpt : (first || rows % r == 0);
      first = false;
      if (!take) continue;
      ClusterCfg c;
      if (f64 ? try_cluster_rpt<double>(g, cs, r, rxn, &c) : try_cluster_rpt<float>(g, cs, r, rxn, &c))
        out.push_back(c);
    }
  }
  return !out.empty();
}

// Per-step cost model of a shape, in row slots per SM: idle slots of a partial
// last segment keep its warps off the fast step (x1.3); 7-8 rows per thread
// run fewer warps with more register pressure (x1.05).  Measured on config 1
// (forward + adjoint ms): 16 rows as 2 x 8 (0.84 + 1.71) < 18 as 3 x 6
// (0.87 + 1.82) < 18 slots as 3 x 6 with 16 rows used.
inline double cluster_cost(const ClusterCfg& c, int U) {
  double cost = (double)c.nseg * c.rpt;
  if (c.rows % c.rpt) cost *= 1.3;
  if (c.rpt >= 7) cost *= 1.05;
  // Co-residency counts clusters that SHARE SMs (several CTAs per SM): only
  // maxc / per_sm clusters get SMs of their own, and a step is as slow as the
  // busiest SM.  Measured (f32, config 1, 8 units, fwd / adj ms with the L(u)
  // store): 10 CTAs x 16 rows, 11 resident at 1 CTA/SM: 0.81 / 0.78; 16 CTAs x
  // 10 rows, 14 resident at 2 CTAs/SM (7 GPCs hold a 16-CTA cluster): 0.90 / 0.93.
  const int own = std::max(1, c.maxc / std::max(1, c.per_sm));
  const int share = std::min(c.per_sm, (U + own - 1) / own);
  return cost * std::max(1, share);
}

// Launch shape for U units: the fewest waves of co-resident clusters (a unit's
// time loop cannot be split, so a second wave doubles the sweep), then the
// cheapest step.
//
// The adjoint step is issue / FP64-pipe bound on each SM sub-partition: a CTA of
// W warps puts ceil(W/4) of them on its busiest SMSP, so its cost is scaled by
// ceil(W/4) / (W/4) (config 1: 10 warps = 3+3+2+2 -> x1.2; 20 warps -> x1).
// Measured (fwd / adj ms): 2 x 8 rows, 10 warps 0.839 / 1.327; 4 x 4, 20 warps
// 0.848 / 1.289.  The forward keeps the <= 512-thread shapes and the plain cost.
inline const ClusterCfg& pick_cluster(const std::vector<ClusterCfg>& c, int U,
                                      bool adjoint = false) {
  size_t best = 0;
  long best_w = -1;
  double best_c = 0.0;
  bool any = false;
  // (f64 forward: the <= 512-thread shapes measured faster; f32: 640 threads as well)
  for (size_t i = 0; i < c.size(); ++i)
    if (adjoint || !c[i].dbl || c[i].threads <= 512) any = true;
  for (size_t i = 0; i < c.size(); ++i) {
    if (any && !adjoint && c[i].dbl && c[i].threads > 512) continue;
    const long w = (U + c[i].maxc - 1) / c[i].maxc;
    double k = cluster_cost(c[i], U);
    if (adjoint) {
      const int W = (c[i].threads + 31) / 32;
      k *= (double)((W + 3) / 4) / (W / 4.0);
    }
    if (best_w < 0 || w < best_w || (w == best_w && k < best_c)) {
      best = i;
      best_w = w;
      best_c = k;
    }
  }
  return c[best];
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
  if (mode == 4)  // DUFWI_STORE_LAP: hist receives L(u[t]) (kernel MODE 3)
    return launch_cluster(cluster_fwd_kernel<RPT, T, 3>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,
                          c.maxrec, c.maxring, unit_begin, U, rec, hist, strips, ubuf);
  return launch_cluster(cluster_fwd_kernel<RPT, T, 2>, c, U, c.smem_fwd, st, g, m, c.cs, c.rows,
                        c.maxrec, c.maxring, unit_begin, U, rec, hist, strips, ubuf);
}

template <int RPT, class T>
inline cudaError_t cluster_adjoint_t(const Geo& g, const Model& m, const ClusterCfg& c, int mode,
                                     int unit_begin, int U, const double* rres, const float* hist,
                                     const float* strips, const float* ubuf, double* acc_part,
                                     int acc_off, cudaStream_t st) {
  if (mode == 4)
    return launch_cluster(cluster_adjlap_kernel<RPT, T>, c, U, c.smem_lap, st, g, m, c.cs, c.rows,
                          c.maxrec, unit_begin, U, rres, hist, acc_part, acc_off);
  if (mode == 1)
    return launch_cluster(cluster_adj_kernel<RPT, T, 1>, c, U, c.smem_adj, st, g, m, c.cs, c.rows,
                          c.maxrec, c.maxring, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off);
  return launch_cluster(cluster_adj_kernel<RPT, T, 2>, c, U, c.smem_adj, st, g, m, c.cs, c.rows,
                        c.maxrec, c.maxring, unit_begin, U, rres, hist, strips, ubuf, acc_part, acc_off);
}

#define DUFWI_CLUSTER_DISPATCH(FN, ...)                                        \
  (c.dbl ? (c.rpt == 2   ? FN<2, double>(__VA_ARGS__)                          \
            : c.rpt == 4 ? FN<4, double>(__VA_ARGS__)                          \
                         : FN<8, double>(__VA_ARGS__))                         \
         : (c.rpt == 2   ? FN<2, float>(__VA_ARGS__)                           \
            : c.rpt == 4 ? FN<4, float>(__VA_ARGS__)                           \
            : c.rpt == 5 ? FN<5, float>(__VA_ARGS__)                           \
            : c.rpt == 6 ? FN<6, float>(__VA_ARGS__)                           \
            : c.rpt == 7 ? FN<7, float>(__VA_ARGS__)                           \
                         : FN<8, float>(__VA_ARGS__)))

inline int cluster_forward(const Geo& g, const Model& m, const ClusterCfg& c, int mode,
                           int unit_begin, int U, float* rec, float* hist, float* strips,
                           float* ubuf, cudaStream_t st) {
  return (int)DUFWI_CLUSTER_DISPATCH(cluster_forward_t, g, m, c, mode, unit_begin, U, rec, hist,
                                     strips, ubuf, st);
}

inline int cluster_adjoint(const Geo& g, const Model& m, const ClusterCfg& c, int mode,
                           int unit_begin, int U, const double* rres, const float* hist,
                           const float* strips, const float* ubuf, double* acc_part, int acc_off,
                           cudaStream_t st) {
  return (int)DUFWI_CLUSTER_DISPATCH(cluster_adjoint_t, g, m, c, mode, unit_begin, U, rres, hist,
                                     strips, ubuf, acc_part, acc_off, st);
}
#undef DUFWI_CLUSTER_DISPATCH

}  // namespace dufwi
