// C ABI of libdufwi.so (include/dufwi.h): plans, workspace layout and the
// sweep drivers for the stepwise and cluster engines.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dufwi.h"
#include "dufwi_api_kernels.cuh"
#include "dufwi_aux_kernels.cuh"
#include "dufwi_cluster_kernels.cuh"
#include "dufwi_step_kernels.cuh"
#include "dufwi_vec_kernels.cuh"
#include "dufwi_lean_kernels.cuh"
#include "dufwi_tile_kernels.cuh"

using namespace dufwi;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(DUFWI_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

#define LAUNCH_CHECK(plan)                                                               \
  do {                                                                                   \
    ++(plan)->launches;                                                                  \
    cudaError_t _e = cudaGetLastError();                                                 \
    if (_e != cudaSuccess)                                                               \
      return fail(DUFWI_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
  } while (0)

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// SMs of the current device (launch sizing; 148 on B200)
int device_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    return 148;
  return n;
}

}  // namespace

struct dufwi_plan {
  Geo geo{};
  int E = 0, has_rho = 0, engine = 0, last_engine = 0;
  double dx = 0, dt = 0;
  bool box_ok = false;  // D == 0 exactly on a rectangle and > 0 elsewhere
  int device = 0;
  int sms = 148;  // SM count of the plan's device (cudaDevAttrMultiProcessorCount)
  int64_t launches = 0;
  // device tables (owned)
  double *px = nullptr, *pz = nullptr, *d2d = nullptr, *pulse = nullptr;
  int *tx = nullptr, *rx_slot = nullptr, *rx_next = nullptr, *node_slot = nullptr;
  int* elements = nullptr;
  int el_box[4] = {0, -1, 0, -1};  // x0, x1, z0, z1 of the elements (gradient mask)
  int* rx_slot_unused = nullptr;
  unsigned char *row_flag = nullptr, *col_flag = nullptr, *rx_head = nullptr;
  double *Ed = nullptr, *dEdc = nullptr, *rho = nullptr, *q = nullptr;
  int* flag = nullptr;
  std::vector<void*> owned;
  ABTables ab{};  // (A, B) tables of the damped update for the stepwise kernels
  // cluster engine
  std::vector<ClusterCfg> ccands;  // launch shapes that fit, one per cluster size
  ClusterCfg ccfg{};                // the forward's shape for all units at once (plan_info)
  ClusterCfg ccfg_adj{};            // the adjoint's
  bool cluster_ok = false;
  int arith = DUFWI_ARITH_F32;  // arithmetic of the sweep kernels (dufwi_geometry_t.arith)
  int lean_tx = 0;      // rows per warp override (DUFWI_LEAN_TX, experiments)
  bool lean_on = true;  // lean stepwise kernels (DUFWI_LEAN=0: the first vec/stream kernels)
  double *Er = nullptr, *fxe = nullptr, *fz = nullptr, *fz0 = nullptr;  // density tables
  float *Edf = nullptr, *Erf = nullptr, *qf = nullptr;  // f32 coefficient streams (lean kernels)
  // f32 tile kernels (DUFWI_ARITH_F32 stepwise path, dufwi_tile_kernels.cuh)
  TileTabs tile{};       // f32 damping tables, receiver-tile flags
  float* hq = nullptr;   // q / 2, replicate-padded [B][nx+2][nz+8]
  bool tile_ok = false;  // tensor maps can be encoded and the tables exist
  bool tile_on = true;   // DUFWI_TILE=0: the f64 lean kernels instead (A/B timing)
};

namespace {

template <class T>
int dev_alloc(dufwi_plan_t* p, T** out, size_t count) {
  void* ptr = nullptr;
  CUDA_TRY(cudaMalloc(&ptr, std::max<size_t>(count, 1) * sizeof(T)));
  p->owned.push_back(ptr);
  *out = static_cast<T*>(ptr);
  return 0;
}

template <class T>
int upload(dufwi_plan_t* p, T** out, const T* host, size_t count) {
  int rc = dev_alloc(p, out, count);
  if (rc) return rc;
  if (count) CUDA_TRY(cudaMemcpy(*out, host, count * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

// ---------------------------------------------------------------- workspace
// Offsets are independent of where the unit range starts; the residual area
// comes first so every store mode finds it at the same place.
struct Layout {
  size_t rres = 0, mis = 0, rec = 0, ubuf = 0, hist = 0, strips = 0, snap = 0, lbuf = 0,
         acc_part = 0, total = 0;
};

// Snapshot checkpointing (DUFWI_STORE_CHECKPOINT): segments of K steps,
// K = ceil(sqrt(2 nt)) minimising the snapshot pairs (2 nt / K fields) plus
// one segment's recomputed history (K fields).
int ck_len(int nt) {
  int k = (int)std::ceil(std::sqrt(2.0 * nt));
  return std::max(2, std::min(k, nt));
}
int ck_segments(int nt) { return (nt + ck_len(nt) - 1) / ck_len(nt); }

// Shot groups of the stepwise kernels for a concrete unit range: groups of up
// to `gs` shots of one phantom; the adjoint keeps one f64 accumulator per group.
struct Groups {
  int gs = 1, gpp = 1, nb = 1, b0 = 0, ngroups = 1, first = 1;
};

int zstrips(const Geo& g) { return (g.nz + kStripZ - 1) / kStripZ; }
long warps_per_group(const Geo& g) { return (long)zstrips(g) * ((g.nx + kRXA - 1) / kRXA); }

// Group count as enumerated by shot_group(): the chunk's first phantom (maybe
// partial), then ceil(S/gs) groups for every further phantom.
Groups make_groups(const Geo& g, int unit_begin, int U, int gs) {
  Groups G;
  G.gs = std::max(1, std::min(gs, g.S));
  G.gpp = (g.S + G.gs - 1) / G.gs;
  G.b0 = unit_begin / g.S;
  G.nb = (unit_begin + U - 1) / g.S - G.b0 + 1;
  const int n_first = std::min(U, (G.b0 + 1) * g.S - unit_begin);
  G.first = (n_first + G.gs - 1) / G.gs;
  G.ngroups = G.first + (G.nb - 1) * G.gpp;
  return G;
}

// Forward: one group per kNSF shots (a thread carries them).
Groups fwd_groups(const Geo& g, int unit_begin, int U) { return make_groups(g, unit_begin, U, kNSF); }

// Adjoint: as many shots per group as the warp target allows (one f64
// accumulator read-modify-write per cell, group and step).
Groups adj_groups(const Geo& g, int unit_begin, int U, bool per_unit, bool vec, bool lean,
                  int sms, bool tile = false) {
  if (per_unit) return make_groups(g, unit_begin, U, 1);
  if (tile) {
    // tile imaging kernel: a CTA per (box tile, group) walks the group's shots;
    // enough groups for ~8 CTAs per SM, at most 64 shots per group (f32 partial
    // sums), at least 4 (the accumulator costs 16 B / gs per cell update)
    const long tiles = (long)((g.Lz + 2 + kTZ - 1) / kTZ + 1) * ((g.Lx + 2 + kTX - 1) / kTX + 1);
    static const long per_sm = [] {
      const char* e = getenv("DUFWI_IMG_CTAS_PER_SM");
      return e ? std::max(1L, atol(e)) : 8L;
    }();
    const long want = std::max(1L, ((long)sms * per_sm + tiles - 1) / tiles);
    // groups never span phantoms: balance the shots of a phantom over its groups
    const long nb = std::max(1L, ((long)U + g.S - 1) / g.S);
    const long gpp = std::max(1L, (want + nb - 1) / nb);
    const long shots = std::min((long)U, (long)g.S);
    const int gs = (int)std::min(64L, std::max(4L, (shots + gpp - 1) / gpp));
    return make_groups(g, unit_begin, U, gs);
  }
  // lean imaging kernel: ~8 groups, enough CTAs for several waves; the
  // accumulator read-modify-write costs 16 B / gs per cell update
  if (lean) return make_groups(g, unit_begin, U, std::max(1, (U + 7) / 8));
  const long wpg = vec ? (long)((g.nz + 127) / 128) * ((g.nx + kVecAdjTX - 1) / kVecAdjTX)
                       : warps_per_group(g);
  // resident warps wanted per launch
  const long target = vec ? (long)sms * 32 : (long)sms * 64;
  const long wanted = std::max(1L, (target + wpg - 1) / wpg);
  int gs = (int)std::max(1L, ((long)U + wanted - 1) / wanted);
  if (!vec) gs = (gs + kNSA - 1) / kNSA * kNSA;
  return make_groups(g, unit_begin, U, gs);
}

// Vectorised stepwise kernels: constant density, rows made of whole float4s.
bool use_vec(const dufwi_plan_t* p) { return !p->has_rho && p->geo.nz % 4 == 0; }
// Lean kernels: additionally separable damping with a rectangular undamped box.
// Lean kernels: rows of whole float4s, separable damping with a rectangular
// undamped box; constant or variable density.
bool use_lean(const dufwi_plan_t* p) {
  return p->geo.nz % 4 == 0 && p->ab.px && p->box_ok && p->lean_on;
}
// f32 tile kernels: the lean kernels' domain (nz % 4 == 0 makes every row a
// multiple of 16 bytes for the tensor maps), f32 arithmetic
bool use_tile(const dufwi_plan_t* p) {
  return p->arith == DUFWI_ARITH_F32 && use_lean(p) && p->tile_ok && p->tile_on;
}

// Tensor maps of one sweep call: a workspace region [slots][U][nx][nz] gets a
// halo'd and a plain map, valid for every step and unit of the call; the
// coefficient maps cover the plan's per-phantom arrays.
struct TileRegion {
  const float* base = nullptr;
  size_t slots = 0;
  CUtensorMap halo, plain;
};
struct TileCtx {
  TileRegion ubuf, lbuf, hist, snap;
  CUtensorMap e_plain, e_halo, h_halo;
  size_t fieldU = 0;
  bool ok = false;
  // region and slot of a field pointer handed to a step launch
  const TileRegion* find(const float* ptr, int* slot) const {
    for (const TileRegion* r : {&ubuf, &lbuf, &hist, &snap}) {
      if (!r->base || ptr < r->base || ptr >= r->base + r->slots * fieldU) continue;
      *slot = (int)((ptr - r->base) / fieldU);
      return r;
    }
    return nullptr;
  }
};

bool tile_region(const dufwi_plan_t* p, TileRegion& r, const float* base, size_t slots, int U) {
  const Geo& g = p->geo;
  r.base = base;
  r.slots = slots;
  if (!base || !slots) { r.base = nullptr; return true; }
  return make_tile_map(&r.halo, base, g.nz, g.nx, (size_t)U, slots, true) &&
         make_tile_map(&r.plain, base, g.nz, g.nx, (size_t)U, slots, false);
}

void tile_ctx_build(const dufwi_plan_t* p, int U, const float* ubuf, const float* lbuf,
                    const float* hist, size_t hist_slots, const float* snap, size_t snap_slots,
                    TileCtx& c) {
  const Geo& g = p->geo;
  c.ok = false;
  if (!use_tile(p)) return;
  c.fieldU = (size_t)U * g.nx * g.nz;
  const float* E = p->has_rho ? p->Erf : p->Edf;
  bool ok = tile_region(p, c.ubuf, ubuf, 2, U) && tile_region(p, c.lbuf, lbuf, lbuf ? 2 : 0, U) &&
            tile_region(p, c.hist, hist, hist_slots, U) && tile_region(p, c.snap, snap, snap_slots, U);
  ok = ok && make_tile_map(&c.e_plain, E, g.nz, g.nx, (size_t)g.B, 0, false) &&
       make_tile_map(&c.e_halo, E, g.nz, g.nx, (size_t)g.B, 0, true);
  if (p->has_rho)
    ok = ok && make_tile_map(&c.h_halo, p->hq, g.nz + 8, g.nx + 2, (size_t)g.B, 0, true);
  else
    c.h_halo = c.e_halo;  // never dereferenced without density
  c.ok = ok;
}

Groups groups_for(const dufwi_plan_t* p, int unit_begin, int U, bool per_unit) {
  return adj_groups(p->geo, unit_begin, U, per_unit, use_vec(p), use_lean(p), p->sms, use_tile(p));
}

// Upper bound of the group count over every placement of U units.
int max_groups(const dufwi_plan_t* p, int U, bool per_unit);

Layout layout(const dufwi_plan_t* p, int mode, int U) {
  const Geo& g = p->geo;
  Layout L;
  const size_t N2 = (size_t)g.nx * g.nz;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  L.rres = take((size_t)g.nt * U * g.M * sizeof(double));
  L.mis = take((size_t)U * kResidualSplit * sizeof(double));
  L.rec = take((size_t)g.nt * U * g.M * sizeof(float));
  L.ubuf = take(2 * (size_t)U * N2 * sizeof(float));
  if (mode == DUFWI_STORE_FULL || mode == DUFWI_STORE_LAP)
    L.hist = take((size_t)g.nt * U * N2 * sizeof(float));
  if (mode == DUFWI_STORE_STRIPS) L.strips = take((size_t)g.nt * U * g.SL * sizeof(float));
  if (mode == DUFWI_STORE_CHECKPOINT) {
    // snapshots (u[s0-1], u[s0-2]) of every segment start + one segment's history
    L.snap = take((size_t)ck_segments(g.nt) * 2 * U * N2 * sizeof(float));
    L.hist = take((size_t)ck_len(g.nt) * U * N2 * sizeof(float));
  }
  if (mode != DUFWI_STORE_NONE) {
    L.lbuf = take(2 * (size_t)U * N2 * sizeof(float));
    const int ng = std::max(max_groups(p, U, false), p->cluster_ok ? max_groups(p, U, true) : 0);
    L.acc_part = take((size_t)ng * N2 * sizeof(double));
  }
  L.total = off;
  return L;
}

int max_groups(const dufwi_plan_t* p, int U, bool per_unit) {
  const Geo& g = p->geo;
  const int total = g.B * g.S;
  int best = 0;
  // the count only depends on the start modulo S (and on clipping at the end)
  for (int start = 0; start < std::min(g.S, std::max(1, total - U + 1)); ++start)
    best = std::max(best, groups_for(p, start, U, per_unit).ngroups);
  return std::max(best, 1);
}

Model model_of(const dufwi_plan_t* p) {
  return Model{p->Ed,  p->has_rho ? p->rho : nullptr, p->q,   p->Er, p->fxe, p->fz,
               p->fz0, p->Edf,                        p->Erf, p->qf};
}

int check_units(const dufwi_plan_t* p, int unit_begin, int U) {
  const int total = p->geo.B * p->geo.S;
  if (U <= 0 || unit_begin < 0 || unit_begin + U > total)
    return fail(DUFWI_EINVAL, "unit range out of bounds");
  if (U > 65535) return fail(DUFWI_EINVAL, "at most 65535 units per call");
  return 0;
}

}  // namespace

// =============================================================== plan lifecycle
extern "C" int dufwi_plan_create(const dufwi_geometry_t* geo, dufwi_plan_t** plan_out) {
  if (!geo || !plan_out) return fail(DUFWI_EINVAL, "null argument");
  *plan_out = nullptr;
  if (geo->nx < 3 || geo->nz < 3 || geo->nt < 3)
    return fail(DUFWI_EINVAL, "grid must be >= 3x3 with nt >= 3");
  if (geo->n_phantoms < 1 || geo->n_shots < 1 || geo->n_rx < 1 || geo->n_elements < 0)
    return fail(DUFWI_EINVAL, "need >= 1 phantom, shot and receiver");
  if (!(geo->dx > 0) || !(geo->dt > 0)) return fail(DUFWI_EINVAL, "dx, dt must be positive");
  if (!geo->tx_host || !geo->rx_host || !geo->pulse_host)
    return fail(DUFWI_EINVAL, "tx, rx and pulse are required");
  if (!geo->px_host && !geo->damping_host) return fail(DUFWI_EINVAL, "damping is required");
  const int nx = geo->nx, nz = geo->nz, S = geo->n_shots, R = geo->n_rx;
  for (int i = 0; i < S; ++i) {
    const int x = geo->tx_host[2 * i], z = geo->tx_host[2 * i + 1];
    if (x < 0 || x >= nx || z < 0 || z >= nz) return fail(DUFWI_EINVAL, "tx node outside grid");
  }
  for (int i = 0; i < S * R; ++i) {
    const int x = geo->rx_host[2 * i], z = geo->rx_host[2 * i + 1];
    if (x < 0 || x >= nx || z < 0 || z >= nz) return fail(DUFWI_EINVAL, "rx node outside grid");
  }

  auto* p = new dufwi_plan();
  cudaGetDevice(&p->device);
  p->sms = device_sms();
  p->E = geo->n_elements;
  p->has_rho = geo->has_rho ? 1 : 0;
  p->engine = geo->engine;
  p->arith = geo->arith == DUFWI_ARITH_F64 ? DUFWI_ARITH_F64 : DUFWI_ARITH_F32;
  p->dx = geo->dx;
  p->dt = geo->dt;
  Geo& g = p->geo;
  g.nx = nx;
  g.nz = nz;
  g.nt = geo->nt;
  g.S = S;
  g.R = R;
  g.B = geo->n_phantoms;
  g.dt = geo->dt;

  // receiver-node slots: one slot per distinct receiver node of the geometry
  std::vector<int> node_slot((size_t)nx * nz, -1);
  std::vector<unsigned char> row_flag(nx, 0), col_flag(nz, 0);
  std::vector<int> rx_slot((size_t)S * R), rx_next((size_t)S * R, -1);
  std::vector<unsigned char> rx_head((size_t)S * R, 1);
  int M = 0;
  std::vector<int2> rx_nodes;  // distinct receiver nodes (cluster IO staging bounds)
  for (int i = 0; i < S * R; ++i) {
    const size_t cell = (size_t)geo->rx_host[2 * i] * nz + geo->rx_host[2 * i + 1];
    if (node_slot[cell] < 0) {
      node_slot[cell] = M++;
      rx_nodes.push_back(make_int2(geo->rx_host[2 * i], geo->rx_host[2 * i + 1]));
    }
    rx_slot[i] = node_slot[cell];
    row_flag[geo->rx_host[2 * i]] = 1;
    col_flag[geo->rx_host[2 * i + 1]] = 1;
  }
  for (int s = 0; s < S; ++s) {  // chain duplicate receiver nodes within a shot
    for (int r = 0; r < R; ++r) {
      const int i = s * R + r;
      if (!rx_head[i]) continue;
      int last = i;
      for (int r2 = r + 1; r2 < R; ++r2) {
        const int j = s * R + r2;
        if (rx_slot[j] == rx_slot[i]) {
          rx_head[j] = 0;
          rx_next[last] = r2;
          last = j;
        }
      }
    }
  }
  g.M = M;

  // damping: separable profiles or a general map; undamped box detection
  std::vector<double> dmap;
  auto D = [&](int x, int z) -> double {
    return geo->px_host ? std::max(geo->px_host[x], geo->pz_host[z])
                        : geo->damping_host[(size_t)x * nz + z];
  };
  int xl = nx, xh = -1, zl = nz, zh = -1;
  for (int x = 0; x < nx; ++x)
    for (int z = 0; z < nz; ++z)
      if (D(x, z) == 0.0) {
        xl = std::min(xl, x); xh = std::max(xh, x);
        zl = std::min(zl, z); zh = std::max(zh, z);
      }
  bool ok = xh >= 0;
  for (int x = 0; x < nx && ok; ++x)
    for (int z = 0; z < nz && ok; ++z) {
      const bool in = x >= xl && x <= xh && z >= zl && z <= zh;
      if (in != (D(x, z) == 0.0)) ok = false;
    }
  p->box_ok = ok;
  if (!ok) { xl = 0; xh = nx - 1; zl = 0; zh = nz - 1; }
  g.x_lo = xl; g.x_hi = xh; g.z_lo = zl; g.z_hi = zh;
  g.Lx = xh - xl + 1;
  g.Lz = zh - zl + 1;
  g.SL = 2 * g.Lz + 2 * g.Lx;

  int rc = 0;
  if (geo->px_host) {
    rc = rc ? rc : upload(p, &p->px, geo->px_host, nx);
    rc = rc ? rc : upload(p, &p->pz, geo->pz_host, nz);
  } else {
    rc = rc ? rc : upload(p, &p->d2d, geo->damping_host, (size_t)nx * nz);
  }
  {
    // (A, B) of the damped update (forward.py:226-234) per axis ramp / per cell
    auto ab_host = [&](double D, double& A, double& B) {
      if (D == 0.0) { A = 2.0; B = -1.0; return; }
      const double ddt = D * geo->dt, den = 1.0 + ddt;
      A = (2.0 - ddt * ddt) / den;
      B = (ddt - 1.0) / den;
    };
    if (geo->px_host) {
      std::vector<double> Ax(nx), Bx(nx), Az(nz), Bz(nz);
      for (int x = 0; x < nx; ++x) ab_host(geo->px_host[x], Ax[x], Bx[x]);
      for (int z = 0; z < nz; ++z) ab_host(geo->pz_host[z], Az[z], Bz[z]);
      double *dAx, *dBx, *dAz, *dBz;
      rc = rc ? rc : upload(p, &dAx, Ax.data(), nx);
      rc = rc ? rc : upload(p, &dBx, Bx.data(), nx);
      rc = rc ? rc : upload(p, &dAz, Az.data(), nz);
      rc = rc ? rc : upload(p, &dBz, Bz.data(), nz);
      if (!rc) { p->ab.Ax = dAx; p->ab.Bx = dBx; p->ab.Az = dAz; p->ab.Bz = dBz; }
    } else {
      std::vector<double> A2((size_t)nx * nz), B2((size_t)nx * nz);
      for (size_t i = 0; i < A2.size(); ++i) ab_host(geo->damping_host[i], A2[i], B2[i]);
      double *dA2, *dB2;
      rc = rc ? rc : upload(p, &dA2, A2.data(), A2.size());
      rc = rc ? rc : upload(p, &dB2, B2.data(), B2.size());
      if (!rc) { p->ab.A2 = dA2; p->ab.B2 = dB2; }
    }
  }
  if (geo->px_host) {
    // f32 increment-form tables: ramps and (A - 2, B + 1) per axis, rounded once from f64
    auto inc_host = [&](const double* prof, int n, std::vector<float>& pf, std::vector<float>& a2,
                        std::vector<float>& b1) {
      pf.resize(n); a2.resize(n); b1.resize(n);
      for (int i = 0; i < n; ++i) {
        const double D = prof[i];
        double A = 2.0, B = -1.0;
        if (D != 0.0) {
          const double ddt = D * geo->dt, den = 1.0 + ddt;
          A = (2.0 - ddt * ddt) / den;
          B = (ddt - 1.0) / den;
        }
        pf[i] = (float)D;
        if (D != 0.0 && pf[i] == 0.f) pf[i] = 1e-30f;  // keep "damped" distinguishable after rounding
        a2[i] = (float)(A - 2.0);
        b1[i] = (float)(B + 1.0);
      }
    };
    std::vector<float> pf, a2, b1;
    float *dp, *da, *db;
    inc_host(geo->px_host, nx, pf, a2, b1);
    rc = rc ? rc : upload(p, &dp, pf.data(), nx);
    rc = rc ? rc : upload(p, &da, a2.data(), nx);
    rc = rc ? rc : upload(p, &db, b1.data(), nx);
    if (!rc) { p->tile.px = dp; p->tile.a2x = da; p->tile.b1x = db; }
    inc_host(geo->pz_host, nz, pf, a2, b1);
    rc = rc ? rc : upload(p, &dp, pf.data(), nz);
    rc = rc ? rc : upload(p, &da, a2.data(), nz);
    rc = rc ? rc : upload(p, &db, b1.data(), nz);
    if (!rc) { p->tile.pz = dp; p->tile.a2z = da; p->tile.b1z = db; }
    // tiles holding a receiver node
    const int tzn = (nz + kTZ - 1) / kTZ, txn = (nx + kTX - 1) / kTX;
    std::vector<unsigned char> trx((size_t)tzn * txn, 0);
    for (int i = 0; i < S * R; ++i)
      trx[(size_t)(geo->rx_host[2 * i] / kTX) * tzn + geo->rx_host[2 * i + 1] / kTZ] = 1;
    unsigned char* dt_ = nullptr;
    rc = rc ? rc : upload(p, &dt_, trx.data(), trx.size());
    if (!rc) p->tile.tile_rx = dt_;
  }
  rc = rc ? rc : upload(p, &p->pulse, geo->pulse_host, geo->nt);
  rc = rc ? rc : upload(p, &p->tx, geo->tx_host, 2 * (size_t)S);
  rc = rc ? rc : upload(p, &p->rx_slot, rx_slot.data(), rx_slot.size());
  rc = rc ? rc : upload(p, &p->rx_next, rx_next.data(), rx_next.size());
  rc = rc ? rc : upload(p, &p->rx_head, rx_head.data(), rx_head.size());
  rc = rc ? rc : upload(p, &p->node_slot, node_slot.data(), node_slot.size());
  rc = rc ? rc : upload(p, &p->row_flag, row_flag.data(), row_flag.size());
  rc = rc ? rc : upload(p, &p->col_flag, col_flag.data(), col_flag.size());
  if (p->E > 0) rc = rc ? rc : upload(p, &p->elements, geo->elements_host, 2 * (size_t)p->E);
  for (int e = 0; e < p->E; ++e) {
    const int ex = geo->elements_host[2 * e], ez = geo->elements_host[2 * e + 1];
    if (e == 0) p->el_box[0] = p->el_box[1] = ex, p->el_box[2] = p->el_box[3] = ez;
    p->el_box[0] = std::min(p->el_box[0], ex), p->el_box[1] = std::max(p->el_box[1], ex);
    p->el_box[2] = std::min(p->el_box[2], ez), p->el_box[3] = std::max(p->el_box[3], ez);
  }
  const size_t BN2 = (size_t)g.B * nx * nz;
  rc = rc ? rc : dev_alloc(p, &p->Ed, BN2);
  rc = rc ? rc : dev_alloc(p, &p->dEdc, BN2);
  rc = rc ? rc : dev_alloc(p, &p->Edf, BN2);
  if (p->has_rho) {
    rc = rc ? rc : dev_alloc(p, &p->Erf, BN2);
    rc = rc ? rc : dev_alloc(p, &p->qf, BN2);
    rc = rc ? rc : dev_alloc(p, &p->rho, BN2);
    rc = rc ? rc : dev_alloc(p, &p->q, BN2);
    rc = rc ? rc : dev_alloc(p, &p->Er, BN2);
    rc = rc ? rc : dev_alloc(p, &p->fxe, (size_t)g.B * (nx + 1) * nz);
    rc = rc ? rc : dev_alloc(p, &p->fz, BN2);
    rc = rc ? rc : dev_alloc(p, &p->fz0, (size_t)g.B * nx);
    rc = rc ? rc : dev_alloc(p, &p->hq, (size_t)g.B * (nx + 2) * (nz + 8));
  }
  rc = rc ? rc : dev_alloc(p, &p->flag, 4);
  if (!rc && cudaMemset(p->flag, 0, 4 * sizeof(int)) != cudaSuccess)
    rc = fail(DUFWI_ECUDA, "memset flag");
  if (rc) {
    dufwi_plan_destroy(p);
    return rc;
  }
  g.px = p->px;
  g.pz = p->pz;
  p->ab.px = p->px;
  p->ab.pz = p->pz;
  g.d2d = p->d2d;
  g.pulse = p->pulse;
  g.tx = p->tx;
  g.node_slot = p->node_slot;
  g.row_flag = p->row_flag;
  g.col_flag = p->col_flag;
  if (const char* e = getenv("DUFWI_LEAN")) p->lean_on = atoi(e) != 0;
  if (const char* e = getenv("DUFWI_LEAN_TX")) p->lean_tx = std::max(0, atoi(e));
  if (const char* e = getenv("DUFWI_TILE")) p->tile_on = atoi(e) != 0;
  p->tile_ok = p->tile.px && encode_tiled_fn() != nullptr;
  {
    auto big = [](const void* f, size_t bytes) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    };
    big((const void*)tile_img_kernel<false, 1>, TileImgSmem::bytes(false));
    big((const void*)tile_img_kernel<false, 2>, TileImgSmem::bytes(false));
    big((const void*)tile_img_kernel<true, 1>, TileImgSmem::bytes(true));
    big((const void*)tile_img_kernel<true, 2>, TileImgSmem::bytes(true));
  }
  {  // lean rings may exceed the 48 KB default of dynamic shared memory
    auto big = [](const void* f, size_t bytes) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    };
    big((const void*)fwd_lean_kernel<0, false>, sizeof(LeanFwdRing<kFwdNSL, false>));
    big((const void*)fwd_lean_kernel<1, false>, sizeof(LeanFwdRing<kFwdNSL, false>));
    big((const void*)fwd_lean_kernel<2, false>, sizeof(LeanFwdRing<kFwdNSL, false>));
    big((const void*)fwd_lean_kernel<0, true>, sizeof(LeanFwdRing<kFwdNSL, true>));
    big((const void*)fwd_lean_kernel<1, true>, sizeof(LeanFwdRing<kFwdNSL, true>));
    big((const void*)fwd_lean_kernel<2, true>, sizeof(LeanFwdRing<kFwdNSL, true>));
    big((const void*)adjlam_lean_kernel<false>, sizeof(LeanAdjRing<kNSL, false>));
    big((const void*)adjlam_lean_kernel<true>, sizeof(LeanAdjRing<kNSL, true>));
    big((const void*)img_lean_kernel<1, false>, sizeof(LeanImgRing<false>));
    big((const void*)img_lean_kernel<2, false>, sizeof(LeanImgRing<false>));
    big((const void*)img_lean_kernel<1, true>, sizeof(LeanImgRing<true>));
    big((const void*)img_lean_kernel<2, true>, sizeof(LeanImgRing<true>));
  }
  p->cluster_ok = cluster_candidates(g, p->has_rho != 0, p->arith == DUFWI_ARITH_F64, rx_nodes,
                                      p->ccands);
  if (p->cluster_ok) {
    p->ccfg = pick_cluster(p->ccands, geo->n_phantoms * geo->n_shots);
    p->ccfg_adj = pick_cluster(p->ccands, geo->n_phantoms * geo->n_shots, true);
  }
  *plan_out = p;
  return DUFWI_OK;
}

extern "C" int dufwi_plan_destroy(dufwi_plan_t* plan) {
  if (!plan) return DUFWI_OK;
  for (void* ptr : plan->owned) cudaFree(ptr);
  delete plan;
  return DUFWI_OK;
}

extern "C" int dufwi_set_model(dufwi_plan_t* p, const double* c_dev, const double* rho_dev,
                               void* stream) {
  if (!p || !c_dev) return fail(DUFWI_EINVAL, "null argument");
  if (p->has_rho && !rho_dev) return fail(DUFWI_EINVAL, "plan expects a density model");
  const Geo& g = p->geo;
  const size_t total = (size_t)g.B * g.nx * g.nz;
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((total + threads - 1) / threads, (size_t)p->sms * 16);
  set_model_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      g, c_dev, p->has_rho ? rho_dev : nullptr, p->Ed, p->dEdc, p->rho, p->q, p->Edf, p->qf, 0.0,
      p->dx * p->dx, total);
  LAUNCH_CHECK(p);
  if (p->has_rho) {
    const size_t te = (size_t)g.B * (g.nx + 1) * g.nz;
    const int b2 = (int)std::min<size_t>((te + threads - 1) / threads, (size_t)p->sms * 16);
    rho_faces_kernel<<<b2, threads, 0, (cudaStream_t)stream>>>(g, g.B, p->Ed, p->rho, p->q, p->Er,
                                                               p->fxe, p->fz, p->fz0, p->Erf);
    LAUNCH_CHECK(p);
    const size_t th = (size_t)g.B * (g.nx + 2) * (g.nz + 8);
    const int b3 = (int)std::min<size_t>((th + threads - 1) / threads, (size_t)p->sms * 16);
    hq_pad_kernel<<<b3, threads, 0, (cudaStream_t)stream>>>(g, g.B, p->qf, p->hq);
    LAUNCH_CHECK(p);
  }
  return DUFWI_OK;
}

extern "C" int dufwi_workspace_bytes(const dufwi_plan_t* p, int32_t mode, int32_t U,
                                     size_t* bytes_out) {
  if (!p || !bytes_out) return fail(DUFWI_EINVAL, "null argument");
  if (mode < 0 || mode > 4) return fail(DUFWI_EINVAL, "bad store mode");
  if (U <= 0) return fail(DUFWI_EINVAL, "unit_count must be positive");
  *bytes_out = layout(p, mode, U).total;
  return DUFWI_OK;
}

namespace {

int ws_check(const dufwi_plan_t* p, int mode, int unit_begin, int U, size_t ws_bytes,
             Layout& L) {
  L = layout(p, mode, U);
  if (ws_bytes < L.total) return fail(DUFWI_EINVAL, "workspace too small");
  if (mode == DUFWI_STORE_STRIPS && !p->box_ok)
    return fail(DUFWI_EINVAL, "strip storage needs a rectangular undamped box");
  if (mode == DUFWI_STORE_LAP && (!p->cluster_ok || p->engine == DUFWI_ENGINE_STEPWISE))
    return fail(DUFWI_EINVAL, "L(u) history storage needs the cluster engine");
  if (mode == DUFWI_STORE_LAP && !p->box_ok)
    return fail(DUFWI_EINVAL, "L(u) history storage needs a rectangular undamped box");
  if (mode == DUFWI_STORE_LAP && p->geo.nz % 4 != 0)
    return fail(DUFWI_EINVAL, "L(u) history storage needs nz % 4 == 0 (16-byte bulk copies)");
  return 0;
}

bool use_cluster(const dufwi_plan_t* p, int mode) {
  if (p->engine == DUFWI_ENGINE_STEPWISE || mode == DUFWI_STORE_CHECKPOINT) return false;
  return p->cluster_ok;
}

// Rows per warp of the stepwise forward / lam-update kernels: enough warps to
// fill the device.
int stepwise_tx(const dufwi_plan_t* p, int U) {
  const Geo& g = p->geo;
  int vtx = 4;
  for (int c : {32, 16, 8, 4}) {
    const long warps = (long)((g.nz + 127) / 128) * ((g.nx + c - 1) / c) * U;
    if (warps >= (long)p->sms * 32) { vtx = c; break; }
  }
  return p->lean_tx > 0 ? p->lean_tx : vtx;
}

// One stepwise forward step (forward.py:301-308) over units [unit_begin,
// unit_begin+U): u[t] -> uo from u1 = u[t-1], u2 = u[t-2] (has1 / has2: those
// exist), receiver samples -> rec_t, ring strips -> st_t (kmode 2).
int fwd_step_launch(dufwi_plan_t* p, const Model& m, int kmode, int t, int unit_begin, int U,
                    const float* u1, const float* u2, float* uo, float* rec_t, float* st_t,
                    int has1, int has2, cudaStream_t st, const TileCtx* tc = nullptr) {
  const Geo& g = p->geo;
  if (tc && tc->ok) {
    // f32 tile kernels: operands by tensor map (region + slot), output by pointer
    int s1 = 0, s2 = 0;
    const TileRegion* r1 = tc->find(u1, &s1);
    const TileRegion* r2 = tc->find(u2, &s2);
    if (!r1 || !r2) return fail(DUFWI_EINVAL, "tile forward: operand outside the mapped regions");
    const dim3 tgrid((g.nz + kTZ - 1) / kTZ, (g.nx + kTX - 1) / kTX, U);
#define DUFWI_TILE_FWD(R, M)                                                                     \
  tile_fwd_kernel<R, M><<<tgrid, kTT, TileFwdSmem::bytes(R), st>>>(                              \
      r1->halo, r2->plain, tc->e_plain, tc->h_halo, g, p->tile, t, unit_begin, s1, s2, has1, has2, \
      uo, rec_t, st_t)
    if (p->has_rho) {
      if (kmode == 2) DUFWI_TILE_FWD(true, 2); else DUFWI_TILE_FWD(true, 0);
    } else {
      if (kmode == 2) DUFWI_TILE_FWD(false, 2); else DUFWI_TILE_FWD(false, 0);
    }
#undef DUFWI_TILE_FWD
    LAUNCH_CHECK(p);
    return 0;
  }
  const Groups G = fwd_groups(g, unit_begin, U);
  const int vtx = stepwise_tx(p, U);
  const dim3 vgrid((g.nz + 127) / 128, (g.nx + kPipeWarps * vtx - 1) / (kPipeWarps * vtx), U);
  const dim3 lgrid((g.nz + kSW - 1) / kSW, (g.nx + kLeanWarps * vtx - 1) / (kLeanWarps * vtx),
                   (U + kSPW - 1) / kSPW);
  const dim3 block(kWarpsX * 32);
  const dim3 grid(zstrips(g), (g.nx + kWarpsX * kRXF - 1) / (kWarpsX * kRXF), G.ngroups);
#define DUFWI_FWD(R, M)                                                                         \
  fwd_stream_kernel<R, M><<<grid, block, 0, st>>>(g, m, p->ab, t, unit_begin, U, G.gs, u1, u2,   \
                                                  uo, rec_t, st_t, has1, has2)
#define DUFWI_VEC(M)                                                                            \
  fwd_vec_kernel<M><<<vgrid, kPipeWarps * 32, sizeof(FwdRing), st>>>(g, m, p->ab, t, unit_begin, \
                                                      vtx, u1, u2, uo, rec_t, st_t, has1, has2)
#define DUFWI_LEAN(M, R)                                                                        \
  fwd_lean_kernel<M, R><<<lgrid, kLeanT, sizeof(LeanFwdRing<kFwdNSL, R>), st>>>(                 \
      g, m, p->ab, t, unit_begin, U, vtx, u1, u2, uo, rec_t, st_t, has1, has2)
  if (use_lean(p)) {
    if (p->has_rho) {
      if (kmode == 2) DUFWI_LEAN(2, true); else DUFWI_LEAN(0, true);
    } else {
      if (kmode == 2) DUFWI_LEAN(2, false); else DUFWI_LEAN(0, false);
    }
  } else if (use_vec(p)) {
    if (kmode == 2) DUFWI_VEC(2); else DUFWI_VEC(0);
  } else if (p->has_rho) {
    if (kmode == 2) DUFWI_FWD(true, 2); else DUFWI_FWD(true, 0);
  } else {
    if (kmode == 2) DUFWI_FWD(false, 2); else DUFWI_FWD(false, 0);
  }
#undef DUFWI_FWD
#undef DUFWI_VEC
#undef DUFWI_LEAN
  LAUNCH_CHECK(p);
  return 0;
}

// One stepwise adjoint step (adjoint.py:125-131): lam[t] -> l2o from l1 =
// lam[t+1] and l2o = lam[t+2] (in place), residual injection, and for t >= 1
// the imaging term with u[t-1]: kmode 1 reads it from F, kmode 2 reconstructs
// it into ut / utm1 from the strips st_tm1 / st_tm2.
int adj_step_launch(dufwi_plan_t* p, const Model& m, int kmode, int t, int unit_begin, int U,
                    const Groups& G, const float* l1, float* l2o, const double* rres_t,
                    const float* F, float* ut, const float* utm1, const float* st_tm1,
                    const float* st_tm2, double* acc_part, cudaStream_t st,
                    const TileCtx* tc = nullptr) {
  const Geo& g = p->geo;
  const int has1 = t <= g.nt - 2, has2 = t <= g.nt - 3;
  const int do_img = t >= 1, do_recon = t >= 2;
  if (tc && tc->ok) {
    int s1 = 0, s2 = 0;
    const TileRegion* r1 = tc->find(l1, &s1);
    const TileRegion* r2 = tc->find(l2o, &s2);
    if (!r1 || !r2) return fail(DUFWI_EINVAL, "tile adjoint: operand outside the mapped regions");
    const dim3 tgrid((g.nz + kTZ - 1) / kTZ, (g.nx + kTX - 1) / kTX, U);
    if (p->has_rho)
      tile_adj_kernel<true><<<tgrid, kTT, TileAdjSmem::bytes(true), st>>>(
          r1->halo, r2->plain, tc->e_halo, tc->h_halo, g, p->tile, unit_begin, s1, s2, has1, has2,
          l2o, rres_t);
    else
      tile_adj_kernel<false><<<tgrid, kTT, TileAdjSmem::bytes(false), st>>>(
          r1->halo, r2->plain, tc->e_halo, tc->h_halo, g, p->tile, unit_begin, s1, s2, has1, has2,
          l2o, rres_t);
    LAUNCH_CHECK(p);
    if (do_img) {
      // imaging operand u[t-1]: the full history (kmode 1) or the field buffer
      int su = 0, sut = 0;
      const TileRegion* ru = tc->find(kmode == 1 ? F : utm1, &su);
      const TileRegion* rt = tc->find(ut, &sut);
      if (!ru || !rt) return fail(DUFWI_EINVAL, "tile imaging: operand outside the mapped regions");
      // tiles touching the undamped box and its 1-cell ring (kmode 2) / the whole grid
      int tx0 = 0, tx1 = (g.nx - 1) / kTX, tz0 = 0, tz1 = (g.nz - 1) / kTZ;
      if (kmode == 2) {
        tx0 = std::max(0, g.x_lo - 1) / kTX;
        tx1 = std::min(g.nx - 1, g.x_hi + 1) / kTX;
        tz0 = std::max(0, g.z_lo - 1) / kTZ;
        tz1 = std::min(g.nz - 1, g.z_hi + 1) / kTZ;
      }
      const dim3 igrid(tz1 - tz0 + 1, tx1 - tx0 + 1, G.ngroups);
#define DUFWI_TILE_IMG(R, M)                                                                    \
  tile_img_kernel<R, M><<<igrid, kTT, TileImgSmem::bytes(R), st>>>(                             \
      ru->halo, r2->plain, rt->plain, tc->e_plain, tc->h_halo, g, t, unit_begin, U, G.gs, su, s2, \
      sut, tx0, tz0, ut, st_tm2, acc_part, do_recon)
      if (kmode == 1) {
        if (p->has_rho) DUFWI_TILE_IMG(true, 1); else DUFWI_TILE_IMG(false, 1);
      } else {
        if (p->has_rho) DUFWI_TILE_IMG(true, 2); else DUFWI_TILE_IMG(false, 2);
      }
#undef DUFWI_TILE_IMG
      LAUNCH_CHECK(p);
    }
    return 0;
  }
  const int vtx = stepwise_tx(p, U);
  if (use_lean(p)) {
    // split adjoint: lam update (12 B/update) then imaging + reconstruction
    const dim3 lgrid((g.nz + kSW - 1) / kSW, (g.nx + kLeanWarps * vtx - 1) / (kLeanWarps * vtx),
                     (U + kSPW - 1) / kSPW);
    if (p->has_rho)
      adjlam_lean_kernel<true><<<lgrid, kLeanT, sizeof(LeanAdjRing<kNSL, true>), st>>>(
          g, m, p->ab, t, unit_begin, U, vtx, l1, l2o, rres_t, has1, has2);
    else
      adjlam_lean_kernel<false><<<lgrid, kLeanT, sizeof(LeanAdjRing<kNSL, false>), st>>>(
          g, m, p->ab, t, unit_begin, U, vtx, l1, l2o, rres_t, has1, has2);
    LAUNCH_CHECK(p);
    if (do_img) {
      const int rows = kmode == 2 ? g.Lx : g.nx;
      const dim3 igrid((g.nz + kSW - 1) / kSW,
                       (rows + kLeanWarps * kImgTX * kSPW - 1) / (kLeanWarps * kImgTX * kSPW),
                       G.ngroups);
#define DUFWI_IMG(M, R)                                                                         \
  img_lean_kernel<M, R><<<igrid, kLeanT, sizeof(LeanImgRing<R>), st>>>(                          \
      g, m, t, unit_begin, U, G.gs, l2o, F, ut, utm1, st_tm2, acc_part, do_recon)
      if (kmode == 1) {
        if (p->has_rho) DUFWI_IMG(1, true); else DUFWI_IMG(1, false);
      } else {
        if (p->has_rho) DUFWI_IMG(2, true); else DUFWI_IMG(2, false);
      }
#undef DUFWI_IMG
      LAUNCH_CHECK(p);
    }
    return 0;
  }
  if (use_vec(p)) {
    const dim3 lgrid((g.nz + 127) / 128, (g.nx + kPipeWarps * vtx - 1) / (kPipeWarps * vtx), U);
    adjlam_pipe_kernel<<<lgrid, kPipeWarps * 32, sizeof(AdjRing), st>>>(
        g, m, p->ab, t, unit_begin, vtx, l1, l2o, rres_t, has1, has2);
    LAUNCH_CHECK(p);
    if (do_img) {
      const dim3 igrid((g.nz + 127) / 128,
                       (g.nx + kVecAdjWarps * kVecAdjTX - 1) / (kVecAdjWarps * kVecAdjTX), G.ngroups);
      if (kmode == 1)
        img_vec_kernel<1><<<igrid, kVecAdjWarps * 32, 0, st>>>(g, m, t, unit_begin, U, G.gs, l2o, F, ut, utm1, st_tm1, acc_part, do_recon);
      else
        img_vec_kernel<2><<<igrid, kVecAdjWarps * 32, 0, st>>>(g, m, t, unit_begin, U, G.gs, l2o, F, ut, utm1, st_tm1, acc_part, do_recon);
      LAUNCH_CHECK(p);
    }
    return 0;
  }
  const dim3 block(kWarpsX * 32);
  const dim3 grid(zstrips(g), (g.nx + kWarpsX * kRXA - 1) / (kWarpsX * kRXA), G.ngroups);
#define DUFWI_ADJ(R, M)                                                                          \
  adj_stream_kernel<R, M><<<grid, block, 0, st>>>(g, m, p->ab, t, unit_begin, U, G.gs, l1, l2o,  \
                                                  F, ut, utm1, st_tm1,                            \
                                                  rres_t, acc_part, has1, has2, do_img, do_recon)
  if (p->has_rho) {
    if (kmode == 1) DUFWI_ADJ(true, 1); else DUFWI_ADJ(true, 2);
  } else {
    if (kmode == 1) DUFWI_ADJ(false, 1); else DUFWI_ADJ(false, 2);
  }
#undef DUFWI_ADJ
  LAUNCH_CHECK(p);
  return 0;
}

}  // namespace

// ================================================================== forward
extern "C" int dufwi_history_offset(const dufwi_plan_t* p, int32_t U, size_t* off) {
  if (!p || !off || U <= 0) return fail(DUFWI_EINVAL, "bad argument");
  *off = layout(p, DUFWI_STORE_FULL, U).hist;
  return DUFWI_OK;
}

extern "C" int dufwi_forward(dufwi_plan_t* p, int32_t mode, int32_t unit_begin, int32_t U,
                             float* traces_dev, int32_t* nonfinite_dev, void* ws, size_t ws_bytes,
                             void* stream) {
  if (!p || !ws) return fail(DUFWI_EINVAL, "null argument");
  if (mode < 0 || mode > 4) return fail(DUFWI_EINVAL, "bad store mode");
  int rc = check_units(p, unit_begin, U);
  if (rc) return rc;
  Layout L;
  rc = ws_check(p, mode, unit_begin, U, ws_bytes, L);
  if (rc) return rc;
  if (p->engine == DUFWI_ENGINE_CLUSTER && !p->cluster_ok)
    return fail(DUFWI_EINVAL, "cluster engine requested but the grid does not fit");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->geo;
  const Model m = model_of(p);
  char* base = static_cast<char*>(ws);
  float* rec = reinterpret_cast<float*>(base + L.rec);
  float* ubuf = reinterpret_cast<float*>(base + L.ubuf);
  float* hist = reinterpret_cast<float*>(base + L.hist);
  float* strips = reinterpret_cast<float*>(base + L.strips);
  float* snap = reinterpret_cast<float*>(base + L.snap);
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t fieldU = (size_t)U * N2;

  if (use_cluster(p, mode)) {
    p->last_engine = DUFWI_ENGINE_CLUSTER;
    rc = cluster_forward(g, m, pick_cluster(p->ccands, U), mode, unit_begin, U, rec,
                         (mode == DUFWI_STORE_FULL || mode == DUFWI_STORE_LAP) ? hist : nullptr,
                         mode == DUFWI_STORE_STRIPS ? strips : nullptr, ubuf, st);
    if (rc) return fail(DUFWI_ECUDA, std::string("cluster forward: ") + cudaGetErrorString((cudaError_t)rc));
    ++p->launches;
  } else {
    p->last_engine = DUFWI_ENGINE_STEPWISE;
    const int K = ck_len(g.nt);
    TileCtx tc;
    tile_ctx_build(p, U, ubuf, nullptr, mode == DUFWI_STORE_FULL ? hist : nullptr, (size_t)g.nt,
                   nullptr, 0, tc);
    // no silent change of kernels (and arithmetic) under a plan that reports "tile"
    if (use_tile(p) && !tc.ok)
      return fail(DUFWI_ECUDA, "tensor map encoding failed (workspace not 16-byte aligned?)");
    for (int t = 0; t < g.nt; ++t) {
      float* rec_t = rec + (size_t)t * U * g.M;
      const int has1 = t >= 1, has2 = t >= 2;
      const float *u1, *u2;
      float* uo;
      float* st_t = mode == DUFWI_STORE_STRIPS ? strips + (size_t)t * U * g.SL : nullptr;
      if (mode == DUFWI_STORE_FULL) {
        u1 = has1 ? hist + (size_t)(t - 1) * fieldU : hist;
        u2 = has2 ? hist + (size_t)(t - 2) * fieldU : hist;
        uo = hist + (size_t)t * fieldU;
      } else {
        u1 = ubuf + (size_t)((t - 1) & 1) * fieldU;
        uo = ubuf + (size_t)(t & 1) * fieldU;
        u2 = uo;
      }
      if (mode == DUFWI_STORE_CHECKPOINT && t % K == 0) {
        // segment start: keep (u[t-1], u[t-2]) for the adjoint's recomputation
        float* sp = snap + (size_t)(t / K) * 2 * fieldU;
        if (t == 0) {
          CUDA_TRY(cudaMemsetAsync(sp, 0, 2 * fieldU * sizeof(float), st));
        } else {
          CUDA_TRY(cudaMemcpyAsync(sp, u1, fieldU * sizeof(float), cudaMemcpyDeviceToDevice, st));
          CUDA_TRY(cudaMemcpyAsync(sp + fieldU, u2, fieldU * sizeof(float),
                                   cudaMemcpyDeviceToDevice, st));
        }
      }
      rc = fwd_step_launch(p, m, mode == DUFWI_STORE_STRIPS ? 2 : 0, t, unit_begin, U, u1, u2, uo,
                           rec_t, st_t, has1, has2, st, &tc);
      if (rc) return rc;
    }
  }
  if (traces_dev) {
    const size_t total = (size_t)U * g.R * g.nt;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)p->sms * 16);
    gather_traces_kernel<<<blocks, 256, 0, st>>>(g, unit_begin, U, rec, p->rx_slot, traces_dev,
                                                 nonfinite_dev ? nonfinite_dev : p->flag);
    LAUNCH_CHECK(p);
  }
  return DUFWI_OK;
}

// ================================================================= residual
extern "C" int dufwi_residual(dufwi_plan_t* p, int32_t unit_begin, int32_t U,
                              const float* traces_dev, const double* obs_dev, double* misfit_dev,
                              void* ws, size_t ws_bytes, void* stream) {
  if (!p || !traces_dev || !obs_dev || !misfit_dev || !ws)
    return fail(DUFWI_EINVAL, "null argument");
  int rc = check_units(p, unit_begin, U);
  if (rc) return rc;
  const Layout L = layout(p, DUFWI_STORE_NONE, U);
  if (ws_bytes < L.rec) return fail(DUFWI_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->geo;
  char* base = static_cast<char*>(ws);
  double* rres = reinterpret_cast<double*>(base + L.rres);
  double* mu = reinterpret_cast<double*>(base + L.mis);
  const size_t rres_bytes = (size_t)g.nt * U * g.M * sizeof(double);
  CUDA_TRY(cudaMemsetAsync(rres, 0, rres_bytes, st));
  residual_kernel<256><<<dim3(kResidualSplit, U), 256, 0, st>>>(g, unit_begin, U, traces_dev, obs_dev, p->rx_slot,
                                          p->rx_next, p->rx_head, rres, mu);
  LAUNCH_CHECK(p);
  misfit_sum_kernel<<<1, 32, 0, st>>>(g, unit_begin, U, mu, misfit_dev);
  LAUNCH_CHECK(p);
  return DUFWI_OK;
}

// ================================================================== adjoint
extern "C" int dufwi_adjoint(dufwi_plan_t* p, int32_t mode, int32_t unit_begin, int32_t U,
                             void* ws, size_t ws_bytes, double* acc_dev, void* stream) {
  if (!p || !ws || !acc_dev) return fail(DUFWI_EINVAL, "null argument");
  if (mode != DUFWI_STORE_FULL && mode != DUFWI_STORE_STRIPS && mode != DUFWI_STORE_CHECKPOINT &&
      mode != DUFWI_STORE_LAP)
    return fail(DUFWI_EINVAL, "adjoint needs FULL, STRIPS, CHECKPOINT or LAP history");
  int rc = check_units(p, unit_begin, U);
  if (rc) return rc;
  Layout L;
  rc = ws_check(p, mode, unit_begin, U, ws_bytes, L);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->geo;
  const Model m = model_of(p);
  char* base = static_cast<char*>(ws);
  const double* rres = reinterpret_cast<const double*>(base + L.rres);
  float* rec = reinterpret_cast<float*>(base + L.rec);
  float* ubuf = reinterpret_cast<float*>(base + L.ubuf);
  float* hist = reinterpret_cast<float*>(base + L.hist);
  float* strips = reinterpret_cast<float*>(base + L.strips);
  float* snap = reinterpret_cast<float*>(base + L.snap);
  float* lbuf = reinterpret_cast<float*>(base + L.lbuf);
  double* acc_part = reinterpret_cast<double*>(base + L.acc_part);
  const size_t N2 = (size_t)g.nx * g.nz;
  const size_t fieldU = (size_t)U * N2;

  const bool clus = use_cluster(p, mode);
  const Groups G = groups_for(p, unit_begin, U, clus);
  if (clus) {
    p->last_engine = DUFWI_ENGINE_CLUSTER;
    // per-unit accumulators: with one shot per group, group index == chunk-local unit
    const int acc_off = 0;
    rc = cluster_adjoint(g, m, pick_cluster(p->ccands, U, true), mode, unit_begin, U, rres,
                         (mode == DUFWI_STORE_FULL || mode == DUFWI_STORE_LAP) ? hist : nullptr,
                         mode == DUFWI_STORE_STRIPS ? strips : nullptr, ubuf, acc_part, acc_off,
                         st);
    if (rc) return fail(DUFWI_ECUDA, std::string("cluster adjoint: ") + cudaGetErrorString((cudaError_t)rc));
    ++p->launches;
  } else {
    p->last_engine = DUFWI_ENGINE_STEPWISE;
    CUDA_TRY(cudaMemsetAsync(acc_part, 0, (size_t)G.ngroups * N2 * sizeof(double), st));
    TileCtx tc;
    {
      const bool ck = mode == DUFWI_STORE_CHECKPOINT;
      const bool hh = mode == DUFWI_STORE_FULL || ck;
      tile_ctx_build(p, U, ubuf, lbuf, hh ? hist : nullptr, ck ? (size_t)ck_len(g.nt) : (size_t)g.nt,
                     ck ? snap : nullptr, ck ? (size_t)ck_segments(g.nt) * 2 : 0, tc);
      if (use_tile(p) && !tc.ok)
        return fail(DUFWI_ECUDA, "tensor map encoding failed (workspace not 16-byte aligned?)");
    }
    auto adj_step = [&](int t, const float* F) {
      const float* l1 = lbuf + (size_t)((t + 1) & 1) * fieldU;
      float* l2o = lbuf + (size_t)(t & 1) * fieldU;
      const double* rres_t = rres + (size_t)t * U * g.M;
      float* ut = ubuf + (size_t)(t & 1) * fieldU;
      const float* utm1 = ubuf + (size_t)((t - 1) & 1) * fieldU;
      const bool strip = mode == DUFWI_STORE_STRIPS;
      const float* st_tm1 = (strip && t >= 1) ? strips + (size_t)(t - 1) * U * g.SL : nullptr;
      const float* st_tm2 = (strip && t >= 2) ? strips + (size_t)(t - 2) * U * g.SL : nullptr;
      return adj_step_launch(p, m, strip ? 2 : 1, t, unit_begin, U, G, l1, l2o, rres_t,
                             t >= 1 ? F : nullptr, ut, utm1, st_tm1, st_tm2, acc_part, st, &tc);
    };
    if (mode == DUFWI_STORE_CHECKPOINT) {
      // segments last to first: recompute the segment's fields u[s0-1 .. s1-2]
      // from its snapshot (the same kernels on the same f32 inputs: the same
      // bits as the first forward), then run its adjoint steps on them
      const int K = ck_len(g.nt), nseg = ck_segments(g.nt);
      for (int sgi = nseg - 1; sgi >= 0; --sgi) {
        const int s0 = sgi * K, s1 = std::min(g.nt, s0 + K);
        const float* sp = snap + (size_t)sgi * 2 * fieldU;
        CUDA_TRY(cudaMemcpyAsync(hist, sp, fieldU * sizeof(float), cudaMemcpyDeviceToDevice, st));
        for (int t = s0; t <= s1 - 2; ++t) {
          const float* u1 = hist + (size_t)(t - s0) * fieldU;
          const float* u2 = t == s0 ? sp + fieldU : hist + (size_t)(t - s0 - 1) * fieldU;
          rc = fwd_step_launch(p, m, 0, t, unit_begin, U, u1, u2, hist + (size_t)(t - s0 + 1) * fieldU,
                               rec + (size_t)t * U * g.M, nullptr, t >= 1, t >= 2, st, &tc);
          if (rc) return rc;
        }
        for (int t = s1 - 1; t >= s0; --t) {
          rc = adj_step(t, hist + (size_t)(t - s0) * fieldU);  // F = u[t-1]
          if (rc) return rc;
        }
      }
    } else {
      for (int t = g.nt - 1; t >= 0; --t) {
        const float* F = (mode == DUFWI_STORE_FULL && t >= 1) ? hist + (size_t)(t - 1) * fieldU : nullptr;
        rc = adj_step(t, F);
        if (rc) return rc;
      }
    }
  }
  {
    const size_t total = (size_t)G.nb * N2;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)p->sms * 16);
    // the lean density kernels sum D(u) lam; L_rho = rho D: scale by rho once here
    const double* scale = (!clus && p->has_rho && use_lean(p)) ? p->rho : nullptr;
    reduce_groups_kernel<<<blocks, 256, 0, st>>>(g, G.b0, G.nb, G.first, G.gpp, acc_part, acc_dev,
                                                 scale);
    LAUNCH_CHECK(p);
  }
  return DUFWI_OK;
}
// ================================================================= finalize
extern "C" int dufwi_finalize_gradient(dufwi_plan_t* p, const double* acc_dev, int32_t apply_mask,
                                       int32_t guard, double* grad_dev, int32_t* nonfinite_dev,
                                       void* stream) {
  if (!p || !acc_dev || !grad_dev || !nonfinite_dev) return fail(DUFWI_EINVAL, "null argument");
  if (guard < 0) return fail(DUFWI_EINVAL, "guard radius must be >= 0");
  const Geo& g = p->geo;
  const size_t total = (size_t)g.B * g.nx * g.nz;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)p->sms * 16);
  finalize_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      g, acc_dev, p->dEdc, p->elements, p->E, p->el_box[0], p->el_box[1], p->el_box[2], p->el_box[3],
      apply_mask, guard, p->dx * p->dx, grad_dev, nonfinite_dev);
  LAUNCH_CHECK(p);
  return DUFWI_OK;
}

extern "C" int64_t dufwi_plan_launch_count(const dufwi_plan_t* p) { return p ? p->launches : -1; }
extern "C" int32_t dufwi_plan_last_engine(const dufwi_plan_t* p) { return p ? p->last_engine : -1; }
extern "C" int32_t dufwi_plan_info(const dufwi_plan_t* p, int64_t* out, int32_t n) {
  if (!p || !out) return 0;
  const int64_t v[13] = {p->cluster_ok ? 1 : 0, p->ccfg.cs, p->ccfg.rows, p->ccfg.rpt,
                         p->ccfg.threads, p->ccfg.dbl, (int64_t)p->ccfg.smem_fwd,
                         (int64_t)p->ccfg_adj.smem_adj, p->ccfg.maxc, p->ccfg_adj.cs,
                         p->ccfg_adj.rpt, p->ccfg_adj.threads,
                         use_tile(p) ? 3 : use_lean(p) ? 0 : use_vec(p) ? 1 : 2};
  const int k = n < 13 ? n : 13;
  for (int i = 0; i < k; ++i) out[i] = v[i];
  return k;
}
#ifdef DUFWI_EXP_TIMING
extern "C" int dufwi_debug_counters(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_dbg, sizeof(unsigned long long) * (n < 512 ? n : 512));
  unsigned long long z[512] = {0};  // g_dbg holds 512 counters
  cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
  return 0;
}
#endif
extern "C" const char* dufwi_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* dufwi_version(void) { return "dufwi-b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------- update-net glue
namespace dufwi {
// max |g| per map as ordered bits (|g| >= 0: integer order = float order; NaN sorts last)
__global__ void net_peak_kernel(const double* __restrict__ g, long long n,
                                unsigned long long* __restrict__ peak) {
  const int b = blockIdx.y;
  const double* gb = g + (size_t)b * n;
  unsigned long long m = 0ull;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)__double_as_longlong(fabs(gb[i])));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(peak + b, m);
}
__global__ void net_input_kernel(const double* __restrict__ c, const double* __restrict__ g,
                                 long long n, double offset, double inv_scale,
                                 const unsigned long long* __restrict__ peak,
                                 float* __restrict__ x) {
  const int b = blockIdx.y;
  const double pk = __longlong_as_double((long long)peak[b]);
  const bool pos = pk > 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const size_t k = (size_t)b * n + i;
    // (c - offset) * (1 / scale): the scalar division of torch's CUDA kernels
    x[(size_t)b * 2 * n + i] = __double2float_rn(__dmul_rn(__dsub_rn(c[k], offset), inv_scale));
    x[(size_t)b * 2 * n + n + i] = pos ? __double2float_rn(__ddiv_rn(g[k], pk)) : 0.f;
  }
}
__global__ void apply_update_kernel(const double* __restrict__ c, const float* __restrict__ h,
                                    long long count, double scale, double lo, double hi,
                                    double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = __dadd_rn(c[i], __dmul_rn((double)h[i], scale));
    out[i] = v < lo ? lo : (v > hi ? hi : v);
  }
}
}  // namespace dufwi

extern "C" int dufwi_net_input(const double* c_dev, const double* g_dev, int32_t B, int64_t n,
                               double offset, double scale, double* peak_ws, float* x_out,
                               void* stream) {
  using namespace dufwi;
  if (!c_dev || !g_dev || !peak_ws || !x_out) return fail(DUFWI_EINVAL, "null argument");
  if (B <= 0 || n <= 0) return fail(DUFWI_EINVAL, "need B > 0 maps of n > 0 cells");
  if (!(scale != 0.0)) return fail(DUFWI_EINVAL, "scale must be non-zero");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(peak_ws, 0, (size_t)B * sizeof(double), st));
  const int bx = (int)std::min<long long>((n + 255) / 256, device_sms());
  const dim3 grid(bx, B);
  net_peak_kernel<<<grid, 256, 0, st>>>(g_dev, n, reinterpret_cast<unsigned long long*>(peak_ws));
  CUDA_TRY(cudaGetLastError());
  net_input_kernel<<<grid, 256, 0, st>>>(c_dev, g_dev, n, offset, 1.0 / scale,
                                         reinterpret_cast<const unsigned long long*>(peak_ws), x_out);
  CUDA_TRY(cudaGetLastError());
  return DUFWI_OK;
}

extern "C" int dufwi_apply_update(const double* c_dev, const float* h_dev, int64_t count,
                                  double scale, double lo, double hi, double* c_out, void* stream) {
  using namespace dufwi;
  if (!c_dev || !h_dev || !c_out) return fail(DUFWI_EINVAL, "null argument");
  if (count <= 0) return fail(DUFWI_EINVAL, "count must be positive");
  if (!(lo < hi)) return fail(DUFWI_EINVAL, "bounds must satisfy lo < hi");
  const int blocks = (int)std::min<long long>((count + 255) / 256, (long long)device_sms() * 8);
  apply_update_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(c_dev, h_dev, count, scale, lo, hi,
                                                                c_out);
  CUDA_TRY(cudaGetLastError());
  return DUFWI_OK;
}

// ----------------------------------------------------- field utilities
extern "C" int dufwi_laplacian(const double* u_dev, int64_t batch, int32_t nx, int32_t nz,
                               double dx, double* out_dev, void* stream) {
  using namespace dufwi;
  if (!u_dev || !out_dev) return fail(DUFWI_EINVAL, "null argument");
  if (batch < 0 || nx < 1 || nz < 1) return fail(DUFWI_EINVAL, "bad field shape");
  if (!(dx > 0)) return fail(DUFWI_EINVAL, "dx must be positive");
  if (u_dev == out_dev) return fail(DUFWI_EINVAL, "out must not alias u");
  const long long total = batch * (long long)nx * nz;
  if (total == 0) return DUFWI_OK;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)device_sms() * 8);
  laplacian_f64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(u_dev, batch, nx, nz, dx * dx,
                                                                 out_dev);
  CUDA_TRY(cudaGetLastError());
  return DUFWI_OK;
}

extern "C" int dufwi_step_field(const double* u1_dev, const double* u2_dev, const double* c_dev,
                                const double* d_dev, const double* s_dev, int32_t nx, int32_t nz,
                                double dx, double dt, double* out_dev, void* stream) {
  using namespace dufwi;
  if (!u1_dev || !u2_dev || !c_dev || !d_dev || !s_dev || !out_dev)
    return fail(DUFWI_EINVAL, "null argument");
  if (nx < 1 || nz < 1) return fail(DUFWI_EINVAL, "bad field shape");
  if (!(dx > 0) || !(dt > 0)) return fail(DUFWI_EINVAL, "dx, dt must be positive");
  if (out_dev == u1_dev) return fail(DUFWI_EINVAL, "out must not alias u_prev");
  const long long n = (long long)nx * nz;
  const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)device_sms() * 8);
  step_field_f64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(u1_dev, u2_dev, c_dev, d_dev,
                                                                  s_dev, nx, nz, dx * dx, dt,
                                                                  out_dev);
  CUDA_TRY(cudaGetLastError());
  return DUFWI_OK;
}
