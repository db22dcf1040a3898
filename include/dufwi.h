/*
 * dufwi.h — C ABI of the B200-native DUFWI physics step (libdufwi.so).
 *
 * The reference (fwilab, pure Python/NumPy) has no FFI; its hot-path seam is
 *   forward._propagate(c, d, grid, pulse, tx (P,2), rx (P,R,2), store_fields)
 *       reference: pkg/src/fwilab/forward.py:273-313
 * plus the inline reverse sweep of
 *   adjoint.misfit_and_gradient(sos, m_obs, pulse, damping, mask, guard_radius)
 *       reference: pkg/src/fwilab/adjoint.py:94-138
 * Each entry point below replaces one piece of that seam (cited per function).
 * INTEGRATION.md shows the ctypes binding the reference would add.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no torch types.
 *   - "dev" pointers are CUDA device memory owned by the caller; "host"
 *     pointers are read during the call only.  The library never frees caller
 *     memory.  A plan owns the small derived tables it allocates.
 *   - Work is enqueued on the caller's stream (cudaStream_t passed as void*);
 *     calls return after enqueueing, except where noted.
 *   - Reentrant: no mutable global state other than a thread-local last-error
 *     string.  Different plans may be used concurrently from different threads.
 *   - Return codes: 0 ok, 1 invalid argument, 2 CUDA error, 3 non-finite values.
 *
 * Grid layout: every field is row-major [nx][nz] (z contiguous), matching the
 * reference's (nx, nz) arrays.  A "unit" is one (phantom b, shot s) pair,
 * u = b*S + s; units are processed in contiguous ranges [unit_begin,
 * unit_begin+unit_count) so callers can bound memory and shard across GPUs.
 */
#ifndef DUFWI_H_
#define DUFWI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DUFWI_OK 0
#define DUFWI_EINVAL 1
#define DUFWI_ECUDA 2
#define DUFWI_ENONFINITE 3

/* Wavefield history strategy for the adjoint. */
#define DUFWI_STORE_NONE 0   /* forward only: no history (simulate_all)            */
#define DUFWI_STORE_FULL 1   /* full f32 history [nt][units][nx][nz] in workspace  */
#define DUFWI_STORE_STRIPS 2 /* 1-cell ring around the undamped box per step + the
                                last two states; interior reconstructed backwards */
#define DUFWI_STORE_LAP 4  /* cluster engine: the forward stores L(u[t]) of every cell
                              of the undamped box and step (f32), the imaging operand, so
                              the adjoint carries only lam: no u state, no reconstruction
                              (masked gradients, like STRIPS) */
#define DUFWI_STORE_CHECKPOINT 3 /* snapshots (u[s0-1], u[s0-2]) every K = ceil(sqrt(2 nt))
                                    steps; the adjoint recomputes each segment's fields
                                    from its snapshot (any damping; bit-identical to FULL) */

/* Engine selection (dufwi_geometry_t.engine). */
#define DUFWI_ENGINE_AUTO 0    /* persistent cluster sweep when the grid fits, else stepwise */
#define DUFWI_ENGINE_STEPWISE 1/* one launch per time step over all units                    */
#define DUFWI_ENGINE_CLUSTER 2 /* one launch per sweep, one thread-block cluster per unit    */

/* Arithmetic of the sweep kernels (dufwi_geometry_t.arith).  Fields, traces and
 * strips are f32 in HBM either way.
 *   F32: every update in f32, in the increment form
 *        u[t] = u1 + ((u1 - u2) + (A-2) u1 + (B+1) u2 + E L(u1)),
 *        L by differences (u_j - u_c): the error of "f64 arithmetic, f32 storage"
 *        (traces ~5e-7, fixed-observation gradients ~5e-6 against the reference),
 *        inside the 1e-4 / 1e-3 bars at every BASELINE size.  The fast path.
 *   F64: every update in f64 in the reference's operation order (forward.py:301-308);
 *        on the cluster engine the whole sweep is then a float64 computation
 *        (traces ~3e-8).  For callers that difference misfits (fd_gradient_oracle)
 *        or iterate to convergence on a shrinking residual (ADMM-TV FWI). */
#define DUFWI_ARITH_F32 0
#define DUFWI_ARITH_F64 1

typedef struct dufwi_geometry {
  int32_t nx, nz, nt;       /* grid and time axis (grid.py:42-84)                 */
  int32_t n_phantoms;       /* B                                                  */
  int32_t n_shots;          /* S transmissions per phantom                        */
  int32_t n_rx;             /* R receivers per transmission                       */
  int32_t n_elements;       /* E element nodes (for the gradient guard mask)      */
  int32_t has_rho;          /* 1: variable density model         */
  int32_t engine;           /* DUFWI_ENGINE_*                                     */
  int32_t arith;            /* DUFWI_ARITH_* (0 = f32, the default)               */
  double dx, dt;
  const int32_t* tx_host;       /* [S][2]   transmit node (ix, iz) per shot       */
  const int32_t* rx_host;       /* [S][R][2] receiver nodes per shot              */
  const int32_t* elements_host; /* [E][2]   all element nodes                     */
  const double* px_host;        /* [nx] damping profile along x, or NULL          */
  const double* pz_host;        /* [nz] damping profile along z, or NULL          */
  const double* damping_host;   /* [nx][nz] general damping, used iff px_host NULL*/
  const double* pulse_host;     /* [nt] source samples                            */
} dufwi_geometry_t;

typedef struct dufwi_plan dufwi_plan_t;

/* Build the derived device tables (receiver slots, damping, pulse).
 * Replaces the per-call setup of forward._propagate / _check_simulation_inputs
 * (forward.py:256-270, 289-299).  Allocates on the current CUDA device. */
int dufwi_plan_create(const dufwi_geometry_t* geo, dufwi_plan_t** plan_out);
int dufwi_plan_destroy(dufwi_plan_t* plan);

/* Load the speed map c [B][nx][nz] (and rho [B][nx][nz] or NULL), computing the
 * per-cell coefficients E/dx^2 and dE/dc on device.
 * Replaces step_coefficients (forward.py:226-234) and adjoint.py:116-117. */
int dufwi_set_model(dufwi_plan_t* plan, const double* c_dev, const double* rho_dev,
                    void* stream);

/* Workspace bytes for a sweep over unit_count units with the given store mode. */
int dufwi_workspace_bytes(const dufwi_plan_t* plan, int32_t store_mode,
                          int32_t unit_count, size_t* bytes_out);

/* Forward sweep over units [unit_begin, unit_begin+unit_count): update, source
 * injection, receiver sampling, history storage.  traces_dev [units][R][nt] f32
 * in the reference's ChannelData layout (grid.py:164-183), may be NULL.
 * *nonfinite_dev (int32, may be NULL) is set to 1 if a sample is non-finite
 * (forward.py:309-312).  Replaces forward._propagate (forward.py:273-313). */
int dufwi_forward(dufwi_plan_t* plan, int32_t store_mode, int32_t unit_begin,
                  int32_t unit_count, float* traces_dev, int32_t* nonfinite_dev,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Byte offset of the f32 wavefield history [nt][units][nx][nz] inside a
 * DUFWI_STORE_FULL workspace for unit_count units (simulate_wavefield,
 * forward.py:316-332, reads it back). */
int dufwi_history_offset(const dufwi_plan_t* plan, int32_t unit_count, size_t* offset_out);

/* r = 2 (traces - obs) merged per receiver node into the workspace, and the
 * misfit sum((traces-obs)^2) per unit added into misfit_dev [B] (f64).
 * obs_dev [units][R][nt] f64.  Replaces adjoint.py:113-114 (data_misfit :67-72). */
int dufwi_residual(dufwi_plan_t* plan, int32_t unit_begin, int32_t unit_count,
                   const float* traces_dev, const double* obs_dev, double* misfit_dev,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Reverse sweep with residual injection and zero-lag imaging; adds
 * sum_t sum_shots lap(u[t-1]) * lam[t] into acc_dev [B][nx][nz] (f64, not yet
 * scaled by dE/dc / dx^2).  Uses the history written by dufwi_forward with the
 * same store mode and workspace.  Replaces adjoint.py:119-131. */
int dufwi_adjoint(dufwi_plan_t* plan, int32_t store_mode, int32_t unit_begin,
                  int32_t unit_count, void* workspace, size_t workspace_bytes,
                  double* acc_dev, void* stream);

/* grad = mask ? dE/dc * acc / dx^2 : 0 (mask: undamped cells farther than
 * guard_radius from every element).  Sets *nonfinite_dev (int32) to 1 if any
 * accumulated value is non-finite.  Replaces adjoint.py:133-137 and
 * gradient_mask (adjoint.py:75-91). */
int dufwi_finalize_gradient(dufwi_plan_t* plan, const double* acc_dev, int32_t apply_mask,
                            int32_t guard_radius, double* grad_dev, int32_t* nonfinite_dev,
                            void* stream);

/* Input of a DUFWI update network for B maps of n cells each (no plan needed):
 * x_out [B][2][n] f32 = ((c - offset) * (1 / scale), g / max|g|), the second channel 0
 * where max|g| == 0; peak_ws: B doubles of device scratch.  Replaces the
 * reference's normalize_sos / normalize_gradient and channel stack
 * (network.py:56-68, 265) on the device (f64; the first channel multiplies by
 * the reciprocal, as torch's CUDA division by a scalar does). */
int dufwi_net_input(const double* c_dev, const double* g_dev, int32_t B, int64_t n,
                    double offset, double scale, double* peak_ws, float* x_out, void* stream);

/* c_out = clamp(c + scale * h, lo, hi) for count cells, h the network's f32
 * output: the denormalised update and clamp_sos of one unfolded stage
 * (unfold.py:263-265, network.py:229).  NaN propagates as in NumPy's clip. */
int dufwi_apply_update(const double* c_dev, const float* h_dev, int64_t count, double scale,
                       double lo, double hi, double* c_out, void* stream);

/* 5-point Laplacian with zeros outside the grid of `batch` f64 fields [nx][nz]
 * (u_dev, out_dev: batch*nx*nz doubles, out must not alias u), in the
 * reference's accumulation order: out = -4u, += x-1, += x+1, += z-1, += z+1,
 * /= dx*dx — bit-identical to NumPy.  Replaces forward.laplacian
 * (forward.py:211-223). */
int dufwi_laplacian(const double* u_dev, int64_t batch, int32_t nx, int32_t nz, double dx,
                    double* out_dev, void* stream);

/* One explicit step of one f64 field (forward.py:237-253):
 * out = A u1 + B u2 + E lap(u1) + s with A, B, E = step_coefficients(c, d, dt)
 * (forward.py:226-234), every operation rounded as NumPy does.  All arrays
 * [nx][nz]; out must not alias u1.  Replaces forward.step_wavefield. */
int dufwi_step_field(const double* u1_dev, const double* u2_dev, const double* c_dev,
                     const double* d_dev, const double* s_dev, int32_t nx, int32_t nz, double dx,
                     double dt, double* out_dev, void* stream);

/* Number of kernels this plan has launched so far (evidence for benchmarks). */
int64_t dufwi_plan_launch_count(const dufwi_plan_t* plan);

/* Engine actually used for the last forward/adjoint call (DUFWI_ENGINE_*). */
int32_t dufwi_plan_last_engine(const dufwi_plan_t* plan);

/* Engine diagnostics: out[0..12] = cluster_ok, cluster CTAs, rows per CTA,
 * rows per thread, threads per CTA, f64 exchange, smem forward, smem adjoint,
 * co-resident clusters (the forward's shape), then the adjoint's cluster CTAs,
 * rows per thread and threads per CTA — for all units at once — and the
 * stepwise kernel family (0 lean: nz % 4 == 0, separable damping with a
 * rectangular undamped box; 1 vec: other constant-density grids with
 * nz % 4 == 0; 2 stream: everything else).
 * Returns the number of values written (<= n). */
int32_t dufwi_plan_info(const dufwi_plan_t* plan, int64_t* out, int32_t n);

/* Thread-local message for the last non-zero return code on this thread. */
const char* dufwi_last_error(void);

/* Library version string. */
const char* dufwi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DUFWI_H_ */
