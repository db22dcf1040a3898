/*
 * TEST INFRASTRUCTURE — float64 C restatement of the reference's physics step.
 *
 * This is a checker, never a product path: only tests/, bench.py's cpu_baseline
 * leg and the fixture scripts under oracle/ load it (through oracle/c_oracle.py).
 * It restates, for one transmission at a time, exactly the arithmetic of
 * oracle/dufwi_oracle.py, which in turn restates the reference
 * (/root/reference/pkg/src/fwilab):
 *
 *   forward step   forward.py:301-308   u = (A*u1 + B*u2) + E*L(u1); u[tx] += s[t];
 *                                       traces[:, t] = u[rx]
 *   Laplacian      forward.py:211-223   acc = -4u; += x-1; += x+1; += z-1; += z+1;
 *                                       acc /= dx*dx   (zero outside the grid)
 *   adjoint step   adjoint.py:125-131   lam = (A*l1 + L^T(E*l1)) + B*l2;
 *                                       lam[rx_r] += r[r, t] in receiver order;
 *                                       t >= 1: img += L(u[t-1]) * lam
 *   residual       adjoint.py:113-114   r = 2*(traces - obs)
 *
 * Variable density (parity unpinned by the reference) takes the
 * five face-weight maps of oracle.rho_face_weights: L = lap_rho, L^T = lap_rho_T,
 * with the same accumulation order as the NumPy restatement.
 *
 * Differences from the NumPy restatement, all below 1e-13 relative:
 *  - transmissions are independent (forward.py:286-288), so each runs on its own
 *    thread; the imaging sums are returned per transmission without the dE/dc
 *    factor, summed in shot order and scaled once by the caller
 *    (NumPy: grad += dEdc * sum_p(...) every step);
 *  - the forward history is not stored (the reference keeps all nt fields,
 *    forward.py:299): every `seg` steps the state (u[t-1], u[t-2]) is saved and
 *    the adjoint recomputes each segment's fields from its snapshot.  The
 *    recursion is deterministic in float64, so the recomputed fields are
 *    bit-identical to the stored ones (checked by tests/test_c_oracle.py).
 *
 * Build: gcc -O3 -ffp-contract=off -pthread -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps every multiply and add separately rounded, as NumPy does.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef struct {
    int nx, nz, nt;
    double dx2;                 /* dx*dx, as forward.py:222 divides by it */
    const double *A, *B, *E;    /* step_coefficients, forward.py:226-234 */
    const double *w;            /* NULL (lap5) or 5 maps: w_xm, w_xp, w_zm, w_zp, wsum */
    const double *pulse;        /* nt */
} model_t;

/* L(u) at every cell (forward.py:211-223, or oracle.lap_rho). */
static void apply_L(const model_t *m, const double *u, double *out)
{
    const int nx = m->nx, nz = m->nz;
    const double dx2 = m->dx2;
    if (!m->w) {
        for (int i = 0; i < nx; ++i) {
            const double *r = u + (size_t)i * nz;
            const double *up = i > 0 ? r - nz : NULL;
            const double *dn = i < nx - 1 ? r + nz : NULL;
            double *o = out + (size_t)i * nz;
            for (int j = 0; j < nz; ++j) {
                double acc = -4.0 * r[j];
                if (up) acc += up[j];
                if (dn) acc += dn[j];
                if (j > 0) acc += r[j - 1];
                if (j < nz - 1) acc += r[j + 1];
                o[j] = acc / dx2;
            }
        }
        return;
    }
    const size_t N = (size_t)nx * nz;
    const double *wxm = m->w, *wxp = m->w + N, *wzm = m->w + 2 * N, *wzp = m->w + 3 * N,
                 *ws = m->w + 4 * N;
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < nz; ++j) {
            const size_t k = (size_t)i * nz + j;
            double acc = -ws[k] * u[k];
            if (i > 0) acc += wxm[k] * u[k - nz];
            if (i < nx - 1) acc += wxp[k] * u[k + nz];
            if (j > 0) acc += wzm[k] * u[k - 1];
            if (j < nz - 1) acc += wzp[k] * u[k + 1];
            out[k] = acc / dx2;
        }
    }
}

/* L^T(v) (lap5 is symmetric; oracle.lap_rho_T otherwise). */
static void apply_LT(const model_t *m, const double *v, double *out)
{
    if (!m->w) {
        apply_L(m, v, out);
        return;
    }
    const int nx = m->nx, nz = m->nz;
    const size_t N = (size_t)nx * nz;
    const double dx2 = m->dx2;
    const double *wxm = m->w, *wxp = m->w + N, *wzm = m->w + 2 * N, *wzp = m->w + 3 * N,
                 *ws = m->w + 4 * N;
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < nz; ++j) {
            const size_t k = (size_t)i * nz + j;
            double acc = -ws[k] * v[k];
            if (i > 0) acc += wxp[k - nz] * v[k - nz];
            if (i < nx - 1) acc += wxm[k + nz] * v[k + nz];
            if (j > 0) acc += wzp[k - 1] * v[k - 1];
            if (j < nz - 1) acc += wzm[k + 1] * v[k + 1];
            out[k] = acc / dx2;
        }
    }
}

/* One forward step: cur = (A*prev + B*prev2) + E*L(prev); inject; sample. */
static void fwd_step(const model_t *m, const double *prev, const double *prev2, double *cur,
                     double *lap, int t, const int *tx, int R, const int *rx, double *traces)
{
    const size_t N = (size_t)m->nx * m->nz;
    apply_L(m, prev, lap);
    for (size_t k = 0; k < N; ++k)
        cur[k] = (m->A[k] * prev[k] + m->B[k] * prev2[k]) + m->E[k] * lap[k];
    cur[(size_t)tx[0] * m->nz + tx[1]] += m->pulse[t];
    if (traces)
        for (int r = 0; r < R; ++r)
            traces[(size_t)r * m->nt + t] = cur[(size_t)rx[2 * r] * m->nz + rx[2 * r + 1]];
}

static int nonfinite(const double *a, size_t n)
{
    for (size_t k = 0; k < n; ++k)
        if (!(a[k] - a[k] == 0.0)) return 1;
    return 0;
}


/* Shots are handed to n_threads pthreads in index order through a shared counter;
 * every shot writes only its own outputs, so results do not depend on the count. */
typedef struct {
    pthread_mutex_t mu;
    int next, P, bad;
    void (*fn)(void *ctx, int p, int *bad);
    void *ctx;
} pool_t;

static void *pool_worker(void *arg)
{
    pool_t *q = arg;
    for (;;) {
        pthread_mutex_lock(&q->mu);
        const int p = q->next++;
        pthread_mutex_unlock(&q->mu);
        if (p >= q->P) return NULL;
        int bad = 0;
        q->fn(q->ctx, p, &bad);
        if (bad) {
            pthread_mutex_lock(&q->mu);
            q->bad = 1;
            pthread_mutex_unlock(&q->mu);
        }
    }
}

static int run_pool(int P, int n_threads, void (*fn)(void *, int, int *), void *ctx)
{
    pool_t q = {PTHREAD_MUTEX_INITIALIZER, 0, P, 0, fn, ctx};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > P) n_threads = P;
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, pool_worker, &q);
    pool_worker(&q);
    for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
    return q.bad;
}

/* Forward sweep of one shot: traces (R, nt); optional snapshots of (u[s0-1], u[s0-2])
 * at every segment start s0 = s*seg (snap: n_seg x 2 x N). */
static void forward_shot(const model_t *m, const int *tx, int R, const int *rx, double *traces,
                         int seg, double *snap)
{
    const size_t N = (size_t)m->nx * m->nz;
    double *buf = calloc(4 * N, sizeof(double));
    double *prev = buf, *prev2 = buf + N, *cur = buf + 2 * N, *lap = buf + 3 * N;
    for (int t = 0; t < m->nt; ++t) {
        if (snap && t % seg == 0) {
            double *s = snap + (size_t)(t / seg) * 2 * N;
            memcpy(s, prev, N * sizeof(double));
            memcpy(s + N, prev2, N * sizeof(double));
        }
        fwd_step(m, prev, prev2, cur, lap, t, tx, R, rx, traces);
        double *tmp = prev2;
        prev2 = prev;
        prev = cur;
        cur = tmp;
    }
    free(buf);
}

/* Receiver traces of P shots: traces (P, R, nt) (forward.py:273-313). */
typedef struct {
    model_t m;
    const int *tx, *rx;
    int R, seg;
    const double *obs;
    double *traces, *img;
} job_t;

static void forward_job(void *ctx, int p, int *bad)
{
    job_t *j = ctx;
    const size_t RT = (size_t)j->R * j->m.nt;
    double *tr = j->traces + p * RT;
    forward_shot(&j->m, j->tx + 2 * p, j->R, j->rx + (size_t)2 * p * j->R, tr, 1 << 30, NULL);
    *bad = nonfinite(tr, RT);
}

int dufwi_oracle_forward(int nx, int nz, int nt, double dx, const double *A, const double *B,
                         const double *E, const double *w, const double *pulse, int P,
                         const int *tx, int R, const int *rx, double *traces, int n_threads)
{
    job_t j = {{nx, nz, nt, dx * dx, A, B, E, w, pulse}, tx, rx, R, 0, NULL, traces, NULL};
    return run_pool(P, n_threads, forward_job, &j) ? 3 : 0;
}

/* Adjoint sweep of one shot with segment recomputation; img (N) += sum_t L(u[t-1])*lam[t]. */
static void adjoint_shot(const model_t *m, const int *tx, int R, const int *rx, const double *resid,
                         int seg, const double *snap, double *img)
{
    const size_t N = (size_t)m->nx * m->nz;
    const int nt = m->nt;
    double *hist = malloc((size_t)seg * N * sizeof(double)); /* u[s0-1 .. s1-2] */
    double *work = calloc(6 * N, sizeof(double));
    double *l1 = work, *l2 = work + N, *lam = work + 2 * N, *el = work + 3 * N,
           *tmp = work + 4 * N, *lu = work + 5 * N;
    const int n_seg = (nt + seg - 1) / seg;
    for (int s = n_seg - 1; s >= 0; --s) {
        const int s0 = s * seg, s1 = s0 + seg < nt ? s0 + seg : nt;
        /* recompute u[s0-1 .. s1-2] from the snapshot (u[s0-1], u[s0-2]) */
        const double *sp = snap + (size_t)s * 2 * N;
        memcpy(hist, sp, N * sizeof(double));
        const double *pv2 = sp + N;
        for (int t = s0; t <= s1 - 2; ++t) {
            double *cur = hist + (size_t)(t - s0 + 1) * N;
            const double *pv = hist + (size_t)(t - s0) * N;
            fwd_step(m, pv, pv2, cur, tmp, t, tx, R, rx, NULL);
            pv2 = pv;
        }
        for (int t = s1 - 1; t >= s0; --t) {
            /* lam = (A*l1 + L^T(E*l1)) + B*l2  (adjoint.py:126) */
            for (size_t k = 0; k < N; ++k) el[k] = m->E[k] * l1[k];
            apply_LT(m, el, tmp);
            for (size_t k = 0; k < N; ++k) lam[k] = (m->A[k] * l1[k] + tmp[k]) + m->B[k] * l2[k];
            /* np.add.at(lam, rx, r[:, t]) — duplicates accumulate in receiver order (:127) */
            for (int r = 0; r < R; ++r)
                lam[(size_t)rx[2 * r] * m->nz + rx[2 * r + 1]] += resid[(size_t)r * nt + t];
            if (t >= 1) { /* imaging with u[t-1] (:128-130) */
                apply_L(m, hist + (size_t)(t - 1 - (s0 - 1)) * N, lu);
                for (size_t k = 0; k < N; ++k) img[k] += lu[k] * lam[k];
            }
            double *x = l2;
            l2 = l1;
            l1 = lam;
            lam = x;
        }
    }
    free(work);
    free(hist);
}

static void gradient_job(void *ctx, int p, int *bad)
{
    job_t *j = ctx;
    const model_t *m = &j->m;
    const size_t N = (size_t)m->nx * m->nz, RT = (size_t)j->R * m->nt;
    const int n_seg = (m->nt + j->seg - 1) / j->seg;
    double *tr = j->traces + p * RT;
    double *snap = malloc((size_t)n_seg * 2 * N * sizeof(double));
    const int *txp = j->tx + 2 * p, *rxp = j->rx + (size_t)2 * p * j->R;
    forward_shot(m, txp, j->R, rxp, tr, j->seg, snap);
    double *resid = malloc(RT * sizeof(double));
    for (size_t k = 0; k < RT; ++k) resid[k] = 2.0 * (tr[k] - j->obs[p * RT + k]);
    double *img = j->img + (size_t)p * N;
    memset(img, 0, N * sizeof(double));
    adjoint_shot(m, txp, j->R, rxp, resid, j->seg, snap, img);
    *bad = nonfinite(tr, RT) | nonfinite(img, N);
    free(resid);
    free(snap);
}

/* Misfit gradient of P shots (adjoint.py:94-138 without the mask and dE/dc scale).
 * obs (P, R, nt); traces_out (P, R, nt); img_out (P, N) per-shot imaging sums.
 * Returns 0, or 3 when traces or imaging sums are non-finite. */
int dufwi_oracle_gradient(int nx, int nz, int nt, double dx, const double *A, const double *B,
                          const double *E, const double *w, const double *pulse, int P,
                          const int *tx, int R, const int *rx, const double *obs,
                          double *traces_out, double *img_out, int seg, int n_threads)
{
    job_t j = {{nx, nz, nt, dx * dx, A, B, E, w, pulse}, tx, rx, R, seg < 2 ? 2 : seg, obs,
               traces_out, img_out};
    return run_pool(P, n_threads, gradient_job, &j) ? 3 : 0;
}
