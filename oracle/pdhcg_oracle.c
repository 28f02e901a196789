/*
 * CPU ORACLE — test infrastructure only.
 *
 * A plain-C restatement of the reference's fused PDHCG chunk, used as the
 * parity checker for the CUDA path and as the CPU baseline in bench.py.
 * Nothing in the shipped package links or calls this file: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.
 *
 * Follows /root/reference/pkg/src/market_eq/kernels.py:
 *   orc_g_eval       <- _g_eval       (kernels.py:22-30)
 *   orc_row_root     <- _row_root     (kernels.py:33-96)
 *   orc_pdhcg_chunk  <- pdhcg_chunk   (kernels.py:99-145)
 *
 * Arithmetic is written operation-for-operation in the reference's order and
 * must be compiled with -ffp-contract=off (no FMA contraction), so on the
 * same inputs the results are bit-identical to the numba kernel (pinned by
 * tests/test_oracle.py against tests/golden/ vectors produced by running the
 * reference itself, see oracle/gen_golden.py).  Index layout is the B200
 * layout: int64 row offsets, int32 column indices and transpose permutation,
 * int64 transpose offsets (the reference accepts int32 there too and gives
 * bit-identical results).
 *
 * Parallel loops run on a pthread team over the same axes as numba's
 * prange; every output has one writer and every floating-point reduction is
 * serial in a fixed order, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>

#define ORC_MAX_ROW_PASSES 200          /* kernels.py:16 */
#define ORC_REL_WIDTH_FLOOR 4e-16       /* kernels.py:19 */

/* u . max(0, c + tw*u/s) over entries [a, b)  (kernels.py:22-30) */
static double orc_g_eval(int64_t a, int64_t b, const double *uval,
                         const double *cbuf, double tw, double s)
{
    double acc = 0.0;
    for (int64_t t = a; t < b; ++t) {
        double xv = cbuf[t] + (tw * uval[t]) / s;
        if (xv > 0.0)
            acc += uval[t] * xv;
    }
    return acc;
}

/* Bracketing k-section root of phi(s) = s - g(s)  (kernels.py:33-96).
 * Returns the root; *passes receives the pass count, or -1 on a fault. */
double orc_row_root(int64_t a, int64_t b, const double *uval, const double *cbuf,
                    double tw, double s0, int sections, double tol, int64_t *passes)
{
    double s_t;
    if (s0 > 0.0) {
        s_t = s0;
    } else {
        double usq = 0.0;
        for (int64_t t = a; t < b; ++t)
            usq += uval[t] * uval[t];
        s_t = sqrt(tw * usq);
        if (s_t <= 0.0)
            s_t = 1e-12 * (1.0 + tw);
    }
    double st = orc_g_eval(a, b, uval, cbuf, tw, s_t);
    if (st == s_t) {
        *passes = 0;
        return s_t;
    }
    double lo = st > s_t ? s_t : st;
    double hi = st > s_t ? st : s_t;
    int64_t np = 0;
    for (;;) {
        double floor_w = ORC_REL_WIDTH_FLOOR * (hi > 1.0 ? hi : 1.0);
        double eff = tol > floor_w ? tol : floor_w;
        if (hi - lo <= eff) {
            *passes = np;
            return 0.5 * (lo + hi);
        }
        np += 1;
        if (np > ORC_MAX_ROW_PASSES) {
            *passes = -1;
            return 0.5 * (lo + hi);
        }
        double nhi = hi, nlo = lo, exact = -1.0;
        for (int l = 1; l < sections; ++l) {
            double sl = ((double)(sections - l) * lo + (double)l * hi) / (double)sections;
            if (sl <= lo || sl >= hi)
                continue;
            double gl = orc_g_eval(a, b, uval, cbuf, tw, sl);
            if (gl == sl) {
                exact = sl;
                break;
            }
            double up = sl > gl ? sl : gl;
            double dn = sl > gl ? gl : sl;
            if (up < nhi) nhi = up;
            if (dn > nlo) nlo = dn;
        }
        if (exact >= 0.0) {
            *passes = np;
            return exact;
        }
        if (nhi == hi && nlo == lo) {
            *passes = np;
            return 0.5 * (lo + hi);
        }
        hi = nhi;
        lo = nlo;
    }
}

/* ---- a minimal pthread team (the image's gcc has no libgomp) ---- */
static int g_threads = 1;

typedef struct {
    void (*fn)(void *ctx, int64_t lo, int64_t hi, int64_t *acc);
    void *ctx;
    int64_t n, grain;
    atomic_llong next;
    int64_t acc[2];
    pthread_mutex_t mu;
} orc_job;

static void *orc_worker(void *arg)
{
    orc_job *job = (orc_job *)arg;
    int64_t local[2] = {0, 0};
    for (;;) {
        int64_t lo = atomic_fetch_add(&job->next, job->grain);
        if (lo >= job->n)
            break;
        int64_t hi = lo + job->grain < job->n ? lo + job->grain : job->n;
        job->fn(job->ctx, lo, hi, local);
    }
    pthread_mutex_lock(&job->mu);
    job->acc[0] += local[0];
    job->acc[1] += local[1];
    pthread_mutex_unlock(&job->mu);
    return NULL;
}

/* Runs fn over [0, n) in chunks of `grain`; integer accumulators are summed
 * (order-free), floating-point work never crosses a chunk boundary. */
static void orc_parallel_for(int64_t n, int64_t grain,
                             void (*fn)(void *, int64_t, int64_t, int64_t *),
                             void *ctx, int64_t acc_out[2])
{
    orc_job job;
    job.fn = fn;
    job.ctx = ctx;
    job.n = n;
    job.grain = grain < 1 ? 1 : grain;
    atomic_init(&job.next, 0);
    job.acc[0] = job.acc[1] = 0;
    pthread_mutex_init(&job.mu, NULL);
    int nt = g_threads;
    if ((int64_t)nt > (n + job.grain - 1) / job.grain)
        nt = (int)((n + job.grain - 1) / job.grain);
    if (nt <= 1) {
        orc_worker(&job);
    } else {
        pthread_t tid[256];
        if (nt > 256)
            nt = 256;
        for (int k = 1; k < nt; ++k)
            pthread_create(&tid[k], NULL, orc_worker, &job);
        orc_worker(&job);
        for (int k = 1; k < nt; ++k)
            pthread_join(tid[k], NULL);
    }
    pthread_mutex_destroy(&job.mu);
    if (acc_out) {
        acc_out[0] = job.acc[0];
        acc_out[1] = job.acc[1];
    }
}

typedef struct {
    const int64_t *indptr, *tindptr;
    const int32_t *colind, *tperm;
    const double *uval, *w;
    double *x, *x_prev, *p, *xbar, *pbar, *cbuf;
    double tau, sigma, subtol, wold, wnew;
    int sections;
} orc_state;

/* dual step: per-good ascending-row sum of 2x - x_prev (kernels.py:111-116) */
static void orc_dual(void *vs, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_state *S = (orc_state *)vs;
    (void)acc;
    for (int64_t j = lo; j < hi; ++j) {
        double a = 0.0;
        for (int64_t t = S->tindptr[j]; t < S->tindptr[j + 1]; ++t) {
            int64_t k = S->tperm[t];
            a += 2.0 * S->x[k] - S->x_prev[k];
        }
        S->p[j] += S->sigma * (a - 1.0);
    }
}

/* x_prev <- x (kernels.py:117-118) */
static void orc_copy(void *vs, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_state *S = (orc_state *)vs;
    (void)acc;
    memcpy(S->x_prev + lo, S->x + lo, (size_t)(hi - lo) * sizeof(double));
}

/* primal row step (kernels.py:120-136); acc[0] = passes, acc[1] = faults */
static void orc_primal(void *vs, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_state *S = (orc_state *)vs;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t a = S->indptr[i], b = S->indptr[i + 1];
        if (b == a)
            continue;
        double tw = S->tau * S->w[i];
        double s0 = 0.0;
        for (int64_t t = a; t < b; ++t) {
            S->cbuf[t] = S->x_prev[t] - S->tau * S->p[S->colind[t]];
            s0 += S->uval[t] * S->x_prev[t];
        }
        int64_t np;
        double s = orc_row_root(a, b, S->uval, S->cbuf, tw, s0, S->sections, S->subtol, &np);
        if (np < 0)
            acc[1] += 1;
        else
            acc[0] += np;
        for (int64_t t = a; t < b; ++t) {
            double xv = S->cbuf[t] + (tw * S->uval[t]) / s;
            S->x[t] = xv > 0.0 ? xv : 0.0;
        }
    }
}

/* running averages (kernels.py:138-144) */
static void orc_avg_x(void *vs, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_state *S = (orc_state *)vs;
    (void)acc;
    for (int64_t k = lo; k < hi; ++k)
        S->xbar[k] = S->wold * S->xbar[k] + S->wnew * S->x[k];
}

/* `iters` compact iterations in place  (kernels.py:99-145).
 * Returns the new navg; *faults_out receives the fault count. */
int64_t orc_pdhcg_chunk(int64_t n, int64_t m,
                        const int64_t *indptr, const int32_t *colind, const double *uval,
                        const int32_t *tperm, const int64_t *tindptr, const double *w,
                        double *x, double *x_prev, double *p, double *xbar, double *pbar,
                        int64_t navg, double tau, double sigma, int sections, double subtol,
                        int iters, double *cbuf, int64_t *pass_out, int64_t *faults_out)
{
    const int64_t nnz = indptr[n];
    orc_state S = {indptr, tindptr, colind, tperm, uval, w, x, x_prev, p, xbar, pbar, cbuf,
                   tau, sigma, subtol, 0.0, 0.0, sections};
    int64_t count = navg;
    int64_t faults = 0;
    for (int it = 0; it < iters; ++it) {
        orc_parallel_for(m, 64, orc_dual, &S, NULL);
        orc_parallel_for(nnz, 1 << 16, orc_copy, &S, NULL);
        int64_t acc[2];
        orc_parallel_for(n, 16, orc_primal, &S, acc);
        pass_out[it] = acc[0];
        faults += acc[1];
        count += 1;
        S.wold = ((double)count - 1.0) / (double)count;
        S.wnew = 1.0 / (double)count;
        orc_parallel_for(nnz, 1 << 16, orc_avg_x, &S, NULL);
        for (int64_t j = 0; j < m; ++j)
            pbar[j] = S.wold * pbar[j] + S.wnew * p[j];
    }
    *faults_out = faults;
    return count;
}

int orc_set_threads(int nthreads)
{
    if (nthreads > 0)
        g_threads = nthreads > 256 ? 256 : nthreads;
    return g_threads;
}

/* ---- setup helpers for markets numpy cannot set up in reasonable time
 * (bench.py's CPU legs at config 4, nnz ~1e9); same arithmetic as the
 * reference's numpy setup. ---- */
typedef struct {
    const int64_t *indptr;
    const double *val;
    double *out, *scales;
} orc_norm_ctx;

/* normalize (instance.py:118-138): scale_i = max_j u_ij, u_ij / scale_i */
static void orc_norm_rows(void *vc, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_norm_ctx *C = (orc_norm_ctx *)vc;
    for (int64_t i = lo; i < hi; ++i) {
        double mx = 0.0;
        for (int64_t t = C->indptr[i]; t < C->indptr[i + 1]; ++t)
            if (C->val[t] > mx)
                mx = C->val[t];
        C->scales[i] = mx;
        if (mx == 0.0)
            acc[1] += 1;
        for (int64_t t = C->indptr[i]; t < C->indptr[i + 1]; ++t)
            C->out[t] = C->val[t] / mx;
    }
}

/* returns the number of rows without a positive value (the reference raises) */
int64_t orc_normalize(int64_t n, const int64_t *indptr, const double *val, double *out,
                      double *scales)
{
    orc_norm_ctx C = {indptr, val, out, scales};
    int64_t acc[2];
    orc_parallel_for(n, 4096, orc_norm_rows, &C, acc);
    return acc[1];
}

/* Stable transpose schedule (sparse.py:130-145: argsort(col, stable)):
 * counting sort, each thread scattering a contiguous entry range after the
 * ranges before it, so equal columns keep ascending storage order. */
typedef struct {
    const int32_t *col;
    int64_t nnz, m, nparts;
    int64_t *cnt; /* nparts x m */
    int32_t *tperm;
} orc_tr_ctx;

static void orc_tr_count(void *vc, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_tr_ctx *C = (orc_tr_ctx *)vc;
    (void)acc;
    for (int64_t q = lo; q < hi; ++q) {
        int64_t a = C->nnz * q / C->nparts, b = C->nnz * (q + 1) / C->nparts;
        int64_t *c = C->cnt + q * C->m;
        for (int64_t t = a; t < b; ++t)
            c[C->col[t]]++;
    }
}

static void orc_tr_scatter(void *vc, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_tr_ctx *C = (orc_tr_ctx *)vc;
    (void)acc;
    for (int64_t q = lo; q < hi; ++q) {
        int64_t a = C->nnz * q / C->nparts, b = C->nnz * (q + 1) / C->nparts;
        int64_t *c = C->cnt + q * C->m;
        for (int64_t t = a; t < b; ++t)
            C->tperm[c[C->col[t]]++] = (int32_t)t;
    }
}

/* tperm [nnz] int32, tindptr [m+1] int64; returns -1 when scratch fails */
int orc_transpose(int64_t m, int64_t nnz, const int32_t *col, int32_t *tperm, int64_t *tindptr)
{
    int64_t nparts = g_threads * 4;
    if (nparts < 1)
        nparts = 1;
    int64_t *cnt = (int64_t *)calloc((size_t)(nparts * m), sizeof(int64_t));
    if (!cnt)
        return -1;
    orc_tr_ctx C = {col, nnz, m, nparts, cnt, tperm};
    orc_parallel_for(nparts, 1, orc_tr_count, &C, NULL);
    int64_t run = 0;
    for (int64_t j = 0; j < m; ++j) {
        tindptr[j] = run;
        for (int64_t q = 0; q < nparts; ++q) {
            int64_t c = cnt[q * m + j];
            cnt[q * m + j] = run;
            run += c;
        }
    }
    tindptr[m] = run;
    orc_parallel_for(nparts, 1, orc_tr_scatter, &C, NULL);
    free(cnt);
    return 0;
}

typedef struct {
    const int32_t *tperm;
    const int64_t *tindptr;
    const double *v;
    double *out;
} orc_cs_ctx;

static void orc_cs_cols(void *vc, int64_t lo, int64_t hi, int64_t *acc)
{
    orc_cs_ctx *C = (orc_cs_ctx *)vc;
    (void)acc;
    for (int64_t j = lo; j < hi; ++j) {
        double a = 0.0;
        for (int64_t t = C->tindptr[j]; t < C->tindptr[j + 1]; ++t)
            a += C->v[C->tperm[t]];
        C->out[j] = a;
    }
}

/* column sums in ascending storage order (np.bincount(col, weights=v)) */
void orc_colsums(int64_t m, const int32_t *tperm, const int64_t *tindptr, const double *v,
                 double *out)
{
    orc_cs_ctx C = {tperm, tindptr, v, out};
    orc_parallel_for(m, 64, orc_cs_cols, &C, NULL);
}
