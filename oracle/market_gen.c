/*
 * CPU restatement of the device market generator — TEST INFRASTRUCTURE.
 *
 * Regenerates, on the host, byte for byte the synthetic markets that
 * paper_2506_06258_b200/csrc/generate.cu builds on the GPU (BASELINE configs
 * 3-5; the reference's own generator, instance.py:141-226, draws n*m host
 * uniforms and cannot reach them).  Used so that the CPU reference arm of
 * bench.py and the parity tests build their instance without the product's
 * CUDA library.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * load it.
 *
 * What must match the device exactly:
 *  - cuRAND's Philox4x32-10 (curand_init(seed, subsequence, 0) and
 *    curand_uniform_double = (x + 1) 2^-32 of the next 32-bit output),
 *    restated from its published algorithm (Salmon et al., "Parallel random
 *    numbers: as easy as 1, 2, 3", SC'11; cuRAND's counter/key layout);
 *  - the generator's log / exp, which both sides build from correctly
 *    rounded IEEE operations only (compile with -ffp-contract=off; fma() is
 *    the correctly rounded C99 fma).
 * Rows are independent (one Philox subsequence each), so any row range can be
 * produced on a pthread team, results independent of the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

/* ------------------------------------------------------------ Philox4x32-10 */
typedef struct {
    uint32_t ctr[4], out[4], key[2];
    int state;
} philox_t;

static void philox10(const uint32_t cin[4], const uint32_t kin[2], uint32_t o[4])
{
    uint32_t c0 = cin[0], c1 = cin[1], c2 = cin[2], c3 = cin[3];
    uint32_t k0 = kin[0], k1 = kin[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (r < 9) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
    }
    o[0] = c0; o[1] = c1; o[2] = c2; o[3] = c3;
}

/* curand_init(seed, subsequence, offset 0): counter (0, 0, lo, hi) */
static void ph_init(philox_t *s, uint64_t seed, uint64_t subseq)
{
    s->ctr[0] = s->ctr[1] = 0;
    s->ctr[2] = (uint32_t)subseq;
    s->ctr[3] = (uint32_t)(subseq >> 32);
    s->key[0] = (uint32_t)seed;
    s->key[1] = (uint32_t)(seed >> 32);
    s->state = 0;
    philox10(s->ctr, s->key, s->out);
}

static uint32_t ph_next(philox_t *s)
{
    const uint32_t r = s->out[s->state++];
    if (s->state == 4) {
        if (++s->ctr[0] == 0 && ++s->ctr[1] == 0 && ++s->ctr[2] == 0) ++s->ctr[3];
        philox10(s->ctr, s->key, s->out);
        s->state = 0;
    }
    return r;
}

/* (0, 1]: (x + 1) / 2^32, exact */
static double ph_uniform(philox_t *s) { return ((double)ph_next(s) + 1.0) * 2.3283064365386963e-10; }

/* ------------------------------------------------------------ log / exp */
static const double LN2_HI = 6.93147180369123816490e-01;
static const double LN2_LO = 1.90821492927058770002e-10;
static const double INV_LN2 = 1.4426950408889634;

static double gm_log(double x)
{
    int e;
    double m = frexp(x, &e);
    if (m < 0.70710678118654752440) {
        m = m * 2.0;
        e -= 1;
    }
    const double f = m - 1.0;
    const double s = f / (2.0 + f);
    const double z = s * s;
    static const double c[11] = {0.043478260869565216, 0.047619047619047616, 0.05263157894736842,
                                 0.058823529411764705, 0.06666666666666667, 0.07692307692307693,
                                 0.09090909090909091,  0.1111111111111111,  0.14285714285714285,
                                 0.2,                  0.3333333333333333};
    double r = c[0];
    for (int k = 1; k < 11; ++k) r = fma(r, z, c[k]);
    const double t = (s * z) * r;
    const double lm = 2.0 * (s + t);
    const double de = (double)e;
    return de * LN2_HI + (de * LN2_LO + lm);
}

static double gm_exp(double y)
{
    const double n = floor(y * INV_LN2 + 0.5);
    double r = y - n * LN2_HI;
    r = r - n * LN2_LO;
    static const double c[12] = {2.08767569878681e-09,  2.505210838544172e-08,
                                 2.755731922398589e-07, 2.7557319223985893e-06,
                                 2.48015873015873e-05,  0.0001984126984126984,
                                 0.001388888888888889,  0.008333333333333333,
                                 0.041666666666666664,  0.16666666666666666,
                                 0.5,                   1.0};
    double p = 1.6059043836821613e-10;
    for (int k = 0; k < 12; ++k) p = fma(p, r, c[k]);
    p = fma(p, r, 1.0);
    return ldexp(p, (int)n);
}

/* ------------------------------------------------------------ rows */
typedef struct {
    int64_t m;
    double q, alpha, dmin;
    int q_mode;
    uint64_t seed;
} gen_t;

static double row_rate(const gen_t *g, int64_t row)
{
    if (g->q_mode == 0) return g->q;
    philox_t st;
    ph_init(&st, g->seed ^ 0x9e3779b97f4a7c15ull, (uint64_t)row);
    const double u = ph_uniform(&st);
    const double k = -1.0 / (g->alpha - 1.0);
    double d = g->dmin * gm_exp(k * gm_log(u));
    if (d > (double)g->m) d = (double)g->m;
    return d / (double)g->m;
}

/* the support of one row, ascending (cols may be NULL: count only) */
static int64_t walk_row(const gen_t *g, int64_t row, int32_t *cols)
{
    const double q = row_rate(g, row);
    philox_t st;
    ph_init(&st, g->seed, (uint64_t)row);
    int64_t cnt = 0;
    if (q >= 1.0) {
        if (cols)
            for (int64_t j = 0; j < g->m; ++j) cols[j] = (int32_t)j;
        return g->m;
    }
    const double lq = gm_log(1.0 - q);
    int64_t pos = -1;
    for (;;) {
        const double u = ph_uniform(&st);
        const double skip = floor(gm_log(u) / lq);
        if (skip >= (double)(g->m - 1 - pos)) break;
        pos += (int64_t)skip + 1;
        if (cols) cols[cnt] = (int32_t)pos;
        ++cnt;
    }
    if (cnt == 0) {
        int64_t j = (int64_t)(ph_uniform(&st) * (double)g->m);
        if (j >= g->m) j = g->m - 1;
        if (cols) cols[0] = (int32_t)j;
        cnt = 1;
    }
    return cnt;
}

typedef struct {
    const gen_t *g;
    int64_t row0, lo, hi;
    int64_t *deg;
    const int64_t *row_ptr;
    int32_t *col;
    double *val, *w;
} task_t;

static void *deg_worker(void *arg)
{
    task_t *t = (task_t *)arg;
    for (int64_t r = t->lo; r < t->hi; ++r) t->deg[r] = walk_row(t->g, t->row0 + r, NULL);
    return NULL;
}

static void *fill_worker(void *arg)
{
    task_t *t = (task_t *)arg;
    for (int64_t r = t->lo; r < t->hi; ++r) {
        const int64_t row = t->row0 + r;
        const int64_t a = t->row_ptr[r];
        const int64_t k = walk_row(t->g, row, t->col + a);
        philox_t vs;
        ph_init(&vs, t->g->seed + 0x5851f42d4c957f2dull, (uint64_t)row);
        for (int64_t e = 0; e < k; ++e) t->val[a + e] = ph_uniform(&vs);
        if (t->w) {
            philox_t ws;
            ph_init(&ws, t->g->seed + 0x14057b7ef767814full, (uint64_t)row);
            t->w[r] = ph_uniform(&ws);
        }
    }
    return NULL;
}

static void run_team(task_t *proto, int64_t nrows, int threads, void *(*fn)(void *))
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    task_t tk[256];
    /* interleaved blocks of rows keep power-law rows balanced */
    const int64_t per = (nrows + threads - 1) / threads;
    for (int i = 0; i < threads; ++i) {
        tk[i] = *proto;
        tk[i].lo = i * per < nrows ? i * per : nrows;
        tk[i].hi = (i + 1) * per < nrows ? (i + 1) * per : nrows;
        pthread_create(&th[i], NULL, fn, &tk[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
}

int orc_gen_degrees(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                    double dmin, uint64_t seed, int64_t *deg, int threads)
{
    gen_t g = {m, q, alpha, dmin, q_mode, seed};
    task_t t = {&g, row0, 0, 0, deg, NULL, NULL, NULL, NULL};
    run_team(&t, nrows, threads, deg_worker);
    return 0;
}

int orc_gen_fill(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                 double dmin, uint64_t seed, const int64_t *row_ptr, int32_t *col, double *val,
                 double *w, int threads)
{
    gen_t g = {m, q, alpha, dmin, q_mode, seed};
    task_t t = {&g, row0, 0, 0, NULL, row_ptr, col, val, w};
    run_team(&t, nrows, threads, fill_worker);
    return 0;
}

/* the device gm_log / gm_exp restated, for the known-answer test */
double orc_gm_log(double x) { return gm_log(x); }
double orc_gm_exp(double y) { return gm_exp(y); }
