// Device instance generator for markets the reference's O(n*m) host generator
// cannot reach (BASELINE configs 3-5; instance.py:141-226 semantics):
// every buyer row draws a Bernoulli(q_i) support over the m goods by
// geometric skipping, values U(0,1], budgets U(0,1].  q_i = q (uniform
// markets) or d_i / m with a truncated power-law degree d_i (skewed markets).
// Each row owns a Philox subsequence, so a row's content does not depend on
// the launch configuration or on how rows are split across GPUs: rank r can
// generate exactly its shard.  The transcendentals are the bit-specified
// gm_log / gm_exp (mq_genmath.cuh), so oracle/market_gen.c regenerates any
// market byte for byte on the host (the reference arm's instance, tests).
#include <curand_kernel.h>

#include "mq_common.cuh"
#include "mq_genmath.cuh"

namespace mq {

struct GenParams {
    int64_t m;
    double q;          // Bernoulli rate (q_mode 0)
    double alpha;      // power-law exponent (q_mode 1): d = dmin * U^(-1/(alpha-1))
    double dmin;
    int q_mode;
    unsigned long long seed;
};

__device__ __forceinline__ double row_rate(const GenParams &g, int64_t row) {
    if (g.q_mode == 0) return g.q;
    curandStatePhilox4_32_10_t st;
    curand_init(g.seed ^ 0x9e3779b97f4a7c15ull, (unsigned long long)row, 0, &st);
    const double u = curand_uniform_double(&st);  // (0, 1]
    const double k = -1.0 / (g.alpha - 1.0);
    double d = __dmul_rn(g.dmin, gm_exp(__dmul_rn(k, gm_log(u))));
    if (d > (double)g.m) d = (double)g.m;
    return d / (double)g.m;
}

// Walks row `row`'s support; emit(j) for every selected column (ascending).
// Returns the count; an empty draw is repaired with one uniform column.
template <typename Emit>
__device__ int64_t walk_row(const GenParams &g, int64_t row, Emit emit) {
    const double q = row_rate(g, row);
    curandStatePhilox4_32_10_t st;
    curand_init(g.seed, (unsigned long long)row, 0, &st);
    int64_t cnt = 0;
    if (q >= 1.0) {
        for (int64_t j = 0; j < g.m; ++j) emit(j);
        return g.m;
    }
    const double lq = gm_log(__dadd_rn(1.0, -q));
    int64_t pos = -1;
    for (;;) {
        const double u = curand_uniform_double(&st);
        const double skip = floor(__ddiv_rn(gm_log(u), lq));
        if (skip >= (double)(g.m - 1 - pos)) break;
        pos += (int64_t)skip + 1;
        emit(pos);
        ++cnt;
    }
    if (cnt == 0) {  // repair: one uniformly placed entry (instance.py:165-194)
        int64_t j = (int64_t)__dmul_rn(curand_uniform_double(&st), (double)g.m);
        if (j >= g.m) j = g.m - 1;
        emit(j);
        cnt = 1;
    }
    return cnt;
}

__global__ void gen_degrees_kernel(GenParams g, int64_t row0, int64_t nrows, int64_t *deg) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x)
        deg[r] = walk_row(g, row0 + r, [](int64_t) {});
}

__global__ void gen_fill_kernel(GenParams g, int64_t row0, int64_t nrows,
                                const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col,
                                double *__restrict__ val, double *__restrict__ w) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + r;
        int32_t *c = col + row_ptr[r];
        int64_t k = 0;
        walk_row(g, row, [&](int64_t j) { c[k++] = (int32_t)j; });
        curandStatePhilox4_32_10_t vs;
        curand_init(g.seed + 0x5851f42d4c957f2dull, (unsigned long long)row, 0, &vs);
        double *v = val + row_ptr[r];
        for (int64_t t = 0; t < k; ++t) v[t] = curand_uniform_double(&vs);
        if (w) {
            curandStatePhilox4_32_10_t ws;
            curand_init(g.seed + 0x14057b7ef767814full, (unsigned long long)row, 0, &ws);
            w[r] = curand_uniform_double(&ws);
        }
    }
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_gen_degrees(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                   double dmin, unsigned long long seed, int64_t *deg, void *stream) {
    GenParams g{m, q, alpha, dmin, q_mode, seed};
    const int grid = grid_for(nrows, 128, 148 * 64);
    gen_degrees_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(g, row0, nrows, deg);
    return check_launch("mq_gen_degrees");
}

int mq_gen_fill(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                double dmin, unsigned long long seed, const int64_t *row_ptr, int32_t *col,
                double *val, double *w, void *stream) {
    GenParams g{m, q, alpha, dmin, q_mode, seed};
    const int grid = grid_for(nrows, 128, 148 * 64);
    gen_fill_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(g, row0, nrows, row_ptr, col, val, w);
    return check_launch("mq_gen_fill");
}

}  // extern "C"
