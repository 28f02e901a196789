// Restarted lifted PDHG (algo="pdhg"): kernels.py:146-197 (pdhg_chunk) with
// the state plumbing of driver.py:184-268 (_LiftedRun), on device.
//
// One iteration = the price step (dual_kernel of fast.cu: p += sigma (2 cs -
// cs_prev - 1), p averaged) + pdhg_rows_kernel (per buyer: y and t updates,
// the entry-wise x update, the averages) + the fixed-point column sums of the
// new x (shared with the PDHCG path).  The reference's row sums of
// u (2x - x_prev) are carried as ru = u.x^k and ru_prev = u.x^{k-1}, so x_prev
// is never stored; every sum is deterministic (fixed-order or integer).
#include "mq_common.cuh"

namespace mq {

int launch_dual(const mq_market *mk, double *p, double *pbar, double *cs, double *cs_prev,
                const double *steps, const int64_t *navg, int it, cudaStream_t s,
                double *drift = nullptr);                                           // fast.cu
int launch_cs_from_fixed(const mq_market *mk, unsigned long long *fix, double *cs, double *csbar,
                         const int64_t *navg, int it, cudaStream_t s,
                         double *drift = nullptr);                                  // fast.cu
int sm_count_reduce();                                                              // reduce.cu

namespace {

struct AvgW {
    double wold, wnew;
};
__device__ __forceinline__ AvgW avg_w(const int64_t *navg, int it) {
    const int64_t count = *navg + it + 1;  // kernels.py:190-192
    return {((double)count - 1.0) / (double)count, 1.0 / (double)count};
}

__device__ __forceinline__ void fix_add(const mq_market &mk, unsigned long long *fix, int64_t *faults,
                                        int j, double xe) {
    if (xe < mk.cs_xmax)
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(fix + j), "l"(__double2ull_rn(xe * mk.cs_scale))
                     : "memory");
    else
        atomicAdd(reinterpret_cast<unsigned long long *>(faults), 1ull);
}

// ---------------------------------------------------------------- iteration
__global__ void __launch_bounds__(256)
pdhg_rows_kernel(const mq_market mk, const mq_lstate ls, int it) {
    const double tau = ls.steps[0], sigma = ls.steps[1];
    const AvgW av = avg_w(ls.navg, it);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < mk.n; i += nw) {
        const int64_t a = mk.row_ptr[i], b = mk.row_ptr[i + 1];
        const double ti = ls.t[i], tp = ls.t_prev[i];
        // y += sigma ((2 t - t_prev) - u.(2 x - x_prev))          (kernels.py:164-168)
        const double yi = ls.y[i] + sigma * ((2.0 * ti - tp) - (2.0 * ls.ru[i] - ls.ru_prev[i]));
        // t: positive root of t^2 + (tau y - t_k) t - tau w = 0   (kernels.py:173-181)
        const double wi = mk.w[i];
        const double d = tau * yi - ti;
        const double root = sqrt(d * d + 4.0 * tau * wi);
        const double tn = d > 0.0 ? 2.0 * tau * wi / (d + root) : 0.5 * (root - d);
        double acc = 0.0;
        // restrict-qualified views: loads of later entries may be issued
        // before the stores of earlier ones (no aliasing between the arrays)
        double *__restrict__ X = ls.x;
        double *__restrict__ XB = ls.xbar;
        const double *__restrict__ P = ls.p;
        const double *__restrict__ U = mk.u;
        const int32_t *__restrict__ C = mk.col;
#pragma unroll 4
        for (int64_t e = a + lane; e < b; e += 32) {  // kernels.py:182-185
            const int j = C[e];
            const double ue = U[e];
            const double xv = X[e] - tau * (__ldg(P + j) - ue * yi);
            const double xn = xv > 0.0 ? xv : 0.0;
            X[e] = xn;
            XB[e] = av.wold * XB[e] + av.wnew * xn;
            acc += ue * xn;
            if (xn > 0.0) fix_add(mk, ls.fix, ls.faults, j, xn);
        }
        acc = group_sum<32>(acc);
        if (lane == 0) {
            ls.y[i] = yi;
            ls.t_prev[i] = ti;
            ls.t[i] = tn;
            ls.ru_prev[i] = ls.ru[i];
            ls.ru[i] = acc;
            ls.tbar[i] = av.wold * ls.tbar[i] + av.wnew * tn;
            ls.ybar[i] = av.wold * ls.ybar[i] + av.wnew * yi;
        }
    }
}

__global__ void navg_add_kernel(int64_t *navg, int iters) { *navg += iters; }

// out_i = u_i . x_i (normalized or original utilities), one warp per row
__global__ void __launch_bounds__(256)
row_dot_kernel(const mq_market mk, const double *__restrict__ x, int use_norm,
               double *__restrict__ out) {
    const double *__restrict__ U = use_norm ? mk.u : mk.u_orig;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < mk.n; i += nw) {
        double acc = 0.0;
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) acc += U[e] * x[e];
        acc = group_sum<32>(acc);
        if (lane == 0) out[i] = acc;
    }
}

// ---------------------------------------------------------------- residuals
// order-preserving u64 key of a double (signed max with integer atomics)
__device__ __forceinline__ unsigned long long okey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

constexpr int kRows = 8 * MQ_MAX_BLOCKS;  // misc words after the partial slots

// kkt.py:29-76 row / entry part of residuals_lifted, for (x, t*s, p, y/s)
// with s = row scales (use_norm = 0: original instance) or s = 1 (the
// normalized instance of the omega_0 norms, driver.py:222-232)
__global__ void __launch_bounds__(256)
resid_lifted_rows_kernel(const mq_market mk, const double *__restrict__ scales,
                         const double *__restrict__ x, const double *__restrict__ t,
                         const double *__restrict__ y, const double *__restrict__ p, int use_norm,
                         unsigned long long *__restrict__ colkey, double *__restrict__ scratch) {
    const double *__restrict__ U = use_norm ? mk.u : mk.u_orig;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double *misc = scratch + kRows;
    double rgmax = 0.0, wtmax = 0.0, ymax = 0.0, dtmax = 0.0, gmax = 0.0, xmax = 0.0, emax = 0.0;
    double nbad = 0.0, s_rg = 0.0, s_dt = 0.0;
    for (int64_t i = w0; i < mk.n; i += nw) {
        const double sc = use_norm ? 1.0 : scales[i];
        const double to = t[i] * sc, yo = y[i] / sc;
        double ux = 0.0;
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) ux += U[e] * x[e];
        ux = group_sum<32>(ux);
        if (lane == 0) {
            const double rg = to - ux;
            rgmax = fmax(rgmax, fabs(rg));
            s_rg += rg * rg;
            ymax = fmax(ymax, fabs(yo));
            if (!(to > 0.0)) {
                nbad += 1.0;
            } else {
                const double wt = mk.w[i] / to;
                wtmax = fmax(wtmax, fabs(wt));
                dtmax = fmax(dtmax, fabs(wt - yo));
                s_dt += (wt - yo) * (wt - yo);
            }
        }
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) {
            const int j = mk.col[e];
            const double uy = U[e] * yo;
            const unsigned long long kk = okey(uy);
            if (kk > __ldcg(colkey + j)) atomicMax(colkey + j, kk);  // skip covered values
            const double es = fmax(p[j] - uy, 0.0);
            const double xv = x[e];
            gmax = fmax(gmax, xv * es);
            xmax = fmax(xmax, fabs(xv));
            emax = fmax(emax, es);
        }
    }
    gmax = group_max<32>(gmax);
    xmax = group_max<32>(xmax);
    emax = group_max<32>(emax);
    if (lane == 0) {
        atomic_max_nonneg(misc + 0, rgmax);
        atomic_max_nonneg(misc + 1, wtmax);
        atomic_max_nonneg(misc + 2, ymax);
        atomic_max_nonneg(misc + 3, dtmax);
        atomic_max_nonneg(misc + 4, gmax);
        atomic_max_nonneg(misc + 5, xmax);
        atomic_max_nonneg(misc + 6, emax);
    }
    __shared__ double sm[32];
    const double b0 = block_sum(nbad, sm);
    const double b1 = block_sum(s_rg, sm);
    const double b2 = block_sum(s_dt, sm);
    if (threadIdx.x == 0) {
        scratch[0 * MQ_MAX_BLOCKS + blockIdx.x] = b0;
        scratch[1 * MQ_MAX_BLOCKS + blockIdx.x] = b1;
        scratch[2 * MQ_MAX_BLOCKS + blockIdx.x] = b2;
    }
}

// fixed-order sum of the first `nslots` partial slots -> out[s]
__global__ void slots_sum_kernel(const double *__restrict__ partials, int nblocks, int nslots,
                                 double *__restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < nslots; s += blockDim.x >> 5) {
        double acc = 0.0;
        for (int b = lane; b < nblocks; b += 32) acc += partials[s * MQ_MAX_BLOCKS + b];
        acc = group_sum<32>(acc);
        if (lane == 0) out[s] = acc;
    }
}

__global__ void resid_lifted_finish(const double *__restrict__ scratch, const double *__restrict__ sums,
                                    double *__restrict__ row_out) {
    const double *misc = scratch + kRows;
    for (int k = 0; k < 7; ++k) row_out[k] = misc[k];
    row_out[7] = sums[0];
    row_out[8] = sums[1];
    row_out[9] = sums[2];
}

__global__ void colkey_decode_kernel(int64_t m, unsigned long long *__restrict__ key) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double v = key[j] ? okey_inv(key[j]) : -INFINITY;
        reinterpret_cast<double *>(key)[j] = v;
    }
}

// restart moves, row part (driver.py:242-252): sums of dt^2, dy^2 and
// (dt - u.dx) dy over this shard (u normalized)
__global__ void __launch_bounds__(256)
moves_lifted_kernel(const mq_market mk, const double *__restrict__ xbar,
                    const double *__restrict__ x0, const double *__restrict__ tbar,
                    const double *__restrict__ t0, const double *__restrict__ ybar,
                    const double *__restrict__ y0, double *__restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t i = w0; i < mk.n; i += nw) {
        double udx = 0.0;
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32)
            udx += mk.u[e] * (xbar[e] - x0[e]);
        udx = group_sum<32>(udx);
        if (lane == 0) {
            const double dt = tbar[i] - t0[i], dy = ybar[i] - y0[i];
            a += dt * dt;
            b += dy * dy;
            c += (dt - udx) * dy;
        }
    }
    __shared__ double sm[32];
    const double ra = block_sum(a, sm);
    const double rb = block_sum(b, sm);
    const double rc = block_sum(c, sm);
    if (threadIdx.x == 0) {
        scratch[0 * MQ_MAX_BLOCKS + blockIdx.x] = ra;
        scratch[1 * MQ_MAX_BLOCKS + blockIdx.x] = rb;
        scratch[2 * MQ_MAX_BLOCKS + blockIdx.x] = rc;
    }
}

// lifted operator power step (pdhg.py:157-161): out_y = vt - u.vx per row,
// back_x = out_p[col] - u out_y[row]; partial sums of back_x^2 and out_y^2
__global__ void __launch_bounds__(256)
opnorm_rows_kernel(const mq_market mk, const double *__restrict__ vx, const double *__restrict__ vt,
                   const double *__restrict__ out_p, double *__restrict__ out_y,
                   double *__restrict__ wx, double *__restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sx = 0.0, sy = 0.0;
    for (int64_t i = w0; i < mk.n; i += nw) {
        double uv = 0.0;
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) uv += mk.u[e] * vx[e];
        uv = group_sum<32>(uv);
        const double oy = vt[i] - uv;
        if (lane == 0) {
            out_y[i] = oy;
            sy += oy * oy;
        }
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) {
            const double bx = out_p[mk.col[e]] - mk.u[e] * oy;
            wx[e] = bx;
            sx += bx * bx;
        }
    }
    __shared__ double sm[32];
    const double rx = block_sum(sx, sm);
    const double ry = block_sum(sy, sm);
    if (threadIdx.x == 0) {
        scratch[0 * MQ_MAX_BLOCKS + blockIdx.x] = rx;
        scratch[1 * MQ_MAX_BLOCKS + blockIdx.x] = ry;
    }
}

int row_grid(int64_t n) { return grid_for(n, 8, MQ_MAX_BLOCKS); }  // <= MQ_MAX_BLOCKS partials

}  // namespace
}  // namespace mq

using namespace mq;

extern "C" {

int mq_pdhg_step(const mq_market *mk, const mq_lstate *ls, int it, void *stream) {
    if (!mk || !ls) return set_error(cudaErrorInvalidValue, "mq_pdhg_step: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_dual(mk, ls->p, ls->pbar, ls->cs, ls->cs_prev, ls->steps, ls->navg, it, s);
    if (rc) return rc;
    if (mk->n > 0)
        pdhg_rows_kernel<<<grid_for(mk->n, 8, sm_count_reduce() * 16), 256, 0, s>>>(*mk, *ls, it);
    if ((rc = check_launch("mq_pdhg_step"))) return rc;
    return launch_cs_from_fixed(mk, ls->fix, ls->cs, ls->csbar, ls->navg, it, s);
}

int mq_pdhg_colsum_only(const mq_market *mk, const mq_lstate *ls, int it, void *stream) {
    // N ranks: the primal part without the conversion (the host all-reduces
    // the integer sums first, then calls mq_pdhg_finish_colsum)
    if (!mk || !ls) return set_error(cudaErrorInvalidValue, "mq_pdhg_colsum_only: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_dual(mk, ls->p, ls->pbar, ls->cs, ls->cs_prev, ls->steps, ls->navg, it, s);
    if (rc) return rc;
    if (mk->n > 0)
        pdhg_rows_kernel<<<grid_for(mk->n, 8, sm_count_reduce() * 16), 256, 0, s>>>(*mk, *ls, it);
    return check_launch("mq_pdhg_colsum_only");
}

int mq_pdhg_finish_colsum(const mq_market *mk, const mq_lstate *ls, int it, void *stream) {
    if (!mk || !ls) return set_error(cudaErrorInvalidValue, "mq_pdhg_finish_colsum: null argument");
    return launch_cs_from_fixed(mk, ls->fix, ls->cs, ls->csbar, ls->navg, it, (cudaStream_t)stream);
}

int mq_pdhg_chunk_end(const mq_lstate *ls, int iters, void *stream) {
    if (!ls) return set_error(cudaErrorInvalidValue, "mq_pdhg_chunk_end: null argument");
    navg_add_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(ls->navg, iters);
    return check_launch("mq_pdhg_chunk_end");
}

int mq_row_dot(const mq_market *mk, const double *x, int use_norm, double *out, void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_row_dot: null argument");
    if (mk->n > 0)
        row_dot_kernel<<<grid_for(mk->n, 8, sm_count_reduce() * 16), 256, 0, (cudaStream_t)stream>>>(
            *mk, x, use_norm, out);
    return check_launch("mq_row_dot");
}

int mq_pdhg_resid_rows(const mq_market *mk, const double *scales, const double *x, const double *t,
                       const double *y, const double *p, int use_norm, double *colbest,
                       double *row_out, double *scratch, void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_pdhg_resid_rows: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = row_grid(mk->n);
    cudaMemsetAsync(scratch + kRows, 0, 8 * sizeof(double), s);
    cudaMemsetAsync(colbest, 0, (size_t)mk->m * sizeof(double), s);
    resid_lifted_rows_kernel<<<grid, 256, 0, s>>>(*mk, scales, x, t, y, p, use_norm,
                                                  reinterpret_cast<unsigned long long *>(colbest),
                                                  scratch);
    slots_sum_kernel<<<1, 96, 0, s>>>(scratch, grid, 3, scratch + kRows + 16);
    resid_lifted_finish<<<1, 1, 0, s>>>(scratch, scratch + kRows + 16, row_out);
    colkey_decode_kernel<<<grid_for(mk->m, 256, 1024), 256, 0, s>>>(
        mk->m, reinterpret_cast<unsigned long long *>(colbest));
    return check_launch("mq_pdhg_resid_rows");
}

int mq_pdhg_moves(const mq_market *mk, const double *xbar, const double *x0, const double *tbar,
                  const double *t0, const double *ybar, const double *y0, double *out,
                  double *scratch, void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_pdhg_moves: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = row_grid(mk->n);
    moves_lifted_kernel<<<grid, 256, 0, s>>>(*mk, xbar, x0, tbar, t0, ybar, y0, scratch);
    slots_sum_kernel<<<1, 96, 0, s>>>(scratch, grid, 3, out);
    return check_launch("mq_pdhg_moves");
}

int mq_pdhg_opnorm_step(const mq_market *mk, const double *vx, const double *vt, const double *out_p,
                        double *out_y, double *wx, double *sums, double *scratch, void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_pdhg_opnorm_step: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = row_grid(mk->n);
    opnorm_rows_kernel<<<grid, 256, 0, s>>>(*mk, vx, vt, out_p, out_y, wx, scratch);
    slots_sum_kernel<<<1, 64, 0, s>>>(scratch, grid, 2, sums);
    return check_launch("mq_pdhg_opnorm_step");
}

}  // extern "C"
