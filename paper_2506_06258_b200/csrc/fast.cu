// Fast PDHCG iteration for sm_100a: exact per-buyer prox (active-set closed
// form) fused with the allocation average, deterministic column sums, and the
// price step.  One iteration = mq_dual_step + mq_primal_step + mq_colsum_step;
// all scalars (tau, sigma, navg) are device-resident so a chunk is captured
// once as a CUDA graph and replayed.
//
// Reference semantics: kernels.py:99-145 (pdhcg_chunk).  The row subproblem
// min_{x>=0} -w log(u.x) + p.x + |x - x^k|^2 / (2 tau) is solved exactly
// instead of by the reference's k-section bracket search (kernels.py:33-96):
// for a trial s, entry j is active iff c_j s + tau w u_j > 0 (c = x^k - tau p);
// on a fixed active set S the fixed point s = A_S + tau w B_S / s has the
// closed-form root; starting from any lower bound of the root, the
// re-evaluated active set can only shrink and the root only grow, so the
// iteration is monotone and ends, exactly, when the set stops changing.
#include "mq_common.cuh"

namespace mq {

constexpr int kPrimalThreads = 256;
constexpr int kMaxSweeps = 4096;

struct Avg {
    double wold, wnew;
};
__device__ __forceinline__ Avg avg_weights(const int64_t *navg, int it) {
    const int64_t count = *navg + it + 1;  // kernels.py:138-140
    Avg a;
    a.wold = ((double)count - 1.0) / (double)count;
    a.wnew = 1.0 / (double)count;
    return a;
}

// ------------------------------------------------------------ price step
__global__ void dual_kernel(int64_t m, double *__restrict__ p, double *__restrict__ pbar,
                            double *__restrict__ cs, double *__restrict__ cs_prev,
                            const double *__restrict__ steps, const int64_t *__restrict__ navg,
                            int it) {
    const double sigma = steps[1];
    const Avg w = avg_weights(navg, it);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double c = cs[j];
        const double acc = 2.0 * c - cs_prev[j];  // colsum(2 x^k - x^{k-1})
        const double pj = p[j] + sigma * (acc - 1.0);
        p[j] = pj;
        pbar[j] = w.wold * pbar[j] + w.wnew * pj;
        cs_prev[j] = c;
    }
}

// ------------------------------------------------------------ primal step
// One G-lane group per row, PER entries per lane held in registers.
template <int G, int PER>
__global__ void __launch_bounds__(kPrimalThreads)
primal_group_kernel(const mq_market mk, const mq_state st, int it,
                    double *__restrict__ x_prev_out, int64_t bin_lo, int64_t bin_hi) {
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & (G - 1);
    const int gsub = (threadIdx.x & 31) / G;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double tau = st.steps[0];
    const Avg av = avg_weights(st.navg, it);
    const double *__restrict__ U = mk.u;
    const int32_t *__restrict__ COL = mk.col;
    const double *__restrict__ P = st.p;
    double *__restrict__ X = st.x;
    double *__restrict__ XB = st.xbar;
    int64_t my_sweeps = 0;
    int my_faults = 0;

    for (int64_t base = bin_lo + warp_id * GPW; base < bin_hi; base += nwarps * GPW) {
        const int64_t r = base + gsub;
        const bool has_row = r < bin_hi;
        int64_t a = 0, b = 0;
        double tw = 0.0;
        if (has_row) {
            const int64_t i = mk.bin_rows[r];
            a = mk.row_ptr[i];
            b = mk.row_ptr[i + 1];
            tw = tau * mk.w[i];
        }
        double c[PER], u[PER];
        double s0p = 0.0, ap = 0.0, bp = 0.0;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int64_t t = a + lane + (int64_t)e * G;
            if (t < b) {
                const double ue = __ldg(U + t);
                const double xe = X[t];
                const double pe = __ldg(P + __ldg(COL + t));
                if (x_prev_out) x_prev_out[t] = xe;
                u[e] = ue;
                c[e] = xe - tau * pe;
                s0p += ue * xe;
                ap += ue * c[e];
                bp += ue * ue;
            } else {
                u[e] = 0.0;
                c[e] = 0.0;
            }
        }
        const double s0 = group_sum<G>(s0p);
        const double A = group_sum<G>(ap);
        const double B = group_sum<G>(bp);
        const int len = (int)(b - a);
        bool done = !has_row || len == 0;

        // lower bound: root with every entry active (its h(s) <= g(s))
        double s = done ? 1.0 : active_root(A, B, tw);
        int prev_cnt = len;
        int sweeps = 0;

        auto sweep = [&](double q, double &As, double &Bs, int &cnt) {
            double a_ = 0.0, b_ = 0.0;
            int k_ = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                if (fma(c[e], q, tw * u[e]) > 0.0 && u[e] > 0.0) {
                    a_ += u[e] * c[e];
                    b_ += u[e] * u[e];
                    ++k_;
                }
            }
            As = group_sum<G>(a_);
            Bs = group_sum<G>(b_);
            cnt = group_sum_int<G>(k_);
        };

        // the previous iterate's utility s0 is usually next to the root
        const bool try_s0 = !done && s0 > s;
        if (__any_sync(MQ_FULL, try_s0)) {
            double A0, B0;
            int k0;
            sweep(try_s0 ? s0 : s, A0, B0, k0);
            if (try_s0) {
                ++sweeps;
                const double g0 = A0 + tw * B0 / s0;
                if (g0 >= s0) {          // s0 below the root: step from its set
                    s = fmax(active_root(A0, B0, tw), s0);
                    prev_cnt = k0;
                } else if (g0 > s) {     // g(s0) is a lower bound above s
                    s = g0;
                    prev_cnt = -1;
                }
            }
        }
        for (int k = 0; k < kMaxSweeps; ++k) {
            if (!__any_sync(MQ_FULL, !done)) break;
            double As, Bs;
            int cnt;
            sweep(s, As, Bs, cnt);
            if (!done) {
                ++sweeps;
                if (cnt == prev_cnt || cnt == 0) {
                    done = true;  // s is the root of its own active set
                } else {
                    s = fmax(active_root(As, Bs, tw), s);
                    prev_cnt = cnt;
                }
            }
        }
        if (has_row && len > 0 && lane == 0) {
            my_sweeps += sweeps;
            if (!done) ++my_faults;
        }
        const double inv_s = 1.0 / s;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int64_t t = a + lane + (int64_t)e * G;
            if (t < b) {
                const double xn = fmax(c[e] + tw * u[e] * inv_s, 0.0);
                X[t] = xn;
                XB[t] = av.wold * XB[t] + av.wnew * xn;
            }
        }
    }
    __shared__ int64_t red[32];
    const int64_t tot = block_sum_i64(my_sweeps, red);
    if (threadIdx.x == 0 && tot) atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)tot);
    const int64_t fl = block_sum_i64((int64_t)my_faults, red);
    if (threadIdx.x == 0 && fl) atomicAdd((unsigned long long *)st.faults, (unsigned long long)fl);
}

// Long rows: one CTA per row; every sweep re-reads the row (L1/L2 resident).
__device__ __forceinline__ void block_sum3(double &a, double &b, double &c, double *sm /*[96]*/) {
    a = group_sum<32>(a);
    b = group_sum<32>(b);
    c = group_sum<32>(c);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
        sm[warp] = a;
        sm[32 + warp] = b;
        sm[64 + warp] = c;
    }
    __syncthreads();
    double ra = 0.0, rb = 0.0, rc = 0.0;
    if (lane < nw) {
        ra = sm[lane];
        rb = sm[32 + lane];
        rc = sm[64 + lane];
    }
    a = group_sum<32>(ra);
    b = group_sum<32>(rb);
    c = group_sum<32>(rc);
}

__global__ void __launch_bounds__(kPrimalThreads)
primal_long_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out,
                   int64_t bin_lo, int64_t bin_hi) {
    __shared__ double sm[96];
    const double tau = st.steps[0];
    const Avg av = avg_weights(st.navg, it);
    int64_t my_sweeps = 0;
    int my_faults = 0;
    for (int64_t r = bin_lo + blockIdx.x; r < bin_hi; r += gridDim.x) {
        const int64_t i = mk.bin_rows[r];
        const int64_t a = mk.row_ptr[i], b = mk.row_ptr[i + 1];
        const double tw = tau * mk.w[i];
        double s0 = 0.0, A = 0.0, B = 0.0;
        for (int64_t t = a + threadIdx.x; t < b; t += blockDim.x) {
            const double ue = mk.u[t], xe = st.x[t];
            const double ce = xe - tau * st.p[mk.col[t]];
            s0 += ue * xe;
            A += ue * ce;
            B += ue * ue;
        }
        block_sum3(s0, A, B, sm);
        double s = active_root(A, B, tw);
        int prev_cnt = (int)(b - a);
        int sweeps = 0;
        bool done = false;
        auto sweep = [&](double q, double &As, double &Bs, double &cnt) {
            As = 0.0;
            Bs = 0.0;
            cnt = 0.0;
            for (int64_t t = a + threadIdx.x; t < b; t += blockDim.x) {
                const double ue = mk.u[t];
                const double ce = st.x[t] - tau * st.p[mk.col[t]];
                if (fma(ce, q, tw * ue) > 0.0) {
                    As += ue * ce;
                    Bs += ue * ue;
                    cnt += 1.0;
                }
            }
            block_sum3(As, Bs, cnt, sm);
        };
        if (s0 > s) {
            double A0, B0, k0;
            sweep(s0, A0, B0, k0);
            ++sweeps;
            const double g0 = A0 + tw * B0 / s0;
            if (g0 >= s0) {
                s = fmax(active_root(A0, B0, tw), s0);
                prev_cnt = (int)k0;
            } else if (g0 > s) {
                s = g0;
                prev_cnt = -1;
            }
        }
        for (int k = 0; k < kMaxSweeps && !done; ++k) {
            double As, Bs, kc;
            sweep(s, As, Bs, kc);
            ++sweeps;
            const int cnt = (int)kc;
            if (cnt == prev_cnt || cnt == 0) {
                done = true;
            } else {
                s = fmax(active_root(As, Bs, tw), s);
                prev_cnt = cnt;
            }
        }
        if (threadIdx.x == 0) {
            my_sweeps += sweeps;
            if (!done) ++my_faults;
        }
        const double inv_s = 1.0 / s;
        __syncthreads();  // every sweep has read x before it is overwritten
        for (int64_t t = a + threadIdx.x; t < b; t += blockDim.x) {
            const double xe = st.x[t];
            if (x_prev_out) x_prev_out[t] = xe;
            const double xn = fmax(xe - tau * st.p[mk.col[t]] + tw * mk.u[t] * inv_s, 0.0);
            st.x[t] = xn;
            st.xbar[t] = av.wold * st.xbar[t] + av.wnew * xn;
        }
        __syncthreads();
    }
    __shared__ int64_t red[32];
    const int64_t tot = block_sum_i64(my_sweeps, red);
    if (threadIdx.x == 0 && tot) atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)tot);
    const int64_t fl = block_sum_i64((int64_t)my_faults, red);
    if (threadIdx.x == 0 && fl) atomicAdd((unsigned long long *)st.faults, (unsigned long long)fl);
}

// ------------------------------------------------------------ column sums
// One warp per good, lanes stride the good's entries in transpose-schedule
// order, four independent gathers in flight per lane, fixed butterfly tree.
__global__ void __launch_bounds__(256)
colsum_kernel(int64_t m, const int64_t *__restrict__ tptr, const int32_t *__restrict__ tperm,
              const double *__restrict__ v, double *__restrict__ out, double *__restrict__ csbar,
              const int64_t *__restrict__ navg, int it) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    Avg av = {0.0, 0.0};
    if (csbar) av = avg_weights(navg, it);
    for (int64_t j = warp_id; j < m; j += nwarps) {
        const int64_t beg = tptr[j], end = tptr[j + 1];
        double acc = 0.0;
        int64_t t = beg + lane;
        for (; t + 96 < end; t += 128) {
            const int32_t k0 = __ldg(tperm + t), k1 = __ldg(tperm + t + 32);
            const int32_t k2 = __ldg(tperm + t + 64), k3 = __ldg(tperm + t + 96);
            const double v0 = v[k0], v1 = v[k1], v2 = v[k2], v3 = v[k3];
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; t < end; t += 32) acc += v[__ldg(tperm + t)];
        acc = group_sum<32>(acc);
        if (lane == 0) {
            out[j] = acc;
            if (csbar) csbar[j] = av.wold * csbar[j] + av.wnew * acc;
        }
    }
}

__global__ void colsum_finalize_kernel(int64_t m, const double *__restrict__ cs,
                                       double *__restrict__ csbar, const int64_t *__restrict__ navg,
                                       int it) {
    const Avg av = avg_weights(navg, it);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        csbar[j] = av.wold * csbar[j] + av.wnew * cs[j];
}

__global__ void chunk_end_kernel(int64_t *navg, int iters) { *navg += iters; }

// ------------------------------------------------------------ launchers
static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int G, int PER>
static void launch_group(const mq_market &mk, const mq_state &st, int it, double *xprev,
                         int64_t lo, int64_t hi, cudaStream_t s) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return;
    const int per_block = kPrimalThreads / G;
    const int grid = grid_for(rows, per_block, sm_count() * 16);
    primal_group_kernel<G, PER><<<grid, kPrimalThreads, 0, s>>>(mk, st, it, xprev, lo, hi);
}

int primal_launch(const mq_market *mk, const mq_state *st, int it, double *xprev, cudaStream_t s) {
    const int64_t *o = mk->bin_off;
    launch_group<4, 1>(*mk, *st, it, xprev, o[0], o[1], s);    // len <= 4
    launch_group<8, 1>(*mk, *st, it, xprev, o[1], o[2], s);    // <= 8
    launch_group<16, 1>(*mk, *st, it, xprev, o[2], o[3], s);   // <= 16
    launch_group<32, 1>(*mk, *st, it, xprev, o[3], o[4], s);   // <= 32
    launch_group<32, 2>(*mk, *st, it, xprev, o[4], o[5], s);   // <= 64
    launch_group<32, 4>(*mk, *st, it, xprev, o[5], o[6], s);   // <= 128
    launch_group<32, 8>(*mk, *st, it, xprev, o[6], o[7], s);   // <= 256
    launch_group<32, 16>(*mk, *st, it, xprev, o[7], o[8], s);  // <= 512
    const int64_t nlong = o[9] - o[8];
    if (nlong > 0) {
        const int grid = grid_for(nlong, 1, sm_count() * 8);
        primal_long_kernel<<<grid, kPrimalThreads, 0, s>>>(*mk, *st, it, xprev, o[8], o[9]);
    }
    return check_launch("mq_primal_step");
}

int colsum_launch(const mq_market *mk, const double *v, double *out, double *csbar,
                  const int64_t *navg, int it, cudaStream_t s) {
    const int grid = grid_for(mk->m, 8, sm_count() * 32);
    colsum_kernel<<<grid, 256, 0, s>>>(mk->m, mk->tptr, mk->tperm, v, out, csbar, navg, it);
    return check_launch("colsum");
}

int dual_launch(const mq_market *mk, const mq_state *st, int it, cudaStream_t s) {
    const int grid = grid_for(mk->m, 256, sm_count() * 8);
    dual_kernel<<<grid, 256, 0, s>>>(mk->m, st->p, st->pbar, st->cs, st->cs_prev, st->steps,
                                     st->navg, it);
    return check_launch("mq_dual_step");
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_dual_step(const mq_market *mk, const mq_state *st, int it, void *stream) {
    return dual_launch(mk, st, it, (cudaStream_t)stream);
}

int mq_primal_step(const mq_market *mk, const mq_state *st, int it, double *x_prev_out,
                   void *stream) {
    return primal_launch(mk, st, it, x_prev_out, (cudaStream_t)stream);
}

int mq_colsum_step(const mq_market *mk, const mq_state *st, int it, int finalize, void *stream) {
    return colsum_launch(mk, st->x, st->cs, finalize ? st->csbar : nullptr, st->navg, it,
                         (cudaStream_t)stream);
}

int mq_colsum_finalize(const mq_market *mk, const mq_state *st, int it, void *stream) {
    const int grid = grid_for(mk->m, 256, sm_count() * 8);
    colsum_finalize_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(mk->m, st->cs, st->csbar,
                                                                   st->navg, it);
    return check_launch("mq_colsum_finalize");
}

int mq_chunk_end(const mq_state *st, int iters, void *stream) {
    chunk_end_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(st->navg, iters);
    return check_launch("mq_chunk_end");
}

int mq_fast_chunk(const mq_market *mk, const mq_state *st, int iters, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    for (int it = 0; it < iters; ++it) {
        if ((rc = dual_launch(mk, st, it, s))) return rc;
        if ((rc = primal_launch(mk, st, it, nullptr, s))) return rc;
        if ((rc = colsum_launch(mk, st->x, st->cs, st->csbar, st->navg, it, s))) return rc;
    }
    return mq_chunk_end(st, iters, stream);
}

int mq_colsum(const mq_market *mk, const double *v, double *out, void *stream) {
    return colsum_launch(mk, v, out, nullptr, nullptr, 0, (cudaStream_t)stream);
}

}  // extern "C"
