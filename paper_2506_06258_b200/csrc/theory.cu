// Theory diagnostics on the device (kkt.py:88-168): the scaled KKT residual
// and the smoothed duality gap, whose allocation part is row-separable and
// solved by the exact row prox with step 1/xi (the same monotone active-set
// iteration as the PDHCG kernels, here a warp per row with c kept in a
// global scratch array).  Sums are deterministic (fixed-size block partials,
// fixed-order final pass); maxima are not needed.
#include "mq_common.cuh"

namespace mq {
int sm_count_reduce();  // reduce.cu

namespace {

constexpr int kMaxSweepsT = 4096;

__global__ void slots_sum_kernel_t(const double *__restrict__ partials, int nblocks, int nslots,
                                   double *__restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < nslots; s += blockDim.x >> 5) {
        double acc = 0.0;
        for (int b = lane; b < nblocks; b += 32) acc += partials[s * MQ_MAX_BLOCKS + b];
        acc = group_sum<32>(acc);
        if (lane == 0) out[s] = acc;
    }
}

// scaled KKT residual, row and entry parts on the ORIGINAL utilities:
// sums of (t y - w)^2, (t - u.x)^2, (x - [x - slack/xi]_+)^2, min(slack, 0)^2
// with slack = p_j - u_ij y_i  (kkt.py:88-111)
__global__ void __launch_bounds__(256)
skkt_rows_kernel(const mq_market mk, const double *__restrict__ x, const double *__restrict__ t,
                 const double *__restrict__ p, const double *__restrict__ y, double xi,
                 double *__restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double s_comp = 0.0, s_viol = 0.0, s_bud = 0.0, s_link = 0.0;
    for (int64_t i = w0; i < mk.n; i += nw) {
        const double yi = y[i];
        double ux = 0.0;
        for (int64_t e = mk.row_ptr[i] + lane; e < mk.row_ptr[i + 1]; e += 32) {
            const double ue = mk.u_orig[e], xe = x[e];
            const double slack = p[mk.col[e]] - ue * yi;
            const double comp = xe - fmax(xe - slack / xi, 0.0);
            const double viol = fmin(slack, 0.0);
            s_comp += comp * comp;
            s_viol += viol * viol;
            ux += ue * xe;
        }
        ux = group_sum<32>(ux);
        if (lane == 0) {
            const double bud = t[i] * yi - mk.w[i];
            const double link = t[i] - ux;
            s_bud += bud * bud;
            s_link += link * link;
        }
    }
    __shared__ double sm[32];
    const double r0 = block_sum(s_bud, sm), r1 = block_sum(s_comp, sm);
    const double r2 = block_sum(s_viol, sm), r3 = block_sum(s_link, sm);
    if (threadIdx.x == 0) {
        scratch[0 * MQ_MAX_BLOCKS + blockIdx.x] = r0;
        scratch[1 * MQ_MAX_BLOCKS + blockIdx.x] = r1;
        scratch[2 * MQ_MAX_BLOCKS + blockIdx.x] = r2;
        scratch[3 * MQ_MAX_BLOCKS + blockIdx.x] = r3;
    }
}

// Smoothed gap, allocation part (kkt.py:150-166): per buyer the exact
// minimizer x_hat of -w log(u.x) + p.x + xi/2 |x - x_c|^2 (tau = 1/xi), then
// -w log(u.x_hat) + p.x_hat + xi/2 |x_hat - x_c|^2 summed over buyers.
// cbuf (nnz) holds c = x_c - tau p[col] during the sweeps.
__global__ void __launch_bounds__(256)
gap_rows_kernel(const mq_market mk, const double *__restrict__ xc, const double *__restrict__ p,
                double xi, double *__restrict__ cbuf, double *__restrict__ scratch,
                int64_t *__restrict__ faults) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double tau = 1.0 / xi;
    double acc = 0.0;
    int nfault = 0;
    for (int64_t i = w0; i < mk.n; i += nw) {
        const int64_t a = mk.row_ptr[i], b = mk.row_ptr[i + 1];
        const double tw = tau * mk.w[i];
        double A = 0.0, B = 0.0;
        for (int64_t e = a + lane; e < b; e += 32) {
            const double ue = mk.u_orig[e];
            const double ce = xc[e] - tau * p[mk.col[e]];
            cbuf[e] = ce;
            A += ue * ce;
            B += ue * ue;
        }
        A = group_sum<32>(A);
        B = group_sum<32>(B);
        double s = active_root(A, B, tw);  // every entry active: a lower bound
        int prev = (int)(b - a);
        bool done = (b == a);
        for (int k = 0; k < kMaxSweepsT && !done; ++k) {
            double As = 0.0, Bs = 0.0;
            int cnt = 0;
            for (int64_t e = a + lane; e < b; e += 32) {
                const double ue = mk.u_orig[e], ce = cbuf[e];
                if (fma(ce, s, tw * ue) > 0.0) {
                    As += ue * ce;
                    Bs += ue * ue;
                    ++cnt;
                }
            }
            As = group_sum<32>(As);
            Bs = group_sum<32>(Bs);
            cnt = (int)group_sum<32>((double)cnt);
            if (cnt == prev || cnt == 0) done = true;
            else {
                s = fmax(active_root(As, Bs, tw), s);
                prev = cnt;
            }
        }
        if (!done && lane == 0) ++nfault;
        const double inv_s = 1.0 / s;
        double ux = 0.0, px = 0.0, dd = 0.0;
        for (int64_t e = a + lane; e < b; e += 32) {
            const double ue = mk.u_orig[e];
            const double xh = fmax(cbuf[e] + tw * ue * inv_s, 0.0);
            const double d = xh - xc[e];
            ux += ue * xh;
            px += p[mk.col[e]] * xh;
            dd += d * d;
        }
        ux = group_sum<32>(ux);
        px = group_sum<32>(px);
        dd = group_sum<32>(dd);
        if (lane == 0) acc += -mk.w[i] * log(ux) + px + 0.5 * xi * dd;
    }
    __shared__ double sm[32];
    const double r = block_sum(acc, sm);
    if (threadIdx.x == 0) scratch[blockIdx.x] = r;
    if (lane == 0 && nfault) atomicAdd(reinterpret_cast<unsigned long long *>(faults),
                                       (unsigned long long)nfault);
}

int row_grid_t(int64_t n) { return grid_for(n, 8, MQ_MAX_BLOCKS); }

}  // namespace
}  // namespace mq

using namespace mq;

extern "C" {

int mq_scaled_kkt_rows(const mq_market *mk, const double *x, const double *t, const double *p,
                       const double *y, double xi, double *out, double *scratch, void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_scaled_kkt_rows: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = row_grid_t(mk->n);
    skkt_rows_kernel<<<grid, 256, 0, s>>>(*mk, x, t, p, y, xi, scratch);
    slots_sum_kernel_t<<<1, 128, 0, s>>>(scratch, grid, 4, out);
    return check_launch("mq_scaled_kkt_rows");
}

int mq_smoothed_gap_rows(const mq_market *mk, const double *xc, const double *p, double xi,
                         double *cbuf, double *out, double *scratch, int64_t *faults,
                         void *stream) {
    if (!mk) return set_error(cudaErrorInvalidValue, "mq_smoothed_gap_rows: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = row_grid_t(mk->n);
    gap_rows_kernel<<<grid, 256, 0, s>>>(*mk, xc, p, xi, cbuf, scratch, faults);
    slots_sum_kernel_t<<<1, 32, 0, s>>>(scratch, grid, 1, out);
    return check_launch("mq_smoothed_gap_rows");
}

}  // extern "C"
