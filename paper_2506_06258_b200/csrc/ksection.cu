// Faithful drop-in for kernels.pdhcg_chunk (kernels.py:99-145) on sm_100a.
//
// Compiled with --fmad=false: every product and sum rounds exactly where the
// reference's does, and every serial sum runs in the reference's order, so
// the output is bit-identical to the numba kernel on the same inputs.
//
// Mapping (the reference's serial loops, parallelised without reordering
// any floating-point reduction):
//  * price step   one thread per good, serial ascending-row sum over the
//                 transpose schedule (kernels.py:111-116);
//  * row search   one warp per buyer; the k-section pass evaluates its
//                 sections-1 candidates (kernels.py:73-88) one per lane, each
//                 a serial row sweep (_g_eval, kernels.py:22-30); the bracket
//                 fold is an order-free min/max, and the "first exact hit in
//                 l order" rule becomes a warp min over l;
//  * averages     elementwise (kernels.py:138-144).
#include "mq_common.cuh"

namespace mq {

constexpr int kMaxRowPasses = 200;          // kernels.py:16
constexpr double kRelWidthFloor = 4e-16;    // kernels.py:19

__global__ void ks_dual_kernel(int64_t m, const int64_t *__restrict__ tindptr,
                               const int32_t *__restrict__ tperm, const double *__restrict__ x,
                               const double *__restrict__ x_prev, double *__restrict__ p,
                               double sigma) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t t = tindptr[j]; t < tindptr[j + 1]; ++t) {
            const int32_t k = tperm[t];
            acc += 2.0 * x[k] - x_prev[k];
        }
        p[j] += sigma * (acc - 1.0);
    }
}

// u . max(0, c + tw*u/s) over [a, b), serial (kernels.py:22-30)
__device__ double ks_g_eval(int64_t a, int64_t b, const double *__restrict__ u,
                            const double *__restrict__ c, double tw, double s) {
    double acc = 0.0;
    for (int64_t t = a; t < b; ++t) {
        const double ut = u[t];
        const double xv = c[t] + (tw * ut) / s;
        if (xv > 0.0) acc += ut * xv;
    }
    return acc;
}

__device__ __forceinline__ double ks_candidate(int sections, int l, double lo, double hi) {
    return ((double)(sections - l) * lo + (double)l * hi) / (double)sections;
}

// One warp per row.  Returns the root; *npass = passes or -1 (fault).
__device__ double ks_row_root(int64_t a, int64_t b, const double *__restrict__ u,
                              const double *__restrict__ c, double tw, double s0, int sections,
                              double tol, int *npass) {
    const int lane = threadIdx.x & 31;
    double s_t;
    if (s0 > 0.0) {
        s_t = s0;
    } else {
        double usq = 0.0;
        for (int64_t t = a; t < b; ++t) usq += u[t] * u[t];
        s_t = sqrt(tw * usq);
        if (s_t <= 0.0) s_t = 1e-12 * (1.0 + tw);
    }
    const double st = ks_g_eval(a, b, u, c, tw, s_t);
    if (st == s_t) {
        *npass = 0;
        return s_t;
    }
    double lo = st > s_t ? s_t : st;
    double hi = st > s_t ? st : s_t;
    int np = 0;
    for (;;) {
        const double floor_w = kRelWidthFloor * (hi > 1.0 ? hi : 1.0);
        const double eff = tol > floor_w ? tol : floor_w;
        if (hi - lo <= eff) {
            *npass = np;
            return 0.5 * (lo + hi);
        }
        np += 1;
        if (np > kMaxRowPasses) {
            *npass = -1;
            return 0.5 * (lo + hi);
        }
        double nhi = hi, nlo = lo;
        int hit = 0x7fffffff;
        for (int l = lane + 1; l < sections; l += 32) {
            const double sl = ks_candidate(sections, l, lo, hi);
            if (sl <= lo || sl >= hi) continue;
            const double gl = ks_g_eval(a, b, u, c, tw, sl);
            if (gl == sl) {
                hit = l;  // first hit of this lane (l increases)
                break;
            }
            const double up = sl > gl ? sl : gl;
            const double dn = sl > gl ? gl : sl;
            if (up < nhi) nhi = up;
            if (dn > nlo) nlo = dn;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hit = min(hit, __shfl_xor_sync(MQ_FULL, hit, o));
        if (hit != 0x7fffffff) {
            *npass = np;
            return ks_candidate(sections, hit, lo, hi);
        }
        nhi = group_min<32>(nhi);
        nlo = group_max<32>(nlo);
        if (nhi == hi && nlo == lo) {
            *npass = np;
            return 0.5 * (lo + hi);
        }
        hi = nhi;
        lo = nlo;
    }
}

__global__ void __launch_bounds__(256)
ks_primal_kernel(int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ colind,
                 const double *__restrict__ uval, const double *__restrict__ w,
                 double *__restrict__ x, const double *__restrict__ x_prev,
                 const double *__restrict__ p, double *__restrict__ cbuf, double tau,
                 int sections, double subtol, unsigned long long *pass_slot,
                 unsigned long long *fault_slot) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t my_pass = 0, my_fault = 0;
    for (int64_t i = warp_id; i < n; i += nwarps) {
        const int64_t a = indptr[i], b = indptr[i + 1];
        if (b == a) continue;
        const double tw = tau * w[i];
        for (int64_t t = a + lane; t < b; t += 32) cbuf[t] = x_prev[t] - tau * p[colind[t]];
        __syncwarp();
        double s0 = 0.0;  // serial, ascending t (kernels.py:126-128)
        for (int64_t t = a; t < b; ++t) s0 += uval[t] * x_prev[t];
        int np;
        const double s = ks_row_root(a, b, uval, cbuf, tw, s0, sections, subtol, &np);
        if (lane == 0) {
            if (np < 0) my_fault += 1;
            else my_pass += np;
        }
        for (int64_t t = a + lane; t < b; t += 32) {
            const double xv = cbuf[t] + (tw * uval[t]) / s;
            x[t] = xv > 0.0 ? xv : 0.0;
        }
        __syncwarp();
    }
    __shared__ int64_t red[32];
    const int64_t tp = block_sum_i64(my_pass, red);
    if (threadIdx.x == 0 && tp) atomicAdd(pass_slot, (unsigned long long)tp);
    const int64_t tf = block_sum_i64(my_fault, red);
    if (threadIdx.x == 0 && tf) atomicAdd(fault_slot, (unsigned long long)tf);
}

__global__ void ks_avg_kernel(int64_t len, double *__restrict__ bar, const double *__restrict__ v,
                              double wold, double wnew) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x)
        bar[k] = wold * bar[k] + wnew * v[k];
}

}  // namespace mq

using namespace mq;

extern "C" int mq_pdhcg_chunk(int64_t n, int64_t m, const int64_t *indptr, const int32_t *colind,
                              const double *uval, const int32_t *tperm, const int64_t *tindptr,
                              const double *w, double *x, double *x_prev, double *p, double *xbar,
                              double *pbar, int64_t navg, double tau, double sigma, int sections,
                              double subtol, int iters, double *c_buf, int64_t *pass_out,
                              int64_t *navg_out_host, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t nnz = 0;
    cudaError_t e = cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return set_error(e, "mq_pdhcg_chunk: nnz");
    unsigned long long *fault_slot = nullptr;
    e = cudaMallocAsync((void **)&fault_slot, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return set_error(e, "mq_pdhcg_chunk: alloc");
    cudaMemsetAsync(fault_slot, 0, sizeof(unsigned long long), s);
    cudaMemsetAsync(pass_out, 0, sizeof(int64_t) * (size_t)iters, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_error(e, "mq_pdhcg_chunk: sync");
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int g_cols = grid_for(m, 128, nsm * 8);
    const int g_rows = grid_for(n, 8, nsm * 16);
    const int g_nnz = grid_for(nnz, 256, nsm * 16);
    const int g_m = grid_for(m, 256, nsm * 4);
    int64_t count = navg;
    for (int it = 0; it < iters; ++it) {
        ks_dual_kernel<<<g_cols, 128, 0, s>>>(m, tindptr, tperm, x, x_prev, p, sigma);
        cudaMemcpyAsync(x_prev, x, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice, s);
        ks_primal_kernel<<<g_rows, 256, 0, s>>>(n, indptr, colind, uval, w, x, x_prev, p, c_buf,
                                                 tau, sections, subtol,
                                                 (unsigned long long *)(pass_out + it), fault_slot);
        count += 1;
        const double wold = ((double)count - 1.0) / (double)count;
        const double wnew = 1.0 / (double)count;
        ks_avg_kernel<<<g_nnz, 256, 0, s>>>(nnz, xbar, x, wold, wnew);
        ks_avg_kernel<<<g_m, 256, 0, s>>>(m, pbar, p, wold, wnew);
    }
    if (check_launch("mq_pdhcg_chunk")) {
        cudaFreeAsync(fault_slot, s);
        return -1;
    }
    unsigned long long faults = 0;
    cudaMemcpyAsync(&faults, fault_slot, sizeof(faults), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(fault_slot, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_error(e, "mq_pdhcg_chunk: final sync");
    if (navg_out_host) *navg_out_host = count;
    return (int)faults;
}
