// Device reductions between chunks: KKT residual ingredients (kkt.py:29-87),
// the omega_0 residual norms (driver.py:123-132), restart moves
// (driver.py:156-162) and the Arrow-Debreu budget map E p (exchange.py:89).
//
// Determinism: maxima of nonnegative values go through order-free integer
// atomics on their bit patterns; sums use one partial per block over a grid
// whose size depends only on the problem size, then a fixed-order final pass.
#include "mq_common.cuh"

namespace mq {

int sm_count_reduce() {  // per device (a process may use several GPUs)
    static int n[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    const int k = dev & 63;
    if (!n[k]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[k] = v > 0 ? v : 148;
    }
    return n[k];
}

// scratch layout (doubles)
constexpr int kSlotObj = 0;          // [0, MAXB)      objective partials
constexpr int kSlotBad = 1;          // [MAXB, 2MAXB)  bad-row counts
constexpr int kMisc = 8 * MQ_MAX_BLOCKS;  // 64 misc words
// misc words: [0..3] row maxima bits, [4] first bad row (int64), [8..11] col maxima bits

__global__ void sum_slots_kernel(const double *__restrict__ partials, int nblocks, int nslots,
                                 double *__restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < nslots; s += blockDim.x >> 5) {
        double acc = 0.0;
        for (int b = lane; b < nblocks; b += 32) acc += partials[s * MQ_MAX_BLOCKS + b];
        acc = group_sum<32>(acc);
        if (lane == 0) out[s] = acc;
    }
}

// One G-lane group per buyer (32/G buyers per warp in flight: the row pass is
// latency-bound, so more rows per warp hide more of it).  The row loop is
// warp-uniform; only the entry loops diverge.
// pc[2j] = p_j and pc[2j+1] = the running column maximum share one 16-byte
// slot, so the entry pass makes one random access per entry for both
template <int G>
__global__ void __launch_bounds__(256)
resid_rows_kernel(const mq_market mk, const double *__restrict__ x, double2 *__restrict__ pc,
                  int use_norm, double *__restrict__ t_out, double *__restrict__ y_out,
                  double *__restrict__ scratch, int skip_long) {
    const double *__restrict__ U = use_norm ? mk.u : mk.u_orig;
    constexpr int RPW = 32 / G;  // rows per warp
    const int lane = threadIdx.x & (G - 1);
    const int gsub = (threadIdx.x & 31) / G;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double *misc = scratch + kMisc;
    double ymax = 0.0, gmax = 0.0, xmax = 0.0, emax = 0.0, obj = 0.0, nbad = 0.0;
    for (int64_t base = warp_id * RPW; base < mk.n; base += nwarps * RPW) {
        const int64_t i = base + gsub;
        bool has = i < mk.n;
        int64_t a = 0, b = 0;
        if (has) {
            a = mk.row_ptr[i];
            b = mk.row_ptr[i + 1];
        }
        if (has && skip_long && b - a > MQ_LONG_ROW) {  // resid_rows_long_kernel's row
            has = false;
            b = a;
        }
        double tp = 0.0;
        for (int64_t t = a + lane; t < b; t += G) tp += U[t] * x[t];
        const double t_i = group_sum<G>(tp);
        const bool ok = has && t_i > 0.0;
        if (has && !ok && lane == 0) {
            nbad += 1.0;
            atomicMin((unsigned long long *)(misc + 4), (unsigned long long)(mk.row_begin + i));
            if (t_out) t_out[i] = t_i;
            if (y_out) y_out[i] = 0.0;
        }
        if (!ok) continue;  // no collectives below
        const double y = mk.w[i] / t_i;
        if (lane == 0) {
            obj += mk.w[i] * log(t_i);
            ymax = fmax(ymax, y);
            if (t_out) t_out[i] = t_i;
            if (y_out) y_out[i] = y;
        }
        for (int64_t t = a + lane; t < b; t += G) {
            const int32_t j = mk.col[t];
            const double uy = U[t] * y;
            const double2 pcj = __ldcg(pc + j);
            // skip the atomic when the column's current maximum already covers
            // uy (a stale read only under-estimates it: still order-free)
            if (uy > pcj.y) atomic_max_nonneg(reinterpret_cast<double *>(pc + j) + 1, uy);
            const double es = fmax(pcj.x - uy, 0.0);
            const double xv = x[t];
            gmax = fmax(gmax, xv * es);
            xmax = fmax(xmax, fabs(xv));
            emax = fmax(emax, es);
        }
    }
    ymax = group_max<32>(ymax);  // each group's lane 0 holds its rows' maximum
    gmax = group_max<32>(gmax);
    xmax = group_max<32>(xmax);
    emax = group_max<32>(emax);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(misc + 0, ymax);
        atomic_max_nonneg(misc + 1, gmax);
        atomic_max_nonneg(misc + 2, xmax);
        atomic_max_nonneg(misc + 3, emax);
    }
    __shared__ double sm[32];
    const double ob = block_sum(obj, sm);
    const double nb = block_sum(nbad, sm);
    if (threadIdx.x == 0) {
        scratch[kSlotObj * MQ_MAX_BLOCKS + blockIdx.x] = ob;
        scratch[kSlotBad * MQ_MAX_BLOCKS + blockIdx.x] = nb;
    }
}

// Both residual row passes of a check (kkt.py:29-87 for the last iterate
// (x, p) and the average (xbar, pbar)) in one sweep: u, col and the x > 0
// flags are read once, x only where flagged, xbar densely, and one 32-byte
// slot per good holds (p, its column max, pbar, its column max), so an entry
// costs one random sector for both.  Same row assignment, lane sums and
// block partials as resid_rows_kernel: bitwise the two separate passes.
#ifndef MQ_RP_MINB
#define MQ_RP_MINB 3  // resident 256-thread CTAs per SM of the fused residual pass
#endif
#ifndef MQ_RP_LB
#define MQ_RP_LB 2  // entries per lane batched ahead of the atomics
#endif
#ifndef MQ_RP_G
#define MQ_RP_G 8  // lanes per row of the residual row passes (32 / MQ_RP_G rows per warp)
#endif
#ifndef MQ_RP_LONG_GRID
#define MQ_RP_LONG_GRID 296  // CTAs of the long-row residual pass (grid + this <= MQ_MAX_BLOCKS)
#endif
#ifndef MQ_RP_GRID
#define MQ_RP_GRID 444  // CTAs of the residual row passes: 3 per SM on 148 SMs; fixes the
                        // order of the objective's block partials (C4 sweep, DESIGN.md §11:
                        // 2/4/1024 -> 12.7 ms, 3/2/444 -> 10.2 ms per check)
#endif
static_assert(MQ_RP_GRID + MQ_RP_LONG_GRID <= MQ_MAX_BLOCKS, "partial slots");
template <int G>
__global__ void __launch_bounds__(256, MQ_RP_MINB)
resid_pair_kernel(const mq_market mk, const double *__restrict__ x,
                  const uint8_t *__restrict__ xflag, const double *__restrict__ xbar,
                  const double *__restrict__ xsum, const int64_t *__restrict__ navg,
                  double4 *__restrict__ pc4, double *__restrict__ sa, double *__restrict__ sb,
                  int skip_long) {
    const double *__restrict__ U = mk.u_orig;
    // xsum != NULL: the average is read as xsum / navg, bit for bit what
    // avg_materialize_kernel would store (one reciprocal, one product)
    const double cnt = xsum ? (double)*navg : 0.0;
    const bool lazy = cnt > 0.0;
    const double inv = lazy ? 1.0 / cnt : 0.0;
    const double *__restrict__ xb = lazy ? xsum : xbar;
    const double sc = lazy ? inv : 1.0;
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & (G - 1);
    const int gsub = (threadIdx.x & 31) / G;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double ym[2] = {0.0, 0.0}, gm[2] = {0.0, 0.0}, xm[2] = {0.0, 0.0}, em[2] = {0.0, 0.0};
    double obj[2] = {0.0, 0.0}, nbad[2] = {0.0, 0.0};
    double *misc[2] = {sa + kMisc, sb + kMisc};
    for (int64_t base = warp_id * RPW; base < mk.n; base += nwarps * RPW) {
        const int64_t i = base + gsub;
        bool has = i < mk.n;
        int64_t a = 0, b = 0;
        if (has) {
            a = mk.row_ptr[i];
            b = mk.row_ptr[i + 1];
        }
        if (has && skip_long && b - a > MQ_LONG_ROW) {  // resid_pair_long_kernel's row
            has = false;  // the group still joins its warp's shuffles
            b = a;
        }
        double tp = 0.0, tq = 0.0;
        for (int64_t t = a + lane; t < b; t += G) {
            const double ut = U[t];
            if (xflag[t]) tp += ut * x[t];  // zero entries add +0.0 exactly
            tq += ut * (xb[t] * sc);
        }
        const double ti[2] = {group_sum<G>(tp), group_sum<G>(tq)};
        bool ok[2];
        double y[2] = {0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            ok[k] = has && ti[k] > 0.0;
            if (has && !ok[k] && lane == 0) {
                nbad[k] += 1.0;
                atomicMin((unsigned long long *)(misc[k] + 4),
                          (unsigned long long)(mk.row_begin + i));
            }
            if (ok[k]) {
                y[k] = mk.w[i] / ti[k];
                if (lane == 0) {
                    obj[k] += mk.w[i] * log(ti[k]);
                    ym[k] = fmax(ym[k], y[k]);
                }
            }
        }
        if (!ok[0] && !ok[1]) continue;
        // LB entries per lane per batch: every load of the batch (and its
        // price-slot gather) is issued before the atomics that consume them
        constexpr int LB = MQ_RP_LB;
        for (int64_t t0 = a + lane; t0 < b; t0 += LB * G) {
            int32_t jv[LB];
            double uv[LB], xv[LB], bv[LB];
            double2 q01[LB], q23[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int64_t t = t0 + q * G;
                const bool in = t < b;
                jv[q] = in ? mk.col[t] : 0;
                MQ_CHECK(jv[q] >= 0 && jv[q] < mk.m);
                uv[q] = in ? U[t] : 0.0;
                xv[q] = (in && xflag[t]) ? x[t] : 0.0;
                bv[q] = in ? xb[t] * sc : 0.0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
#ifdef MQ_RESID_LD2  // two 16-byte loads of the slot (the earlier form)
                q01[q] = __ldcg(reinterpret_cast<const double2 *>(pc4 + jv[q]));
                q23[q] = __ldcg(reinterpret_cast<const double2 *>(pc4 + jv[q]) + 1);
#else  // one 32-byte load (sm_100 LDG.256): one L2 request per entry
                asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(q01[q].x), "=d"(q01[q].y), "=d"(q23[q].x), "=d"(q23[q].y)
                             : "l"(pc4 + jv[q]));
#endif
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                if (t0 + q * G >= b) continue;
                const int32_t j = jv[q];
                if (ok[0]) {
                    const double uy = uv[q] * y[0];
                    if (uy > q01[q].y)
                        atomic_max_nonneg(reinterpret_cast<double *>(pc4 + j) + 1, uy);
                    const double es = fmax(q01[q].x - uy, 0.0);
                    gm[0] = fmax(gm[0], xv[q] * es);
                    xm[0] = fmax(xm[0], fabs(xv[q]));
                    em[0] = fmax(em[0], es);
                }
                if (ok[1]) {
                    const double uy = uv[q] * y[1];
                    if (uy > q23[q].y)
                        atomic_max_nonneg(reinterpret_cast<double *>(pc4 + j) + 3, uy);
                    const double es = fmax(q23[q].x - uy, 0.0);
                    gm[1] = fmax(gm[1], bv[q] * es);
                    xm[1] = fmax(xm[1], fabs(bv[q]));
                    em[1] = fmax(em[1], es);
                }
            }
        }
    }
    __shared__ double sm[32];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double a0 = group_max<32>(ym[k]), a1 = group_max<32>(gm[k]);
        const double a2 = group_max<32>(xm[k]), a3 = group_max<32>(em[k]);
        if ((threadIdx.x & 31) == 0) {
            atomic_max_nonneg(misc[k] + 0, a0);
            atomic_max_nonneg(misc[k] + 1, a1);
            atomic_max_nonneg(misc[k] + 2, a2);
            atomic_max_nonneg(misc[k] + 3, a3);
        }
        const double ob = block_sum(obj[k], sm);
        const double nb = block_sum(nbad[k], sm);
        double *sc = k ? sb : sa;
        if (threadIdx.x == 0) {
            sc[kSlotObj * MQ_MAX_BLOCKS + blockIdx.x] = ob;
            sc[kSlotBad * MQ_MAX_BLOCKS + blockIdx.x] = nb;
        }
    }
}

// resid_rows_kernel's rows longer than MQ_LONG_ROW, one CTA per row with
// resid_pair_long_kernel's assignment and entry-to-thread map (so the two
// passes stay bitwise the fused one).
template <int T>
__global__ void __launch_bounds__(T)
resid_rows_long_kernel(const mq_market mk, const double *__restrict__ x,
                       double2 *__restrict__ pc, int use_norm, double *__restrict__ t_out,
                       double *__restrict__ y_out, double *__restrict__ scratch, int slot0) {
    const double *__restrict__ U = use_norm ? mk.u : mk.u_orig;
    const int tid = threadIdx.x;
    __shared__ double sm[32];
    __shared__ double tb;
    double *misc = scratch + kMisc;
    double ymax = 0.0, gmax = 0.0, xmax = 0.0, emax = 0.0, obj = 0.0, nbad = 0.0;
    for (int64_t r = blockIdx.x; r < mk.nlong; r += gridDim.x) {
        const int64_t i = mk.long_rows[r];
        MQ_CHECK(i >= 0 && i < mk.n);
        const int64_t a = mk.row_ptr[i], b = mk.row_ptr[i + 1];
        double tp = 0.0;
        for (int64_t t = a + tid; t < b; t += T) tp += U[t] * x[t];
        tp = block_sum(tp, sm);
        if (tid == 0) tb = tp;
        __syncthreads();
        const double t_i = tb;
        __syncthreads();
        const bool ok = t_i > 0.0;
        if (!ok) {
            if (tid == 0) {
                nbad += 1.0;
                atomicMin((unsigned long long *)(misc + 4),
                          (unsigned long long)(mk.row_begin + i));
                if (t_out) t_out[i] = t_i;
                if (y_out) y_out[i] = 0.0;
            }
            continue;  // block-uniform
        }
        const double y = mk.w[i] / t_i;
        if (tid == 0) {
            obj += mk.w[i] * log(t_i);
            ymax = fmax(ymax, y);
            if (t_out) t_out[i] = t_i;
            if (y_out) y_out[i] = y;
        }
        for (int64_t t = a + tid; t < b; t += T) {
            const int32_t j = mk.col[t];
            const double uy = U[t] * y;
            const double2 pcj = __ldcg(pc + j);
            if (uy > pcj.y) atomic_max_nonneg(reinterpret_cast<double *>(pc + j) + 1, uy);
            const double es = fmax(pcj.x - uy, 0.0);
            const double xv = x[t];
            gmax = fmax(gmax, xv * es);
            xmax = fmax(xmax, fabs(xv));
            emax = fmax(emax, es);
        }
    }
    ymax = group_max<32>(ymax);
    gmax = group_max<32>(gmax);
    xmax = group_max<32>(xmax);
    emax = group_max<32>(emax);
    if ((tid & 31) == 0) {
        atomic_max_nonneg(misc + 0, ymax);
        atomic_max_nonneg(misc + 1, gmax);
        atomic_max_nonneg(misc + 2, xmax);
        atomic_max_nonneg(misc + 3, emax);
    }
    const double ob = block_sum(obj, sm);
    const double nb = block_sum(nbad, sm);
    if (tid == 0) {
        scratch[kSlotObj * MQ_MAX_BLOCKS + slot0 + blockIdx.x] = ob;
        scratch[kSlotBad * MQ_MAX_BLOCKS + slot0 + blockIdx.x] = nb;
    }
}

// The rows longer than MQ_LONG_ROW (mk.long_rows, longest first) of the
// residual pair, one CTA per row (static cyclic assignment: the partial
// sums' order depends only on the market): on power-law markets a
// G-lane group would leave the few longest rows as the pass's tail.  The
// same per-entry work as resid_pair_kernel; each CTA's objective and
// bad-row partials go to partial slot slot0 + blockIdx.x.
template <int T>
__global__ void __launch_bounds__(T)
resid_pair_long_kernel(const mq_market mk, const double *__restrict__ x,
                       const uint8_t *__restrict__ xflag, const double *__restrict__ xbar,
                       const double *__restrict__ xsum, const int64_t *__restrict__ navg,
                       double4 *__restrict__ pc4, double *__restrict__ sa,
                       double *__restrict__ sb, int slot0) {
    const double *__restrict__ U = mk.u_orig;
    const double cnt = xsum ? (double)*navg : 0.0;
    const bool lazy = cnt > 0.0;
    const double inv = lazy ? 1.0 / cnt : 0.0;
    const double *__restrict__ xb = lazy ? xsum : xbar;
    const double sc = lazy ? inv : 1.0;
    const int tid = threadIdx.x;
    __shared__ double sm[32];
    __shared__ double tb[2];
    double ym[2] = {0.0, 0.0}, gm[2] = {0.0, 0.0}, xm[2] = {0.0, 0.0}, em[2] = {0.0, 0.0};
    double obj[2] = {0.0, 0.0}, nbad[2] = {0.0, 0.0};
    double *misc[2] = {sa + kMisc, sb + kMisc};
    for (int64_t r = blockIdx.x; r < mk.nlong; r += gridDim.x) {
        const int64_t i = mk.long_rows[r];
        MQ_CHECK(i >= 0 && i < mk.n);
        const int64_t a = mk.row_ptr[i], b = mk.row_ptr[i + 1];
        double tp = 0.0, tq = 0.0;
        for (int64_t t = a + tid; t < b; t += T) {
            const double ut = U[t];
            if (xflag[t]) tp += ut * x[t];
            tq += ut * (xb[t] * sc);
        }
        tp = block_sum(tp, sm);
        tq = block_sum(tq, sm);
        if (tid == 0) {
            tb[0] = tp;
            tb[1] = tq;
        }
        __syncthreads();
        const double ti[2] = {tb[0], tb[1]};
        __syncthreads();  // tb is rewritten by the next row
        bool ok[2];
        double y[2] = {0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            ok[k] = ti[k] > 0.0;
            if (!ok[k] && tid == 0) {
                nbad[k] += 1.0;
                atomicMin((unsigned long long *)(misc[k] + 4),
                          (unsigned long long)(mk.row_begin + i));
            }
            if (ok[k]) {
                y[k] = mk.w[i] / ti[k];
                if (tid == 0) {
                    obj[k] += mk.w[i] * log(ti[k]);
                    ym[k] = fmax(ym[k], y[k]);
                }
            }
        }
        if (!ok[0] && !ok[1]) continue;  // block-uniform
        constexpr int LB = MQ_RP_LB;
        for (int64_t t0 = a + tid; t0 < b; t0 += LB * T) {
            int32_t jv[LB];
            double uv[LB], xv[LB], bv[LB];
            double2 q01[LB], q23[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int64_t t = t0 + q * T;
                const bool in = t < b;
                jv[q] = in ? mk.col[t] : 0;
                MQ_CHECK(jv[q] >= 0 && jv[q] < mk.m);
                uv[q] = in ? U[t] : 0.0;
                xv[q] = (in && xflag[t]) ? x[t] : 0.0;
                bv[q] = in ? xb[t] * sc : 0.0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q)
                asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(q01[q].x), "=d"(q01[q].y), "=d"(q23[q].x), "=d"(q23[q].y)
                             : "l"(pc4 + jv[q]));
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                if (t0 + q * T >= b) continue;
                const int32_t j = jv[q];
                if (ok[0]) {
                    const double uy = uv[q] * y[0];
                    if (uy > q01[q].y)
                        atomic_max_nonneg(reinterpret_cast<double *>(pc4 + j) + 1, uy);
                    const double es = fmax(q01[q].x - uy, 0.0);
                    gm[0] = fmax(gm[0], xv[q] * es);
                    xm[0] = fmax(xm[0], fabs(xv[q]));
                    em[0] = fmax(em[0], es);
                }
                if (ok[1]) {
                    const double uy = uv[q] * y[1];
                    if (uy > q23[q].y)
                        atomic_max_nonneg(reinterpret_cast<double *>(pc4 + j) + 3, uy);
                    const double es = fmax(q23[q].x - uy, 0.0);
                    gm[1] = fmax(gm[1], bv[q] * es);
                    xm[1] = fmax(xm[1], fabs(bv[q]));
                    em[1] = fmax(em[1], es);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double a0 = group_max<32>(ym[k]), a1 = group_max<32>(gm[k]);
        const double a2 = group_max<32>(xm[k]), a3 = group_max<32>(em[k]);
        if ((tid & 31) == 0) {
            atomic_max_nonneg(misc[k] + 0, a0);
            atomic_max_nonneg(misc[k] + 1, a1);
            atomic_max_nonneg(misc[k] + 2, a2);
            atomic_max_nonneg(misc[k] + 3, a3);
        }
        const double ob = block_sum(obj[k], sm);
        const double nb = block_sum(nbad[k], sm);
        double *scr = k ? sb : sa;
        if (tid == 0) {
            scr[kSlotObj * MQ_MAX_BLOCKS + slot0 + blockIdx.x] = ob;
            scr[kSlotBad * MQ_MAX_BLOCKS + slot0 + blockIdx.x] = nb;
        }
    }
}

__global__ void pc4_init_kernel(int64_t m, const double *__restrict__ p,
                                const double *__restrict__ pbar, double4 *__restrict__ pc4) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        pc4[j] = make_double4(p[j], 0.0, pbar[j], 0.0);
}
__global__ void pc4_out_kernel(int64_t m, const double4 *__restrict__ pc4,
                               double *__restrict__ cb0, double *__restrict__ cb1) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double4 q = pc4[j];
        cb0[j] = fmax(cb0[j], q.y);
        cb1[j] = fmax(cb1[j], q.w);
    }
}

__global__ void pc_init_kernel(int64_t m, const double *__restrict__ p, double2 *__restrict__ pc) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        pc[j] = make_double2(p[j], 0.0);
}
__global__ void pc_out_kernel(int64_t m, const double2 *__restrict__ pc,
                              double *__restrict__ colbest) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        colbest[j] = fmax(colbest[j], pc[j].y);
}

__global__ void resid_rows_finish(const double *__restrict__ scratch, const double *__restrict__ sums,
                                  double *__restrict__ row_out) {
    const double *misc = scratch + kMisc;
    row_out[0] = misc[0];
    row_out[1] = misc[1];
    row_out[2] = misc[2];
    row_out[3] = misc[3];
    const unsigned long long bad = __double_as_longlong(misc[4]);
    row_out[4] = bad == 0xffffffffffffffffull ? -1.0 : (double)(long long)bad;
    row_out[5] = sums[0];
    row_out[6] = sums[1];
    row_out[7] = 0.0;
}

__global__ void __launch_bounds__(256)
resid_cols_kernel(int64_t m, const double *__restrict__ cs, const double *__restrict__ p,
                  const double *__restrict__ colbest, double *__restrict__ scratch) {
    double *misc = scratch + kMisc;
    double gap = 0.0, csmax = 0.0, dualp = 0.0, slmax = 0.0, sq1 = 0.0, sq2 = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double c = cs[j];
        const double sl = p[j] - colbest[j];
        gap = fmax(gap, fabs(c - 1.0));
        csmax = fmax(csmax, fabs(c));
        dualp = fmax(dualp, fmax(-sl, 0.0));
        slmax = fmax(slmax, sl);
        sq1 += (c - 1.0) * (c - 1.0);
        const double d = fmin(sl, 0.0);
        sq2 += d * d;
    }
    gap = group_max<32>(gap);
    csmax = group_max<32>(csmax);
    dualp = group_max<32>(dualp);
    slmax = group_max<32>(slmax);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(misc + 8, gap);
        atomic_max_nonneg(misc + 9, csmax);
        atomic_max_nonneg(misc + 10, dualp);
        atomic_max_nonneg(misc + 11, slmax);
    }
    __shared__ double sm[32];
    const double a = block_sum(sq1, sm);
    const double b = block_sum(sq2, sm);
    if (threadIdx.x == 0) {
        scratch[2 * MQ_MAX_BLOCKS + blockIdx.x] = a;
        scratch[3 * MQ_MAX_BLOCKS + blockIdx.x] = b;
    }
}

__global__ void resid_cols_finish(const double *__restrict__ scratch, const double *__restrict__ sums,
                                  double *__restrict__ col_out) {
    const double *misc = scratch + kMisc;
    col_out[0] = misc[8];
    col_out[1] = misc[9];
    col_out[2] = misc[10];
    col_out[3] = misc[11];
    col_out[4] = sums[0];
    col_out[5] = sums[1];
}

__global__ void __launch_bounds__(256)
moves_nnz_kernel(int64_t nnz, const double *__restrict__ xbar, const double *__restrict__ x0,
                 double *__restrict__ scratch) {
    double acc = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double d = xbar[k] - x0[k];
        acc += d * d;
    }
    __shared__ double sm[32];
    const double r = block_sum(acc, sm);
    if (threadIdx.x == 0) scratch[blockIdx.x] = r;
}

__global__ void __launch_bounds__(256)
moves_m_kernel(int64_t m, const double *__restrict__ pbar, const double *__restrict__ p0,
               const double *__restrict__ csbar, const double *__restrict__ cs0,
               double *__restrict__ scratch) {
    double a = 0.0, b = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double dp = pbar[j] - p0[j];
        a += dp * dp;
        b += (csbar[j] - cs0[j]) * dp;
    }
    __shared__ double sm[32];
    const double ra = block_sum(a, sm);
    const double rb = block_sum(b, sm);
    if (threadIdx.x == 0) {
        scratch[MQ_MAX_BLOCKS + blockIdx.x] = ra;
        scratch[2 * MQ_MAX_BLOCKS + blockIdx.x] = rb;
    }
}

__global__ void __launch_bounds__(256)
spmv_kernel(int64_t n, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
            const double *__restrict__ val, const double *__restrict__ v, double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp_id; i < n; i += nwarps) {
        double acc = 0.0;
        for (int64_t t = row_ptr[i] + lane; t < row_ptr[i + 1]; t += 32) acc += val[t] * v[col[t]];
        acc = group_sum<32>(acc);
        if (lane == 0) out[i] = acc;
    }
}

__global__ void __launch_bounds__(256)
normalize_kernel(int64_t n, const int64_t *__restrict__ row_ptr, const double *__restrict__ u,
                 double *__restrict__ u_out, double *__restrict__ scales) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp_id; i < n; i += nwarps) {
        const int64_t a = row_ptr[i], b = row_ptr[i + 1];
        double mx = 0.0;
        for (int64_t t = a + lane; t < b; t += 32) mx = fmax(mx, u[t]);
        mx = group_max<32>(mx);
        for (int64_t t = a + lane; t < b; t += 32) u_out[t] = u[t] / mx;
        if (lane == 0) scales[i] = mx;
    }
}

}  // namespace mq

using namespace mq;

extern "C" {

int64_t mq_scratch_doubles(void) { return MQ_SCRATCH_DOUBLES; }

int mq_resid_rows(const mq_market *mk, const double *x, const double *p, int use_norm,
                  double *colbest, double *work, double *t_out, double *y_out, double *row_out,
                  double *scratch, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = grid_for(mk->n, 8, MQ_RP_GRID);
    cudaMemsetAsync(scratch + kMisc, 0, 4 * sizeof(double), s);
    cudaMemsetAsync(scratch + kMisc + 4, 0xff, sizeof(double), s);
    double2 *pc = reinterpret_cast<double2 *>(work);
    if (!pc) {  // no caller workspace: a stream-ordered temporary
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&pc),
                                        (size_t)(mk->m > 0 ? mk->m : 1) * sizeof(double2), s);
        if (e != cudaSuccess) return set_error(e, "mq_resid_rows: workspace");
    }
    const int gm = grid_for(mk->m, 256, MQ_MAX_BLOCKS);
    pc_init_kernel<<<gm, 256, 0, s>>>(mk->m, p, pc);
    const int glong = mk->nlong > 0 && mk->long_rows
                          ? grid_for(mk->nlong, 1, MQ_RP_LONG_GRID) : 0;
    resid_rows_kernel<MQ_RP_G><<<grid, 256, 0, s>>>(*mk, x, pc, use_norm, t_out, y_out, scratch,
                                              glong > 0);
    if (glong)
        resid_rows_long_kernel<256><<<glong, 256, 0, s>>>(*mk, x, pc, use_norm, t_out, y_out,
                                                          scratch, grid);
    pc_out_kernel<<<gm, 256, 0, s>>>(mk->m, pc, colbest);
    if (!work) cudaFreeAsync(pc, s);
    sum_slots_kernel<<<1, 64, 0, s>>>(scratch, grid + glong, 2, scratch + kMisc + 16);
    resid_rows_finish<<<1, 1, 0, s>>>(scratch, scratch + kMisc + 16, row_out);
    return check_launch("mq_resid_rows");
}

int mq_resid_rows_pair(const mq_market *mk, const mq_state *st, double *colbest_last,
                       double *colbest_avg, double *work, double *row_out_last,
                       double *row_out_avg, double *scratch_last, double *scratch_avg,
                       void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!mk || !st || !work) return set_error(cudaErrorInvalidValue, "mq_resid_rows_pair: null");
    const int grid = grid_for(mk->n, 8, MQ_RP_GRID);
    for (double *sc : {scratch_last, scratch_avg}) {
        cudaMemsetAsync(sc + kMisc, 0, 4 * sizeof(double), s);
        cudaMemsetAsync(sc + kMisc + 4, 0xff, sizeof(double), s);
    }
    double4 *pc4 = reinterpret_cast<double4 *>(work);
    const int gm = grid_for(mk->m, 256, MQ_MAX_BLOCKS);
    pc4_init_kernel<<<gm, 256, 0, s>>>(mk->m, st->p, st->pbar, pc4);
    const double *xs = st->xbar_lazy ? st->xsum : nullptr;
    // long rows (if any) get a CTA each; their partials follow the main grid's
    const int glong = mk->nlong > 0 && mk->long_rows
                          ? grid_for(mk->nlong, 1, MQ_RP_LONG_GRID) : 0;
    resid_pair_kernel<MQ_RP_G><<<grid, 256, 0, s>>>(*mk, st->x, st->xflag, st->xbar, xs, st->navg,
                                              pc4, scratch_last, scratch_avg, glong > 0);
    if (glong)
        resid_pair_long_kernel<256><<<glong, 256, 0, s>>>(*mk, st->x, st->xflag, st->xbar, xs,
                                                          st->navg, pc4, scratch_last,
                                                          scratch_avg, grid);
    pc4_out_kernel<<<gm, 256, 0, s>>>(mk->m, pc4, colbest_last, colbest_avg);
    sum_slots_kernel<<<1, 64, 0, s>>>(scratch_last, grid + glong, 2, scratch_last + kMisc + 16);
    resid_rows_finish<<<1, 1, 0, s>>>(scratch_last, scratch_last + kMisc + 16, row_out_last);
    sum_slots_kernel<<<1, 64, 0, s>>>(scratch_avg, grid + glong, 2, scratch_avg + kMisc + 16);
    resid_rows_finish<<<1, 1, 0, s>>>(scratch_avg, scratch_avg + kMisc + 16, row_out_avg);
    return check_launch("mq_resid_rows_pair");
}

int mq_resid_cols(int64_t m, const double *cs, const double *p, const double *colbest,
                  double *col_out, double *scratch, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = grid_for(m, 256, MQ_MAX_BLOCKS);
    cudaMemsetAsync(scratch + kMisc + 8, 0, 4 * sizeof(double), s);
    resid_cols_kernel<<<grid, 256, 0, s>>>(m, cs, p, colbest, scratch);
    sum_slots_kernel<<<1, 64, 0, s>>>(scratch + 2 * MQ_MAX_BLOCKS, grid, 2, scratch + kMisc + 20);
    resid_cols_finish<<<1, 1, 0, s>>>(scratch, scratch + kMisc + 20, col_out);
    return check_launch("mq_resid_cols");
}

int mq_restart_moves(const mq_market *mk, const double *xbar, const double *x0, const double *pbar,
                     const double *p0, const double *csbar, const double *cs0, double *out,
                     double *scratch, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int g1 = grid_for(mk->nnz, 2048, MQ_MAX_BLOCKS);
    const int g2 = grid_for(mk->m, 256, MQ_MAX_BLOCKS);
    moves_nnz_kernel<<<g1, 256, 0, s>>>(mk->nnz, xbar, x0, scratch);
    moves_m_kernel<<<g2, 256, 0, s>>>(mk->m, pbar, p0, csbar, cs0, scratch);
    sum_slots_kernel<<<1, 32, 0, s>>>(scratch, g1, 1, out);
    sum_slots_kernel<<<1, 64, 0, s>>>(scratch + MQ_MAX_BLOCKS, g2, 2, out + 1);
    return check_launch("mq_restart_moves");
}

int mq_normalize_rows(int64_t n, const int64_t *row_ptr, const double *u, double *u_out,
                      double *scales, void *stream) {
    const int grid = grid_for(n, 8, sm_count_reduce() * 16);
    normalize_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, row_ptr, u, u_out, scales);
    return check_launch("mq_normalize_rows");
}

int mq_spmv(int64_t n_rows, const int64_t *row_ptr, const int32_t *col, const double *val,
            const double *v, double *out, void *stream) {
    const int grid = grid_for(n_rows, 8, sm_count_reduce() * 16);
    spmv_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n_rows, row_ptr, col, val, v, out);
    return check_launch("mq_spmv");
}

}  // extern "C"
