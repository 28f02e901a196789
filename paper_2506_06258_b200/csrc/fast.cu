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
//
// One persistent, warp-specialized kernel per iteration (primal_fused_kernel):
//  * a TMA producer warp streams each tile (whole rows, <= MQ_TILE_ENTRIES
//    entries: u, col, x, xbar, row offsets, budgets) into a 3-stage
//    shared-memory ring with cp.async.bulk + mbarrier transaction counts;
//  * 16 solver warps claim row pairs of the current tile (two 16-lane groups
//    per warp) and solve them from shared memory, writing x and xbar;
//  * 4 column-sum warps gather, block by block, the freshly written x of
//    every finished block of tiles from L2 (one thread per good, ascending
//    rows, fixed order), so the price step's column sums cost no extra HBM
//    pass and overlap the streaming.
#include "mq_common.cuh"

// ---- compile-time configuration (tuning variants override with -D) ----
#ifndef MQ_G
#define MQ_G 16
#endif
// column-sum mode: default = sparse fixed-point atomics (no column-sum warps);
// the gather / scatter / bucket modes are kept as measured alternatives
#if defined(MQ_CS_GATHER) || defined(MQ_SCATTER) || defined(MQ_COLSUM_SPLIT) || \
    defined(MQ_COLSUM_PHASED) || defined(MQ_CS_BUCKET)
#define MQ_CS_DENSE 1
#endif
#ifndef MQ_NCW
#ifdef MQ_CS_DENSE
#define MQ_NCW 4
#else
#define MQ_NCW 0
#endif
#endif
#ifndef MQ_NSW
#if defined(MQ_CS_DENSE)
#define MQ_NSW 15
#elif defined(MQ_XPREFETCH)
#define MQ_NSW 18  /* + the x-prefetch warp: 20 warps at 96 registers */
#else
#define MQ_NSW 19  /* no column-sum warps: 20 warps at 96 registers */
#endif
#endif
#ifndef MQ_NGW
#define MQ_NGW 0
#endif
// Shared memory is sized so that the unified L1 keeps >= 60 KB: random
// gathers (p[col], the column sums' x) need L1 lines to track their misses,
// and their throughput halves when the carveout leaves ~28 KB (tools/micro/
// gather_l1.cu).  Two large stages beat three small ones.
#ifndef MQ_ETILE
#define MQ_ETILE MQ_TILE_ENTRIES
#endif
#ifndef MQ_STAGES
#if defined(MQ_CS_DENSE) || defined(MQ_X_DENSE)
#define MQ_STAGES 2
#else
#define MQ_STAGES 3  /* sparse iterate: 13 B/entry stages, 3 fit with 92 KB of L1 */
#endif
#endif
#ifndef MQ_LAG
#define MQ_LAG 4
#endif
#ifndef MQ_REG_PER
#define MQ_REG_PER 8
#endif
#ifndef MQ_CLAIM
#define MQ_CLAIM 2
#endif
#ifndef MQ_CSQ
#define MQ_CSQ 4
#endif
#ifndef MQ_CSU
#define MQ_CSU 8
#endif
#ifndef MQ_CS_CHUNK
#define MQ_CS_CHUNK 512
#endif
#ifndef MQ_SMEM_PAD
#define MQ_SMEM_PAD 0  /* experiment: extra dynamic shared memory (shrinks L1) */
#endif
#ifndef MQ_WAIT_HINT_NS
#define MQ_WAIT_HINT_NS 0
#endif

namespace mq {

constexpr int kMaxSweeps = 4096;

// cycle counters of the fused kernel's waits (mq_debug_counters): 0 solver
// waiting for a tile, 1 solver throttled, 2 producer waiting for a free stage,
// 3 column-sum warps waiting for a block, 4 column-sum gather cycles
__device__ unsigned long long g_wait_cycles[16];
#ifdef MQ_PROFILE_WAITS
// per-thread accumulation, flushed once when the kernel's scope ends
struct ProfAcc {
    unsigned long long v[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    __device__ ~ProfAcc() {
        for (int i = 0; i < 16; ++i)
            if (v[i]) atomicAdd(&g_wait_cycles[i], v[i]);
    }
};
#define MQ_PROF_DECL() ProfAcc _prof
#define MQ_T0() const long long _t0 = clock64()
#define MQ_T1(slot) (_prof.v[slot] += (unsigned long long)(clock64() - _t0))
#define MQ_TS(v) const long long v = clock64()
#define MQ_TA(slot, a, b) if (wl == 0) _prof.v[slot] += (unsigned long long)((b) - (a))
#else
#define MQ_PROF_DECL()
#define MQ_T0()
#define MQ_T1(slot)
#define MQ_TS(v)
#define MQ_TA(slot, a, b)
#endif

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

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if MQ_WAIT_HINT_NS > 0
    // suspend-time hint: a waiting warp sleeps instead of re-polling shared memory
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MQ_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra MQ_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "n"(MQ_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MQ_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MQ_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// order generic-proxy global writes (observed through an acquire) before
// this thread's subsequent bulk copies from global memory
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// price gather p[col]: read-only, L2-resident (m * 8 bytes); optionally kept
// out of L1 so the gathers do not evict the warps' other L1 lines
__device__ __forceinline__ double ld_price(const double *a) {
#ifdef MQ_EXP_NOP  // timing experiment only (wrong results): no price gathers
    return 1e-3 * (double)(reinterpret_cast<uintptr_t>(a) & 7);
#endif
#ifdef MQ_P_NOALLOC
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a));
    return v;
#else
    return __ldg(a);
#endif
}

// Column sums as fixed-point integers: x_e * cs_scale rounded to u64, added
// with fire-and-forget atomics only for the ~1 % of entries with x_e > 0.
// Integer addition is associative, so the sums are bitwise deterministic in
// any order; cs_scale = 2^e is chosen per market so that no column can
// overflow while every x_e < cs_xmax (a larger x_e is counted as a fault).
__device__ __forceinline__ void fixed_colsum_add(const mq_market &mk, const mq_state &st, int j,
                                                 double xe) {
    if (xe < mk.cs_xmax) {
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(reinterpret_cast<unsigned long long *>(
                         st.bucket) + j),
                     "l"(__double2ull_rn(xe * mk.cs_scale))
                     : "memory");
    } else {
        atomicAdd(reinterpret_cast<unsigned long long *>(st.faults), 1ull);
    }
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

// ------------------------------------------------------------ row solve
// Exact root of s = sum_t u_t max(0, c_t + tw u_t / s) for one row held in
// shared memory (u, c), by a G-lane group.  All groups of a warp call this
// together (warp-uniform loops around the shuffles).  Returns s; *sweeps gets
// the number of active-set evaluations, *ok whether it converged.
template <int G>
__device__ __forceinline__ double row_root_exact(const double *__restrict__ su,
                                                 const double *__restrict__ sc, int a, int b,
                                                 int lane, double tw, double s0, double A,
                                                 double B, bool active_row, int *sweeps,
                                                 bool *ok) {
    const int len = b - a;
    bool done = !active_row || len == 0;
    double s = done ? 1.0 : active_root(A, B, tw);  // all entries active: lower bound
    int prev_cnt = len;
    int nsw = 0;
    auto sweep = [&](double q, double &As, double &Bs, int &cnt) {
        double a_ = 0.0, b_ = 0.0;
        int k_ = 0;
        for (int t = a + lane; t < b; t += G) {
            const double ue = su[t], ce = sc[t];
            if (fma(ce, q, tw * ue) > 0.0) {
                a_ += ue * ce;
                b_ += ue * ue;
                ++k_;
            }
        }
        As = group_sum<G>(a_);
        Bs = group_sum<G>(b_);
        cnt = group_sum_int<G>(k_);
    };
    // the previous iterate's utility s0 is usually next to the new root
    const bool try_s0 = !done && s0 > s;
    if (__any_sync(MQ_FULL, try_s0)) {
        double A0, B0;
        int k0;
        sweep(try_s0 ? s0 : s, A0, B0, k0);
        if (try_s0) {
            ++nsw;
            const double g0 = A0 + tw * B0 / s0;
            if (g0 >= s0) {  // s0 below the root: step from its active set
                s = fmax(active_root(A0, B0, tw), s0);
                prev_cnt = k0;
            } else if (g0 > s) {  // g(s0) is a lower bound above s
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
            ++nsw;
            if (cnt == prev_cnt || cnt == 0) {
                done = true;  // s is the root of its own active set
            } else {
                s = fmax(active_root(As, Bs, tw), s);
                prev_cnt = cnt;
            }
        }
    }
    *sweeps = nsw;
    *ok = done;
    return s;
}

// Same iteration with the row held in registers (PER entries per lane):
// sweeps cost no shared-memory traffic.
template <int G, int PER>
__device__ __forceinline__ double row_root_regs(const double (&c)[PER], const double (&u)[PER],
                                                int len, double tw, double s0, double A,
                                                double B, bool active_row, int *sweeps,
                                                bool *ok) {
    bool done = !active_row || len == 0;
    double s = done ? 1.0 : active_root(A, B, tw);
    int prev_cnt = len;
    int nsw = 0;
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
    const bool try_s0 = !done && s0 > s;
    if (__any_sync(MQ_FULL, try_s0)) {
        double A0, B0;
        int k0;
        sweep(try_s0 ? s0 : s, A0, B0, k0);
        if (try_s0) {
            ++nsw;
            const double g0 = A0 + tw * B0 / s0;
            if (g0 >= s0) {
                s = fmax(active_root(A0, B0, tw), s0);
                prev_cnt = k0;
            } else if (g0 > s) {
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
            ++nsw;
            if (cnt == prev_cnt || cnt == 0) {
                done = true;
            } else {
                s = fmax(active_root(As, Bs, tw), s);
                prev_cnt = cnt;
            }
        }
    }
    *sweeps = nsw;
    *ok = done;
    return s;
}

// Warm-started variant for rows held in registers.  s0 = the row's utility
// after the previous prox (srow; <= 0: none).  The first sweep evaluates the
// active set at s0: if g(s0) >= s0, s0 is below the root and the root of that
// set (or s0) is the next lower bound; otherwise g(s0) < s0 is itself a lower
// bound (g is nonincreasing).  Later sweeps compare each lane's active mask
// with the previous one (a ballot, no reduction) and reduce A, B only when
// the set changed, so a row whose set is already right costs one reduction.
// u(e): the lane's e-th utility (registers, or re-read from shared memory)
template <int G, int PER, class UF>
__device__ __forceinline__ double row_root_warm(const double (&c)[PER], UF u,
                                                double tw, double s0, bool active_row,
                                                uint32_t gmask, int *sweeps, bool *ok) {
    auto amask = [&](double q) -> uint32_t {
        uint32_t msk = 0;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const double ue = u(e);
            if (ue > 0.0 && fma(c[e], q, tw * ue) > 0.0) msk |= 1u << e;
        }
        return msk;
    };
    auto sums = [&](uint32_t msk, double &As, double &Bs) {
        double a_ = 0.0, b_ = 0.0;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            if ((msk >> e) & 1u) {
                const double ue = u(e);
                a_ += ue * c[e];
                b_ += ue * ue;
            }
        }
        As = group_sum<G>(a_);
        Bs = group_sum<G>(b_);
    };
    bool done = !active_row;
    double s = 1.0;
    uint32_t prev = 0;
    bool force = false;
    int nsw = 0;
    {
        const bool warm = s0 > 0.0;
        const uint32_t msk = amask(warm ? s0 : 0.0);  // s0 <= 0: every u > 0 entry
        double A0, B0;
        sums(msk, A0, B0);
        const bool any = (__ballot_sync(MQ_FULL, msk != 0u) & gmask) != 0u;
        if (!done) {
            ++nsw;
            if (!warm) {
                if (any) {
                    s = active_root(A0, B0, tw);
                    prev = msk;
                } else {
                    done = true;  // no entry with u > 0
                }
            } else {
                // g(s0) = A0 + tw B0 / s0 >= s0, without the division
                if (fma(A0, s0, tw * B0) >= s0 * s0) {
                    s = fmax(active_root(A0, B0, tw), s0);
                    prev = msk;
                } else {
                    s = A0 + tw * B0 / s0;  // g(s0): a lower bound, active set unknown
                    force = true;
                }
            }
        }
    }
    for (int k = 0; k < kMaxSweeps; ++k) {
        if (!__any_sync(MQ_FULL, !done)) break;
        const uint32_t msk = amask(s);
        const bool chg = (__ballot_sync(MQ_FULL, msk != prev || force) & gmask) != 0u;
        const bool any = (__ballot_sync(MQ_FULL, msk != 0u) & gmask) != 0u;
        bool need = false;
        if (!done) {
            ++nsw;
            if (!chg || !any) done = true;  // s is the root of its own active set
            else need = true;
        }
        if (__any_sync(MQ_FULL, need)) {
            double As, Bs;
            sums(msk, As, Bs);
            if (need) {
                s = fmax(active_root(As, Bs, tw), s);
                prev = msk;
                force = false;
            }
        }
    }
    *sweeps = nsw;
    *ok = done;
    return s;
}

// ------------------------------------------------------------ primal (fused)
#ifdef MQ_SCATTER
constexpr bool kScatter = true;       // column sums from a column-major copy of x
#else
constexpr bool kScatter = false;
#endif
#ifdef MQ_CS_DENSE
constexpr bool kAtomic = false;
#else
constexpr bool kAtomic = true;        // sparse fixed-point column sums (default)
#endif
#ifdef MQ_CS_BUCKET
constexpr bool kBucket = !kScatter;   // solvers store x into L2 buckets in column order
#else
constexpr bool kBucket = false;
#endif
#ifdef MQ_COLSUM_SPLIT
constexpr bool kSplit = !kScatter && !kBucket;  // per block of tiles: primal launch, then gather launch
#else
constexpr bool kSplit = false;
#endif
#if defined(MQ_COLSUM_PHASED) && !defined(MQ_COLSUM_SPLIT) && !defined(MQ_SCATTER) && !defined(MQ_CS_BUCKET)
constexpr bool kPhased = true;        // solve a block of tiles, grid barrier, gather it from L2
#else
constexpr bool kPhased = false;       // default: column-sum warps gather concurrently (fused)
#endif
constexpr int kPhChunk = 4096;
// Sparse iterate (default with the fixed-point column sums): ~99 % of x is 0
// after the first iteration, so x is not streamed.  A byte flag per entry
// (x > 0) is staged instead; only flagged entries load their x, x is written
// only where it is or was nonzero, and the running average is kept as the
// running sum S = sum of x since the restart (atomic adds on nonzero x only),
// materialized as xbar = S / count once per chunk (mq_avg_materialize).
#if !defined(MQ_CS_DENSE) && !defined(MQ_X_DENSE)
constexpr bool kSparse = true;
#else
constexpr bool kSparse = false;
#endif
#ifdef MQ_X_DIRECT
constexpr bool kXDirect = true;   // x is L2-prefetched and loaded by the solvers, not staged
#else
constexpr bool kXDirect = kSparse;
#endif
// software-pipelined solver warps (sparse iterate only): measured slower (a
// warp holds two tiles' stages, so fewer tiles are in flight); opt-in
#if defined(MQ_PIPE) && !defined(MQ_CS_DENSE) && !defined(MQ_X_DENSE) && \
    !defined(MQ_TRIVIAL_SOLVE) && (MQ_NGW == 0)
constexpr bool kPipe = true;
#else
constexpr bool kPipe = false;
#endif
#ifdef MQ_XB_DIRECT
constexpr bool kXBDirect = true;  // xbar likewise
#else
constexpr bool kXBDirect = kSparse;
#endif
static_assert(!kSparse || kAtomic, "the sparse iterate needs the fixed-point column sums");
// one extra warp that, a tile or two ahead of the solvers, pulls the flagged
// (nonzero) x of each staged tile into L2 (otherwise scattered DRAM reads on
// the solvers' critical path)
// (measured +3 % while the x loads were serialized behind the price gathers;
// no gain since they overlap, so opt-in)
#if defined(MQ_XPREFETCH)
constexpr int kPF = kSparse ? 1 : 0;  // (MQ_NSW should drop to 18 to keep 20 warps)
#else
constexpr int kPF = 0;
#endif
static_assert(!(kXDirect || kXBDirect) || ((MQ_NGW == 0 || kSparse) && !kPhased && !kScatter && !kSplit),
              "direct x/xbar loads: default (fused) mode only");        // gathered values staged per round (phased mode)

template <int ETILE, int RTILE, bool HASC>
struct TileLayout {
    // one stage (every region 16-byte aligned for the bulk copies):
    // u, x, xbar, c f64 [ETILE+2] | col i32 [ETILE+4] | row_ptr i64 [RTILE+4] | w f64 [RTILE+2]
    // (c = x - tau p[col] is written by the gather warps, not by TMA)
    static constexpr int kU = 0;
    static constexpr int kX = kU + (ETILE + 2) * 8;
    static constexpr int kXB = kX + (kXDirect ? 0 : (ETILE + 2) * 8);
    static constexpr int kC = kXB + (kXBDirect ? 0 : (ETILE + 2) * 8);
    static constexpr int kCol = kC + (HASC ? (ETILE + 2) * 8 : 0);
    static constexpr int kTp = kCol + (ETILE + 4) * 4;       // tpos (scatter) / bpos (bucket)
    static constexpr int kRp = kTp + ((kScatter || kBucket) ? (ETILE + 4) * 4 : 0);
    static constexpr int kW = kRp + (RTILE + 4) * 8;
    static constexpr int kS = kW + (RTILE + 2) * 8;  // srow: warm-start utilities
    static constexpr int kF = kS + (RTILE + 2) * 8;  // x > 0 flags (sparse iterate), u8
    static constexpr int kStage = (kF + (kSparse ? ETILE + 32 : 0) + 127) / 128 * 128;
    static_assert(kX % 16 == 0 && kCol % 16 == 0 && kRp % 16 == 0 && kW % 16 == 0 && kS % 16 == 0 &&
                      kF % 16 == 0,
                  "bulk-copy destinations must be 16-byte aligned");
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes,
                                              uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// coherent load that does not allocate in L1 (streams read once by this thread)
__device__ __forceinline__ double ld_na(const double *a) {
    double v;
    asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_flag(uint8_t *p, bool v) {
    asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"((int)v) : "memory");
}
// fire-and-forget float add (one writer per address and iteration: the
// result is the plain rounded sum, deterministic)
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// scatter store kept in L2 until its 32-byte sector is complete
__device__ __forceinline__ void st_keep(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// 16-byte-aligned superset of [first, first+count) elements of size S
template <int S>
__device__ __forceinline__ void aligned_span(const void *base, int64_t first, int64_t count,
                                             const unsigned char **src, uint32_t *bytes) {
    const uint32_t d = (uint32_t)((first * S) & 15);
    *src = reinterpret_cast<const unsigned char *>(base) + first * S - d;
    *bytes = (uint32_t)((d + count * S + 15) & ~(int64_t)15);
}

#ifdef MQ_CS_PERWARP
constexpr bool kCsPerWarp = true;     // each column-sum warp publishes its progress
#else
constexpr bool kCsPerWarp = false;    // one publication per CTA
#endif
#ifndef MQ_CS_CAP
#define MQ_CS_CAP 4096
#endif
constexpr int kCsCap = MQ_CS_CAP;         // staged bperm entries per CTA (CTA-level column sums)
constexpr int kCsChunk = MQ_CS_CHUNK; // bperm entries per staged column-sum chunk (per warp)
constexpr int kWCols = MQ_NCW >= 4 ? 320 : 600;  // goods per column-sum warp
constexpr int kClaim = MQ_CLAIM;      // tiles claimed per atomic by a producer
constexpr int kRegPer = MQ_REG_PER;   // entries per lane kept in registers
#ifdef MQ_TRIVIAL_SOLVE
constexpr bool kTrivial = true;       // bandwidth experiments only
#else
constexpr bool kTrivial = false;
#endif
constexpr int kCsCols = 1152;         // goods per CTA (>= QMAX * NCW * 32)
#ifndef MQ_BK_CHUNK
#define MQ_BK_CHUNK 1024
#endif
constexpr int kBkChunk = MQ_BK_CHUNK; // bucket entries per staged chunk (bucket mode)
constexpr int kCsQ = MQ_CSQ, kCsU = MQ_CSU;  // goods x gathers in flight per column-sum thread
constexpr int64_t kLag = MQ_LAG;      // solver blocks ahead of the slowest column-sum CTA
constexpr int64_t kSpinLimit = 4000000000ll;  // ~2 s of clock64: a stalled block is a fault

// named barrier among the NCW column-sum warps (id 1; __syncthreads uses 0)
__device__ __forceinline__ void colsum_sync(int ncw) {
    asm volatile("bar.sync 1, %0;" ::"r"(ncw * 32) : "memory");
}

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// spin (one lane) until *ctr >= target with relaxed loads (an acquiring load
// would invalidate L1 on every poll), then one acquire fence if the caller
// reads data published before the counter; a stall past kSpinLimit is a fault
__device__ __forceinline__ void wait_counter(const int *ctr, int target, int64_t *faults,
                                             bool acquire) {
    if (ld_relaxed(ctr) < target) {
        const long long t0 = clock64();
        while (ld_relaxed(ctr) < target) {
            __nanosleep(200);
            if (clock64() - t0 > kSpinLimit) {
                atomicAdd((unsigned long long *)faults, 1ull << 40);
                break;
            }
        }
    }
    if (acquire) __threadfence();
}


// ---- phased column sums -------------------------------------------------
// Participants: the NSW solver warps and the NCW column-sum warps of the CTA
// (pt = 0..NP-1).  After every CTA has solved block b (grid barrier), the
// participants gather the block's x values of the CTA's goods from L2 into
// shared memory in chunks (independent loads), then each thread adds its
// goods' values in ascending row order (deterministic).
__device__ __forceinline__ void phase_sync(int np) {
    asm volatile("bar.sync 1, %0;" ::"r"(np) : "memory");
}

template <int QM>
__device__ __forceinline__ void phased_gather(const mq_market &mk, const mq_state &st, int64_t b,
                                              int pt, int np, int64_t j_lo, int nc,
                                              double *sval, double (&acc)[QM]) {
    phase_sync(np);  // this CTA has solved all its tiles of block b
    if (pt == 0) {
        int *gb = st.blk_done + mk.nblk + b;
        __threadfence();
        atomicAdd(gb, 1);
        wait_counter(gb, (int)gridDim.x, st.faults, true);
    }
    phase_sync(np);  // every CTA has: block b's x is complete
    if (nc == 0) return;
    const int64_t row0 = b * mk.m;
    const int64_t r_lo = __ldg(mk.bptr + row0 + j_lo), r_hi = __ldg(mk.bptr + row0 + j_lo + nc);
    int32_t lo[QM], hi[QM];
#pragma unroll
    for (int q = 0; q < QM; ++q) {
        const int jl = pt + q * np;
        lo[q] = hi[q] = 0;
        if (jl < nc) {
            lo[q] = __ldg(mk.bptr + row0 + j_lo + jl);
            hi[q] = __ldg(mk.bptr + row0 + j_lo + jl + 1);
        }
    }
    for (int64_t c0 = r_lo; c0 < r_hi; c0 += kPhChunk) {
        const int len = (int)(r_hi - c0 < kPhChunk ? r_hi - c0 : kPhChunk);
        for (int t0 = pt; t0 < len; t0 += np * 4) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * np;
                v[u] = t < len ? __ldcg(st.x + __ldcs(mk.bperm + c0 + t)) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * np;
                if (t < len) sval[t] = v[u];
            }
        }
        phase_sync(np);
        const int64_t c1 = c0 + len;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            int64_t t = lo[q] > c0 ? lo[q] : c0;
            const int64_t e = hi[q] < c1 ? hi[q] : c1;
            double a = acc[q];
            for (; t < e; ++t) a += sval[t - c0];
            acc[q] = a;
        }
        phase_sync(np);
    }
}

// Warps 0..NSW-1 solve rows, warp NSW produces (TMA), warps NSW+1..NSW+NGW
// gather prices (c = x - tau p[col] for the whole tile), the last NCW warps
// sum columns.  full[s]: stage s has landed; ready[s]: its c is computed;
// empty[s]: every solver warp is done with it.  Solver warps claim row pairs
// from a shared counter, so no solver waits for another inside a tile, and
// they never touch global memory before their stores.
template <int G, int NSW, int NGW, int NCW, int ETILE, int RTILE, int NSTAGE, int QMAX>
__global__ void __launch_bounds__((NSW + NGW + NCW + 1 + kPF) * 32, 1)
primal_fused_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out,
                    int write_cs, int64_t tile_lo, int64_t tile_hi, int *tile_ctr) {
    // c (gather warps) is written over the staged x, or into its own region
    // when x is not staged (sparse iterate)
    using L = TileLayout<ETILE, RTILE, (NGW > 0 && kXDirect)>;
    MQ_PROF_DECL();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NSTAGE * L::kStage);
    uint64_t *empty = full + NSTAGE;
    uint64_t *ready = empty + NSTAGE;
    int64_t *stile = reinterpret_cast<int64_t *>(ready + NSTAGE);  // tile held by each stage
    int64_t *smeta = stile + NSTAGE;                               // its r0, r1, e0 per stage
    int *claim = reinterpret_cast<int *>(smeta + 3 * NSTAGE);
    // column-sum staging (16-byte aligned: TMA bulk-copy destination)
    int32_t *cstage = reinterpret_cast<int32_t *>(
        (reinterpret_cast<uintptr_t>(claim + 4 * NSTAGE) + 127) & ~uintptr_t(127));
    constexpr int GPW = 32 / G;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, wl = tid & 31;
    const int64_t tpb_all = mk.tiles_per_block;  // tiles per block (all CTAs)

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NSW);
            mbar_init(&ready[s], NGW > 0 ? NGW : 1);
        }
        claim[2 * NSTAGE] = 0;  // producer done (read by the x-prefetch warp)
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == NSW) {  // ---------------------------------------- producer
        if (wl == 0) {
            const uint64_t pol = policy_evict_first();
            if (kPhased) {
                // blocks of tiles one after the other; within a block tiles are
                // claimed dynamically; a marker stage (-2) ends each block
                int64_t j = 0;
                for (int64_t bk = 0; bk <= mk.nblk; ++bk) {
                    const bool last = bk == mk.nblk;
                    const int64_t lo = bk * tpb_all;
                    const int64_t hi = last ? lo : (lo + tpb_all < mk.ntiles ? lo + tpb_all : mk.ntiles);
                    int *ctr = st.blk_done + (last ? 0 : bk);
                    int64_t batch = last ? hi : lo + atomicAdd(ctr, kClaim);
                    int bpos = 0;
                    for (;;) {
                        int64_t k = hi;
                        if (!last) {
                            if (bpos == kClaim) {
                                batch = lo + atomicAdd(ctr, kClaim);
                                bpos = 0;
                            }
                            k = batch + bpos++;
                        }
                        longlong2 m01 = {0, 0}, m23 = {0, 0};
                        if (k < hi) {
                            const longlong2 *tp = reinterpret_cast<const longlong2 *>(mk.tiles + 4 * k);
                            m01 = __ldg(tp);
                            m23 = __ldg(tp + 1);
                        }
                        const int s = (int)(j % NSTAGE);
                        if (j >= NSTAGE) mbar_wait(&empty[s], (uint32_t)(((j / NSTAGE) - 1) & 1));
                        ++j;
                        claim[s] = 0;
                        claim[NSTAGE + s] = 0;
                        if (k >= hi) {  // end of block (-2) or of the launch (-1)
                            stile[s] = last ? -1 : -2;
                            mbar_expect_tx(&full[s], 0);
                            break;
                        }
                        const int64_t r0 = m01.x, r1 = m01.y, e0 = m23.x, cnt = m23.y - m23.x;
                        stile[s] = k;
                        smeta[3 * s] = r0;
                        smeta[3 * s + 1] = r1;
                        smeta[3 * s + 2] = e0;
                        unsigned char *base = smem + s * L::kStage;
                        const unsigned char *src_rp, *src_w, *src_u, *src_x, *src_xb, *src_c;
                        uint32_t brp, bw, b8 = 0, b4 = 0;
                        aligned_span<8>(mk.row_ptr, r0, r1 - r0 + 1, &src_rp, &brp);
                        aligned_span<8>(mk.w, r0, r1 - r0, &src_w, &bw);
                        aligned_span<8>(mk.u, e0, cnt, &src_u, &b8);
                        aligned_span<8>(st.x, e0, cnt, &src_x, &b8);
                        aligned_span<8>(st.xbar, e0, cnt, &src_xb, &b8);
                        aligned_span<4>(mk.col, e0, cnt, &src_c, &b4);
                        const unsigned char *src_s;
                        aligned_span<8>(st.srow, r0, r1 - r0, &src_s, &bw);
                        mbar_expect_tx(&full[s], brp + 2 * bw + (cnt > 0 ? 3 * b8 + b4 : 0));
                        bulk_g2s(base + L::kRp, src_rp, brp, &full[s]);
                        bulk_g2s(base + L::kW, src_w, bw, &full[s]);
                        bulk_g2s(base + L::kS, src_s, bw, &full[s]);
                        if (cnt > 0) {
                            bulk_g2s_hint(base + L::kU, src_u, b8, &full[s], pol);
                            bulk_g2s(base + L::kX, src_x, b8, &full[s]);
                            bulk_g2s_hint(base + L::kXB, src_xb, b8, &full[s], pol);
                            bulk_g2s_hint(base + L::kCol, src_c, b4, &full[s], pol);
                        }
                    }
                }
                return;
            }
            // tiles are claimed dynamically (global counter, kClaim at a time) so
            // that every block of tiles completes with little skew across CTAs;
            // the next tile's claim and metadata are fetched one step ahead so
            // the producer never waits on a dependent global load
            int64_t batch = tile_lo + atomicAdd(tile_ctr, kClaim);
            int bpos = 0;
            auto next_tile = [&]() -> int64_t {
                if (bpos == kClaim) {
                    batch = tile_lo + atomicAdd(tile_ctr, kClaim);
                    bpos = 0;
                }
                return batch + bpos++;
            };
            auto load_meta = [&](int64_t k, longlong2 &a01, longlong2 &a23) {
                if (k < tile_hi) {
                    const longlong2 *tp = reinterpret_cast<const longlong2 *>(mk.tiles + 4 * k);
                    a01 = __ldg(tp);
                    a23 = __ldg(tp + 1);
                }
            };
            int64_t kn = next_tile();
            longlong2 mn01 = {0, 0}, mn23 = {0, 0};
            load_meta(kn, mn01, mn23);
            int64_t j = 0;
            for (;; ++j) {
                const int s = (int)(j % NSTAGE);
                const int64_t k = kn;
                const longlong2 m01 = mn01, m23 = mn23;
                if (k < tile_hi) {
                    kn = next_tile();
                    load_meta(kn, mn01, mn23);
                }
                if (j >= NSTAGE) {
                    MQ_T0();
                    mbar_wait(&empty[s], (uint32_t)(((j / NSTAGE) - 1) & 1));
                    MQ_T1(2);
                }
                claim[s] = 0;
                claim[NSTAGE + s] = 0;  // solver warps done with this use
                if (k >= tile_hi) {  // sentinel: consumers leave
                    stile[s] = -1;
                    mbar_expect_tx(&full[s], 0);
                    *reinterpret_cast<volatile int *>(&claim[2 * NSTAGE]) = 1;
                    break;
                }
                const int64_t r0 = m01.x, r1 = m01.y, e0 = m23.x, cnt = m23.y - m23.x;
                stile[s] = k;
                smeta[3 * s] = r0;
                smeta[3 * s + 1] = r1;
                smeta[3 * s + 2] = e0;
                // no proxy fence here: a consumer that wrote this stage's shared
                // memory fenced itself before releasing it (a fence on this
                // path would serialise the bulk copies)
                unsigned char *base = smem + s * L::kStage;
                const unsigned char *src_rp, *src_w, *src_u, *src_x, *src_xb, *src_c;
                uint32_t brp, bw, b8 = 0, b4 = 0;
                aligned_span<8>(mk.row_ptr, r0, r1 - r0 + 1, &src_rp, &brp);
                aligned_span<8>(mk.w, r0, r1 - r0, &src_w, &bw);
                aligned_span<8>(mk.u, e0, cnt, &src_u, &b8);
                aligned_span<8>(st.x, e0, cnt, &src_x, &b8);
                aligned_span<8>(st.xbar, e0, cnt, &src_xb, &b8);
                aligned_span<4>(mk.col, e0, cnt, &src_c, &b4);
                const unsigned char *src_tp = nullptr;
                if (kScatter || kBucket)
                    aligned_span<4>(kScatter ? mk.tpos : mk.bpos, e0, cnt, &src_tp, &b4);
                constexpr int n8 = 1 + (kXDirect ? 0 : 1) + (kXBDirect ? 0 : 1);
                const unsigned char *src_s;
                aligned_span<8>(st.srow, r0, r1 - r0, &src_s, &bw);
                const unsigned char *src_f = nullptr;
                uint32_t b1 = 0;
                if (kSparse) aligned_span<1>(st.xflag, e0, cnt, &src_f, &b1);
                mbar_expect_tx(&full[s], brp + 2 * bw +
                                             (cnt > 0 ? n8 * b8 + ((kScatter || kBucket) ? 2 : 1) * b4 + b1
                                                      : 0));
                bulk_g2s(base + L::kRp, src_rp, brp, &full[s]);
                bulk_g2s(base + L::kW, src_w, bw, &full[s]);
                bulk_g2s(base + L::kS, src_s, bw, &full[s]);
                if (cnt > 0) {
                    bulk_g2s_hint(base + L::kU, src_u, b8, &full[s], pol);
                    if (kSparse) bulk_g2s_hint(base + L::kF, src_f, b1, &full[s], pol);
                    else if (kXDirect) prefetch_l2(src_x, b8);
                    else bulk_g2s(base + L::kX, src_x, b8, &full[s]);
                    if (kSparse) {
                    } else if (kXBDirect) prefetch_l2(src_xb, b8);
                    else bulk_g2s_hint(base + L::kXB, src_xb, b8, &full[s], pol);
                    bulk_g2s_hint(base + L::kCol, src_c, b4, &full[s], pol);
                    if (kScatter || kBucket) bulk_g2s_hint(base + L::kTp, src_tp, b4, &full[s], pol);
                }
            }

        }
        return;
    }

    const double tau = st.steps[0];
    if (NGW > 0 && warp > NSW && warp <= NSW + NGW) {  // -------------- price gather
        const int gt = tid - (NSW + 1) * 32;
        for (int64_t j = 0;; ++j) {
            const int s = (int)(j % NSTAGE);
            mbar_wait(&full[s], (uint32_t)((j / NSTAGE) & 1));
            const int64_t k = stile[s];
            if (k >= 0) {
                unsigned char *base = smem + s * L::kStage;
                const int64_t r0 = smeta[3 * s];
                const int lr = (int)(((r0 * 8) & 15) >> 3);
                const int64_t *srp = reinterpret_cast<const int64_t *>(base + L::kRp) + lr;
                const int nrows = (int)(smeta[3 * s + 1] - r0);
                const int64_t e0 = srp[0];
                const int cnt = (int)(srp[nrows] - e0);
                const int d8 = (int)(((e0 * 8) & 15) >> 3), d4 = (int)(((e0 * 4) & 15) >> 2);
                // c = x - tau p[col] replaces x in the stage (the solvers read
                // c and the warm start srow; x itself is not needed again)
                double *sx = reinterpret_cast<double *>(base + L::kX) + d8;
                double *sc = kXDirect ? reinterpret_cast<double *>(base + L::kC) + d8 : sx;
                const int32_t *scol = reinterpret_cast<const int32_t *>(base + L::kCol) + d4;
                const uint8_t *sfl = reinterpret_cast<const uint8_t *>(base + L::kF) + (int)(e0 & 15);
                constexpr int U = 8;
                for (int t0 = gt; t0 < cnt; t0 += NGW * 32 * U) {
                    double pv[U];
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int t = t0 + q * NGW * 32;
                        pv[q] = t < cnt ? ld_price(st.p + scol[t]) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int t = t0 + q * NGW * 32;
                        if (t < cnt) {
                            const double xe = !kXDirect ? sx[t]
                                              : kSparse ? (sfl[t] ? ld_na(st.x + e0 + t) : 0.0)
                                                        : ld_na(st.x + e0 + t);
                            sc[t] = xe - tau * pv[q];
                            if (x_prev_out) x_prev_out[e0 + t] = xe;
                        }
                    }
                }
            }
            fence_proxy_async();  // generic writes before the stage's next bulk refill
            __syncwarp();
            if (wl == 0) mbar_arrive(&ready[s]);
            if (k < 0) break;
        }
        return;
    }
#ifdef MQ_NO_COLSUM  // timing experiment only: solver without column sums
    if (warp > NSW + NGW) return;
#endif
    if ((kScatter || kSplit) && warp > NSW + NGW) return;  // column sums run after the kernel
    // phased mode: goods of this CTA and the participant layout
    constexpr int NP = (NSW + NCW) * 32;
    constexpr int PQ = 2048 / NP + 1;  // goods per participant (<= 2048 goods per CTA)
    const int64_t ph_per = (mk.m + gridDim.x - 1) / gridDim.x;
    const int64_t ph_lo = blockIdx.x * ph_per;
    const int ph_nc = (int)(ph_lo + ph_per < mk.m ? ph_per : (mk.m > ph_lo ? mk.m - ph_lo : 0));
    double *ph_sval = reinterpret_cast<double *>(cstage);
    double ph_acc[PQ];
#pragma unroll
    for (int q = 0; q < PQ; ++q) ph_acc[q] = 0.0;
    if (kPhased && warp > NSW + NGW) {  // column-sum warps: gather phases only
        const int pt = tid - 32 * (1 + NGW);
        for (int64_t bk = 0; bk < mk.nblk; ++bk)
            phased_gather<PQ>(mk, st, bk, pt, NP, ph_lo, ph_nc, ph_sval, ph_acc);
        if (write_cs) {
#pragma unroll
            for (int q = 0; q < PQ; ++q) {
                const int jl = pt + q * NP;
                if (jl < ph_nc) st.cs[ph_lo + jl] = ph_acc[q];
            }
        }
        return;
    }
    if (kPF && warp == NSW + NGW + NCW + 1) {  // ------------- x prefetch (sparse)
        // Follows the full barriers only (never holds a stage): for each
        // staged tile, the flagged entries' x go to L2 with prefetch hints.
        // A late look at a refilled stage only prefetches other valid x.
        for (int64_t j = 0;; ++j) {
            const int s = (int)(j % NSTAGE);
            const uint32_t par = (uint32_t)((j / NSTAGE) & 1);
            bool ok = false;
            for (;;) {  // bounded: stop once the producer has posted the sentinel
                ok = __shfl_sync(MQ_FULL, (int)mbar_test(&full[s], par), 0) != 0;
                if (ok || *reinterpret_cast<volatile int *>(&claim[2 * NSTAGE])) break;
                __nanosleep(64);
            }
            if (!ok) break;
            const int64_t k = stile[s];
            if (k < 0) break;
            // the tile's extent from global memory (consistent even if this
            // warp is late and the stage already holds a newer tile)
            const int64_t e0 = __ldg(mk.tiles + 4 * k + 2);
            const int64_t cnt = __ldg(mk.tiles + 4 * k + 3) - e0;
            const unsigned char *fl = smem + s * L::kStage + L::kF;
            const int lead = (int)(e0 & 15);
            int nw = (lead + (int)cnt + 15) >> 4;
            nw = nw < (ETILE + 32) / 16 ? nw : (ETILE + 32) / 16;
            for (int w16 = wl; w16 < nw; w16 += 32) {
                const uint4 v = reinterpret_cast<const uint4 *>(fl)[w16];
                const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int by = 0; by < 4; ++by) {
                        const int t = w16 * 16 + q * 4 + by - lead;
                        if (((wd[q] >> (8 * by)) & 0xffu) && t >= 0 && t < cnt && e0 + t < mk.nnz)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(st.x + e0 + t));
                    }
                }
            }
        }
        return;
    }
    if (kAtomic && warp > NSW + NGW) return;
    if (kBucket && warp > NSW + NGW) {  // ---------------- column sums (buckets)
        // The CTA's NCW column-sum warps own goods [j_lo, j_hi).  The solvers
        // stored every x of block b at its bpos slot of bucket b % kLag, so the
        // owned goods' values of the block are one contiguous bucket range,
        // in good order and ascending rows inside a good.  Once every CTA has
        // solved the block, the range streams through shared memory in
        // chunks (TMA bulk copies from L2, double-buffered), and each thread
        // adds its goods' values in order (deterministic, the reference's
        // column_sums order).
        const int ct = tid - (NSW + NGW + 1) * 32;
        const int64_t per = (mk.m + gridDim.x - 1) / gridDim.x;
        const int64_t j_lo = blockIdx.x * per;
        const int64_t j_hi = j_lo + per < mk.m ? j_lo + per : mk.m;
        const int nc = (int)(j_hi > j_lo ? j_hi - j_lo : 0);
        int32_t *sbptr = cstage;                                             // [kCsCols + 8]
        double *sval = reinterpret_cast<double *>(cstage + kCsCols + 8);     // [2][kBkChunk + 4]
        uint64_t *cbar = reinterpret_cast<uint64_t *>(sval + 2 * (kBkChunk + 4));  // chunks 0/1, bptr
        if (ct == 0) {
            mbar_init(&cbar[0], 1);
            mbar_init(&cbar[1], 1);
            mbar_init(&cbar[2], 1);
            mbar_fence_init();
        }
        colsum_sync(NCW);
        if (nc == 0) {  // no goods here: still publish progress for the throttle
            if (ct == 0)
                for (int64_t b = 0; b < mk.nblk; ++b) atomicAdd(st.blk_done + mk.nblk + b, 1);
            return;
        }
        auto stage_ptr = [&](int64_t b) {  // bptr slice of the owned goods (one thread)
            const unsigned char *src;
            uint32_t bytes;
            aligned_span<4>(mk.bptr, b * mk.m + j_lo, nc + 1, &src, &bytes);
            mbar_expect_tx(&cbar[2], bytes);
            bulk_g2s(sbptr, src, bytes, &cbar[2]);
        };
        double acc[QMAX];
#pragma unroll
        for (int q = 0; q < QMAX; ++q) acc[q] = 0.0;
        uint32_t use0 = 0, use1 = 0, pphase = 0;
        if (ct == 0) stage_ptr(0);
        for (int64_t b = 0; b < mk.nblk; ++b) {
            const int64_t kb0 = b * tpb_all;
            const int target = (int)((kb0 + tpb_all < mk.ntiles ? kb0 + tpb_all : mk.ntiles) - kb0);
            {
                MQ_T0();
                if (ct == 0) wait_counter(st.blk_done + b, target, st.faults, true);
                colsum_sync(NCW);
                if (ct == 0) MQ_T1(3);
            }
            MQ_T0();
            mbar_wait(&cbar[2], pphase);
            pphase ^= 1u;
            const int32_t *bp = sbptr + (int)((((b * mk.m + j_lo) * 4) & 15) >> 2);
            const int64_t base = __ldg(mk.bptr + b * mk.m);  // the block's first position
            const int64_t rlo = bp[0] - base, rhi = bp[nc] - base;
            const double *slot = st.bucket + (b % kLag) * mk.bcap;
            const int64_t nch = (rhi - rlo + kBkChunk - 1) / kBkChunk;
            auto issue = [&](int64_t g) {  // one thread
                const int buf = (int)(g & 1);
                const int64_t c0 = rlo + g * kBkChunk;
                const int64_t c1 = c0 + kBkChunk < rhi ? c0 + kBkChunk : rhi;
                const unsigned char *src;
                uint32_t bytes;
                aligned_span<8>(slot, c0, c1 - c0, &src, &bytes);
                mbar_expect_tx(&cbar[buf], bytes);
                bulk_g2s(sval + buf * (kBkChunk + 4), src, bytes, &cbar[buf]);
            };
            if (ct == 0) {
                fence_proxy_async_global();
                if (nch > 0) issue(0);
                if (nch > 1) issue(1);
            }
            for (int64_t g = 0; g < nch; ++g) {
                const int buf = (int)(g & 1);
                mbar_wait(&cbar[buf], (buf ? use1 : use0) & 1u);
                if (buf) ++use1; else ++use0;
                const int64_t c0 = rlo + g * kBkChunk;
                const int64_t c1 = c0 + kBkChunk < rhi ? c0 + kBkChunk : rhi;
                const double *sv = sval + buf * (kBkChunk + 4) + (int)(c0 & 1) - c0;
#pragma unroll
                for (int q = 0; q < QMAX; ++q) {
                    const int jl = ct + q * NCW * 32;
                    if (jl >= nc) break;
                    int64_t t = bp[jl] - base, e = bp[jl + 1] - base;
                    t = t > c0 ? t : c0;
                    e = e < c1 ? e : c1;
                    double a = acc[q];
                    for (; t < e; ++t) a += sv[t];
                    acc[q] = a;
                }
                colsum_sync(NCW);  // the chunk buffer is consumed
                if (ct == 0 && g + 2 < nch) {
                    fence_proxy_async();
                    issue(g + 2);
                }
            }
            colsum_sync(NCW);  // bp[] reads done
            if (ct == 0) {
                MQ_T1(4);
                atomicAdd(st.blk_done + mk.nblk + b, 1);  // block b summed: its bucket is free
                if (b + 1 < mk.nblk) {
                    fence_proxy_async();
                    stage_ptr(b + 1);
                }
            }
        }
        if (write_cs) {
#pragma unroll
            for (int q = 0; q < QMAX; ++q) {
                const int jl = ct + q * NCW * 32;
                if (jl < nc) st.cs[j_lo + jl] = acc[q];
            }
        }
        return;
    }
#ifdef MQ_CS_PERWARP
    if (warp > NSW + NGW) {  // ---------------------------------- column sums
        // Each column-sum warp owns a contiguous range of goods and runs its
        // own pipeline (no cross-warp barriers): per block, its slice of the
        // schedule is contiguous in bperm and is staged in chunks with TMA
        // (double-buffered, issued before the block is even solved); once
        // every CTA has solved the block, the warp gathers a chunk's x values
        // from L2 (kCsU independent loads per lane in flight) into shared
        // memory, then each lane adds its goods' values in ascending row
        // order (deterministic).
        const int cw = warp - NSW - NGW - 1;
        const int64_t per = (mk.m + gridDim.x - 1) / gridDim.x;
        const int64_t c_lo = blockIdx.x * per;
        const int64_t c_hi = c_lo + per < mk.m ? c_lo + per : mk.m;
        const int64_t cn = c_hi > c_lo ? c_hi - c_lo : 0;
        const int64_t wper = (cn + NCW - 1) / NCW;
        const int64_t j_lo = c_lo + cw * wper;
        const int64_t j_hi = j_lo + wper < c_hi ? j_lo + wper : c_hi;
        const int nc = (int)(j_hi > j_lo ? j_hi - j_lo : 0);
        // per-warp shared layout:
        // sperm[2][kCsChunk+8] | sbptr[2][kWCols+8] | sval[kCsChunk] | meta[2][4] | cbar[2]
        constexpr int kWarpStage = (2 * (kCsChunk + 8) + 2 * (kWCols + 8)) * 4 + kCsChunk * 8 +
                                   8 * 8 + 2 * 8;
        unsigned char *wbase = reinterpret_cast<unsigned char *>(cstage) +
                               cw * ((kWarpStage + 127) / 128 * 128);
        int32_t *sperm0 = reinterpret_cast<int32_t *>(wbase);
        int32_t *sbptr0 = sperm0 + 2 * (kCsChunk + 8);
        double *sval = reinterpret_cast<double *>(sbptr0 + 2 * (kWCols + 8));
        int64_t *meta = reinterpret_cast<int64_t *>(sval + kCsChunk);
        uint64_t *cbar = reinterpret_cast<uint64_t *>(meta + 8);
        if (wl == 0) {
            mbar_init(&cbar[0], 1);
            mbar_init(&cbar[1], 1);
            mbar_fence_init();
        }
        __syncwarp();
        if (nc == 0) {  // no goods here: still publish progress for the throttle
            if (wl == 0)
                for (int64_t bb = 0; bb < mk.nblk; ++bb) atomicAdd(st.blk_done + mk.nblk + bb, 1);
            return;
        }
        // staging cursor (lane 0 only)
        int64_t g_stage = 0, sb = 0, sc0 = -1, srhi = 0;
        auto stage_next = [&]() {
            if (sb >= mk.nblk) return;
            const int buf = (int)(g_stage & 1);
            const bool first = sc0 < 0;
            const int64_t row0 = sb * mk.m;
            if (first) {
                sc0 = __ldg(mk.bptr + row0 + j_lo);
                srhi = __ldg(mk.bptr + row0 + j_hi);
            }
            const int64_t c1 = sc0 + kCsChunk < srhi ? sc0 + kCsChunk : srhi;
            meta[4 * buf] = sc0;
            meta[4 * buf + 1] = c1;
            meta[4 * buf + 2] = srhi;
            const unsigned char *srcp, *srcb;
            uint32_t bp = 0, bb = 0;
            if (c1 > sc0) aligned_span<4>(mk.bperm, sc0, c1 - sc0, &srcp, &bp);
            if (first) aligned_span<4>(mk.bptr, row0 + j_lo, nc + 1, &srcb, &bb);
            mbar_expect_tx(&cbar[buf], bp + bb);
            if (c1 > sc0) bulk_g2s(sperm0 + buf * (kCsChunk + 8), srcp, bp, &cbar[buf]);
            if (first) bulk_g2s(sbptr0 + (int)(sb & 1) * (kWCols + 8), srcb, bb, &cbar[buf]);
            ++g_stage;
            if (c1 >= srhi) {
                ++sb;
                sc0 = -1;
            } else {
                sc0 = c1;
            }
        };
        double acc[QMAX];
#pragma unroll
        for (int q = 0; q < QMAX; ++q) acc[q] = 0.0;
        if (wl == 0) {
            stage_next();
            stage_next();
        }
        int64_t g = 0;
        for (int64_t blk = 0; blk < mk.nblk; ++blk) {
            const int64_t kb0 = blk * tpb_all;
            const int target = (int)((kb0 + tpb_all < mk.ntiles ? kb0 + tpb_all : mk.ntiles) - kb0);
            {
                MQ_T0();
#ifndef MQ_CS_NOWAIT
                if (wl == 0) wait_counter(st.blk_done + blk, target, st.faults, true);
#endif
                __syncwarp();
                if (wl == 0) MQ_T1(3);
            }
            MQ_T0();
            const int64_t row0 = blk * mk.m;
            const int32_t *sbp = sbptr0 + (int)(blk & 1) * (kWCols + 8) +
                                 (int)((((row0 + j_lo) * 4) & 15) >> 2);
            for (;;) {
                const int buf = (int)(g & 1);
                mbar_wait(&cbar[buf], (uint32_t)((g >> 1) & 1));
                const int64_t c0 = meta[4 * buf], c1 = meta[4 * buf + 1], rhi = meta[4 * buf + 2];
                const int32_t *sp = sperm0 + buf * (kCsChunk + 8) + (int)(((c0 * 4) & 15) >> 2);
                const int len = (int)(c1 - c0);
                for (int t0 = wl; t0 < len; t0 += 32 * kCsU) {
                    double v[kCsU];
#pragma unroll
                    for (int u = 0; u < kCsU; ++u) {
                        const int t = t0 + u * 32;
                        v[u] = t < len ? __ldcg(st.x + sp[t]) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kCsU; ++u) {
                        const int t = t0 + u * 32;
                        if (t < len) sval[t] = v[u];
                    }
                }
                __syncwarp();  // values of the chunk are in shared memory
#pragma unroll
                for (int q = 0; q < QMAX; ++q) {
                    const int jl = wl + q * 32;
                    if (jl < nc) {
                        int64_t lo = sbp[jl], hi = sbp[jl + 1];
                        lo = lo > c0 ? lo : c0;
                        hi = hi < c1 ? hi : c1;
                        double a = acc[q];
                        for (int64_t t = lo; t < hi; ++t) a += sval[t - c0];
                        acc[q] = a;
                    }
                }
                __syncwarp();  // chunk consumed: its buffers may be restaged
                ++g;
                if (wl == 0) stage_next();
                if (c1 >= rhi) break;
            }
            if (wl == 0) {
                MQ_T1(4);
                atomicAdd(st.blk_done + mk.nblk + blk, 1);  // block gathered by this warp
            }
        }
        if (write_cs) {
#pragma unroll
            for (int q = 0; q < QMAX; ++q) {
                const int jl = wl + q * 32;
                if (jl < nc) st.cs[j_lo + jl] = acc[q];
            }
        }
        return;
    }

#else
    if (warp > NSW + NGW) {  // ---------------------------------- column sums
        // The CTA's NCW column-sum warps own goods [j_lo, j_hi); thread ct owns
        // j_lo + ct + q*NCW*32.  Per block, one thread stages the block's
        // schedule slice (bptr for the owned goods, their bperm range) into
        // shared memory with TMA bulk copies, issued before the block is even
        // solved; once every CTA has solved the block, each thread gathers its
        // goods' x values from L2 and adds them in ascending row order.
        const int ct = tid - (NSW + NGW + 1) * 32;
        const int64_t per = (mk.m + gridDim.x - 1) / gridDim.x;
        const int64_t j_lo = blockIdx.x * per;
        const int64_t j_hi = j_lo + per < mk.m ? j_lo + per : mk.m;
        const int nc = (int)(j_hi > j_lo ? j_hi - j_lo : 0);
        int32_t *sperm = cstage;
        int32_t *sbptr = cstage + kCsCap;
        int64_t *meta = reinterpret_cast<int64_t *>(sbptr + kCsCols + 8);  // rlo, rhi, lead
        uint64_t *cbar = reinterpret_cast<uint64_t *>(meta + 4);
        if (ct == 0) {
            mbar_init(cbar, 1);
            mbar_fence_init();
        }
        colsum_sync(NCW);
        if (nc == 0) {  // no goods here: still publish progress for the throttle
            if (ct == 0)
                for (int64_t b = 0; b < mk.nblk; ++b) atomicAdd(st.blk_done + mk.nblk + b, 1);
            return;
        }
        uint32_t cphase = 0;
        // stage chunk [c0, c1) of block b's bperm range (+ the bptr slice on c0 == rlo)
        auto stage = [&](int64_t b, int64_t c0, bool with_ptr) {
            const unsigned char *src;
            uint32_t bytes_p = 0, bytes_b = 0;
            const int64_t row0 = b * mk.m;
            if (with_ptr) {
                const int64_t rlo = __ldg(mk.bptr + row0 + j_lo), rhi = __ldg(mk.bptr + row0 + j_hi);
                meta[0] = rlo;
                meta[1] = rhi;
                c0 = rlo;
            }
            const int64_t c1 = c0 + kCsCap - 4 < meta[1] ? c0 + kCsCap - 4 : meta[1];
            meta[2] = c0;
            meta[3] = c1;
            const unsigned char *srcp;
            aligned_span<4>(mk.bperm, c0, c1 - c0, &srcp, &bytes_p);
            if (with_ptr) aligned_span<4>(mk.bptr, row0 + j_lo, nc + 1, &src, &bytes_b);
            mbar_expect_tx(cbar, (c1 > c0 ? bytes_p : 0) + bytes_b);
            if (c1 > c0) bulk_g2s(sperm, srcp, bytes_p, cbar);
            if (with_ptr) bulk_g2s(sbptr, src, bytes_b, cbar);
        };
        double acc[QMAX];
#pragma unroll
        for (int q = 0; q < QMAX; ++q) acc[q] = 0.0;
        if (ct == 0) stage(0, 0, true);
        for (int64_t b = 0; b < mk.nblk; ++b) {
            const int64_t kb0 = b * tpb_all;
            const int target = (int)((kb0 + tpb_all < mk.ntiles ? kb0 + tpb_all : mk.ntiles) - kb0);
            {
                MQ_T0();
                if (ct == 0) wait_counter(st.blk_done + b, target, st.faults, true);
                colsum_sync(NCW);
                if (ct == 0) MQ_T1(3);
            }
            MQ_T0();
            const int bl = (int)((((b * mk.m + j_lo) * 4) & 15) >> 2);  // lead of the bptr slice
            for (;;) {
                mbar_wait(cbar, cphase);
                cphase ^= 1u;
                const int64_t c0 = meta[2], c1 = meta[3], rhi = meta[1];
                const int pl = (int)(((c0 * 4) & 15) >> 2);
                const int32_t *sp = sperm + pl;
#pragma unroll
                for (int q = 0; q < QMAX; ++q) {
                    const int jl = ct + q * NCW * 32;
                    if (jl >= nc) break;
                    int64_t t = sbptr[bl + jl], e = sbptr[bl + jl + 1];
                    t = t > c0 ? t : c0;
                    e = e < c1 ? e : c1;
                    double a = acc[q];
                    for (; t + 8 <= e; t += 8) {
                        const int32_t *q8 = sp + (t - c0);
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = __ldcg(st.x + q8[u]);
#pragma unroll
                        for (int u = 0; u < 8; ++u) a += v[u];
                    }
                    if (t < e) {  // tail: up to 7 loads in flight, added in order
                        double v[7];
                        const int n_t = (int)(e - t);
#pragma unroll
                        for (int u = 0; u < 7; ++u)
                            v[u] = u < n_t ? __ldcg(st.x + sp[t - c0 + u]) : 0.0;
#pragma unroll
                        for (int u = 0; u < 7; ++u)
                            if (u < n_t) a += v[u];
                    }
                    acc[q] = a;
                }
                colsum_sync(NCW);  // everyone is done with the staged chunk
                if (c1 >= rhi) break;
                if (ct == 0) {
                    fence_proxy_async();
                    stage(b, c1, false);
                }
            }
            if (ct == 0) {
                MQ_T1(4);
                atomicAdd(st.blk_done + mk.nblk + b, 1);  // block b gathered by this CTA
                if (b + 1 < mk.nblk) {
                    fence_proxy_async();
                    stage(b + 1, 0, true);
                }
            }
        }
        if (write_cs) {
#pragma unroll
            for (int q = 0; q < QMAX; ++q) {
                const int jl = ct + q * NCW * 32;
                if (jl < nc) st.cs[j_lo + jl] = acc[q];
            }
        }
        return;
    }

#endif
    // ---------------------------------------------------------- solvers
    const int lane = tid & (G - 1);
    const int gsub = wl / G;
    const uint64_t pkeep = (kScatter || kBucket) ? policy_evict_last() : 0;
    const Avg av = avg_weights(st.navg, it);
    int my_sweeps = 0;  // per warp and launch: < 2^31
    int my_faults = 0;
    int64_t ph_blk = 0;
    if (kPipe) {
        // Software-pipelined solver: while a warp solves its current row
        // pair, the price gathers of its next pair (claimed ahead, possibly
        // from the next tile) are already in flight.  A warp leaves a tile
        // (arrives on empty[s]) once a claim there fails and the pair it still
        // holds from that tile is done.
        constexpr int RP = kRegPer;
        int64_t jt = -1;
        int ts = 0, tn = 0;  // stage / rows of the tile being claimed from
        bool tile_ok = false;
        auto enter_tile = [&]() {
            ++jt;
            ts = (int)(jt % NSTAGE);
            mbar_wait(&full[ts], (uint32_t)((jt / NSTAGE) & 1));
            tile_ok = stile[ts] >= 0;
            tn = tile_ok ? (int)(smeta[3 * ts + 1] - smeta[3 * ts]) : 0;
        };
        auto leave = [&](int s_) {
            __syncwarp();
            if (wl == 0) mbar_arrive(&empty[s_]);
        };
        struct View {  // a staged tile's arrays
            int64_t r0, e0;
            int nrows;
            const int64_t *srp;
            const double *sw, *ss, *su;
            const int32_t *scol;
            const uint8_t *sfl;
        };
        auto view = [&](int s_) {
            View v;
            v.r0 = smeta[3 * s_];
            v.nrows = (int)(smeta[3 * s_ + 1] - v.r0);
            unsigned char *b_ = smem + s_ * L::kStage;
            const int lr = (int)(((v.r0 * 8) & 15) >> 3);
            v.srp = reinterpret_cast<const int64_t *>(b_ + L::kRp) + lr;
            v.sw = reinterpret_cast<const double *>(b_ + L::kW) + lr;
            v.ss = reinterpret_cast<const double *>(b_ + L::kS) + lr;
            v.e0 = v.srp[0];
            v.su = reinterpret_cast<const double *>(b_ + L::kU) + (int)(((v.e0 * 8) & 15) >> 3);
            v.scol = reinterpret_cast<const int32_t *>(b_ + L::kCol) + (int)(((v.e0 * 4) & 15) >> 2);
            v.sfl = reinterpret_cast<const uint8_t *>(b_ + L::kF) + (int)(v.e0 & 15);
            return v;
        };
        int cur_s = -1, defer = -1;
        int nx_s = -1, nx_rb = 0;
        bool nx_reg = false, blocked = false;
        double pn[RP];
        auto claim_next = [&]() {
            nx_s = -1;
            while (tile_ok) {
                int rb = 0;
                if (wl == 0) rb = atomicAdd(&claim[ts], GPW);
                rb = __shfl_sync(MQ_FULL, rb, 0);
                if (rb < tn) {
                    nx_s = ts;
                    nx_rb = rb;
                    return;
                }
                if (cur_s == ts) defer = ts;  // its last pair here is still running
                else leave(ts);
                // the next tile would reuse the stage this warp still holds:
                // claim again once the current pair is done (no deadlock)
                // nor wait for a tile still loading while a pair is in hand
                const int64_t jn = jt + 1;
                // one lane's view of the barrier, so the warp stays converged
                const bool loaded = __shfl_sync(
                    MQ_FULL, (int)mbar_test(&full[(int)(jn % NSTAGE)], (uint32_t)((jn / NSTAGE) & 1)), 0);
                if (cur_s >= 0 && ((defer >= 0 && (int)(jn % NSTAGE) == defer) || !loaded)) {
                    blocked = true;
                    return;
                }
                enter_tile();
            }
        };
        auto issue_next = [&]() {  // the next pair's price gathers
            nx_reg = false;
            if (nx_s < 0) return;
            const View v = view(nx_s);
            const int r = nx_rb + gsub;
            int a = 0, b = 0;
            if (r < v.nrows) {
                a = (int)(v.srp[r] - v.e0);
                b = (int)(v.srp[r + 1] - v.e0);
            }
            nx_reg = __all_sync(MQ_FULL, b - a <= RP * G);
            if (nx_reg) {
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    pn[e] = t < b ? ld_price(st.p + v.scol[t]) : 0.0;
                }
            }
        };
        enter_tile();
        claim_next();
        issue_next();
        while (nx_s >= 0) {
            const int cs_ = nx_s, crb = nx_rb;
            const bool creg = nx_reg;
            double pv[RP];
#pragma unroll
            for (int e = 0; e < RP; ++e) pv[e] = pn[e];
            cur_s = cs_;
            claim_next();
            issue_next();
            // ---- solve the current pair
            const View v = view(cs_);
            const int r = crb + gsub;
            const bool has = r < v.nrows;
            int a = 0, b = 0;
            double tw = 0.0;
            if (has) {
                a = (int)(v.srp[r] - v.e0);
                b = (int)(v.srp[r + 1] - v.e0);
                tw = tau * v.sw[r];
            }
            const int64_t e0 = v.e0;
            int nsw = 0;
            bool ok = true;
            if (creg) {
                double c[RP];
                uint32_t fb = 0;
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    c[e] = 0.0;
                    if (t < b) {
                        const bool f = v.sfl[t] != 0;
                        if (f) fb |= 1u << e;
                        const double xe = f ? ld_na(st.x + e0 + t) : 0.0;
                        if (x_prev_out) x_prev_out[e0 + t] = xe;
                        c[e] = xe - tau * pv[e];
                    }
                }
                const double s0 = has ? v.ss[r] : 0.0;
                const uint32_t gmask = G == 32 ? MQ_FULL : (((1u << G) - 1u) << (gsub * G));
                const uint32_t su_l = smem_addr(v.su + a + lane);
                const int n_l = b - a - lane > 0 ? (b - a - lane + G - 1) / G : 0;
                auto uf = [&](int e) -> double { return e < n_l ? lds_f64(su_l + e * G * 8) : 0.0; };
                const double sr = row_root_warm<G, RP>(c, uf, tw, s0, has, gmask, &nsw, &ok);
                if (has && lane == 0) st.srow[v.r0 + r] = sr;
                const double inv_s = 1.0 / sr;
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    if (t < b) {
                        const double xn = fmax(c[e] + tw * v.su[t] * inv_s, 0.0);
                        const bool nz = xn > 0.0;
                        st_flag(st.xflag + e0 + t, nz);
                        if (nz || ((fb >> e) & 1u)) st.x[e0 + t] = xn;
                        if (nz) {
                            red_add_f64(st.xsum + e0 + t, xn);
                            fixed_colsum_add(mk, st, v.scol[t], xn);
                        }
                    }
                }
            } else {
                // longer rows: c is kept in x (global) across the sweeps
                double *sc = st.x + e0;
                double ap = 0.0, bp = 0.0;
                for (int t = a + lane; t < b; t += G) {
                    const double ue = v.su[t];
                    const double xe = v.sfl[t] ? ld_na(st.x + e0 + t) : 0.0;
                    if (x_prev_out) x_prev_out[e0 + t] = xe;
                    const double ce = xe - tau * ld_price(st.p + v.scol[t]);
                    sc[t] = ce;
                    ap += ue * ce;
                    bp += ue * ue;
                }
                const double s0 = has ? v.ss[r] : 0.0;
                const double A = group_sum<G>(ap);
                const double B = group_sum<G>(bp);
                const double sr =
                    row_root_exact<G>(v.su, sc, a, b, lane, tw, s0, A, B, has, &nsw, &ok);
                if (has && lane == 0) st.srow[v.r0 + r] = sr;
                const double inv_s = 1.0 / sr;
                for (int t = a + lane; t < b; t += G) {
                    const double xn = fmax(sc[t] + tw * v.su[t] * inv_s, 0.0);
                    const bool nz = xn > 0.0;
                    st_flag(st.xflag + e0 + t, nz);
                    st.x[e0 + t] = xn;
                    if (nz) {
                        red_add_f64(st.xsum + e0 + t, xn);
                        fixed_colsum_add(mk, st, v.scol[t], xn);
                    }
                }
            }
            if (has && b > a && lane == 0) {
                my_sweeps += nsw;
                if (!ok) ++my_faults;
            }
            cur_s = -1;
            if (defer == cs_) {
                leave(cs_);
                defer = -1;
            }
            if (blocked) {
                blocked = false;
                enter_tile();
                claim_next();
                issue_next();
            }
        }
    }
    for (int64_t j = 0; !kPipe; ++j) {
        const int s = (int)(j % NSTAGE);
        {
            MQ_T0();
            mbar_wait(NGW > 0 ? &ready[s] : &full[s], (uint32_t)((j / NSTAGE) & 1));
            if (wl == 0) MQ_T1(0);
        }
        const int64_t k = stile[s];
        if (kPhased && k == -2) {  // end of a block: release the stage, then gather
            __syncwarp();
            if (wl == 0) mbar_arrive(&empty[s]);
            phased_gather<PQ>(mk, st, ph_blk, tid, NP, ph_lo, ph_nc, ph_sval, ph_acc);
            ++ph_blk;
            continue;
        }
        if (k < 0) break;  // sentinel
        // throttle: stay within kLag blocks of the column-sum front, so the
        // blocks still to be gathered are L2-resident
        const int64_t blk = k / tpb_all;
        {
            MQ_T0();
#if !defined(MQ_NO_COLSUM) && !defined(MQ_CS_NOWAIT)
            if (!kScatter && !kSplit && !kPhased && !kAtomic && blk >= kLag && wl == 0)
                wait_counter(st.blk_done + mk.nblk + (blk - kLag),
                             (int)gridDim.x * (kCsPerWarp ? NCW : 1), st.faults, false);
#endif
            __syncwarp();
            if (wl == 0) MQ_T1(1);
        }
        const int64_t r0 = smeta[3 * s], r1 = smeta[3 * s + 1];
        const int nrows = (int)(r1 - r0);
        unsigned char *base = smem + s * L::kStage;
        const int lr = (int)(((r0 * 8) & 15) >> 3);
        const int64_t *srp = reinterpret_cast<const int64_t *>(base + L::kRp) + lr;
        const double *sw = reinterpret_cast<const double *>(base + L::kW) + lr;
        const double *ss = reinterpret_cast<const double *>(base + L::kS) + lr;
        const int64_t e0 = srp[0];
        const int d8 = (int)(((e0 * 8) & 15) >> 3), d4 = (int)(((e0 * 4) & 15) >> 2);
        const double *su = reinterpret_cast<const double *>(base + L::kU) + d8;
        double *sx = reinterpret_cast<double *>(base + L::kX) + d8;
        const double *sxb = reinterpret_cast<const double *>(base + L::kXB) + d8;
        // c = x - tau p[col]: from the gather warps, or computed here (then
        // written over x in place for the shared-memory path)
        double *sc = (NGW > 0 && kXDirect) ? reinterpret_cast<double *>(base + L::kC) + d8
                     : kXDirect ? st.x + e0
                                : reinterpret_cast<double *>(base + L::kX) + d8;
        auto ldx = [&](int t) -> double { return kXDirect ? ld_na(st.x + e0 + t) : sx[t]; };
        auto ldxb = [&](int t) -> double { return kXBDirect ? ld_na(st.xbar + e0 + t) : sxb[t]; };
        const int32_t *scol = reinterpret_cast<const int32_t *>(base + L::kCol) + d4;
        const int32_t *stp = reinterpret_cast<const int32_t *>(base + L::kTp) + d4;
        double *bslot = kBucket ? st.bucket + (blk % kLag) * mk.bcap : nullptr;
        const uint8_t *sfl = reinterpret_cast<const uint8_t *>(base + L::kF) + (int)(e0 & 15);
        // sparse iterate: x of flagged entries only, zero otherwise
        auto ldxs = [&](int t) -> double {
#ifdef MQ_EXP_NOX  // timing experiment only (wrong results): no x loads
            return 0.0 * sfl[t];
#endif
            return kSparse ? (sfl[t] ? ld_na(st.x + e0 + t) : 0.0) : ldx(t);
        };
        // store x^{k+1} (+ its flag and running sum, or the running average)
        auto put_x = [&](int t, double xn, bool was_nz, bool dense_x) {
            if (kSparse) {
                const bool nz = xn > 0.0;
                st_flag(st.xflag + e0 + t, nz);
                if (nz || was_nz || dense_x) st.x[e0 + t] = xn;
                if (nz) red_add_f64(st.xsum + e0 + t, xn);
            } else {
                st.x[e0 + t] = xn;
            }
        };

        MQ_TA(13, 0, 1);  // tile visits
#ifdef MQ_STATIC_PAIRS
        // static: warp w takes row pairs w, w + NSW, ... of the tile (no claims)
        for (int pp = warp;; pp += NSW) {
            MQ_TS(tc0);
            const int rb = pp * GPW;
#elif defined(MQ_CLAIM_AHEAD)
        // the next claim is issued before the current pair is solved, so its
        // shared-atomic round trip is off the critical path
        int rb_ahead = 0;
        if (wl == 0) rb_ahead = atomicAdd(&claim[s], GPW);
        for (;;) {
            MQ_TS(tc0);
            const int rb = __shfl_sync(MQ_FULL, rb_ahead, 0);
            if (rb < nrows && wl == 0) rb_ahead = atomicAdd(&claim[s], GPW);
#else
        for (;;) {
            MQ_TS(tc0);
            int rb = 0;
            if (wl == 0) rb = atomicAdd(&claim[s], GPW);
            rb = __shfl_sync(MQ_FULL, rb, 0);
#endif
            MQ_TS(tc1);
            MQ_TA(8, tc0, tc1);
            if (rb >= nrows) break;  // warp-uniform
            MQ_TA(12, 0, 1);  // row pairs
            const int r = rb + gsub;
            const bool has = r < nrows;
            int a = 0, b = 0;
            double tw = 0.0;
            if (has) {
                a = (int)(srp[r] - e0);
                b = (int)(srp[r + 1] - e0);
                tw = tau * sw[r];
            }
            int nsw = 0;
            bool ok = true;
#ifdef MQ_TRIVIAL_SOLVE  // bandwidth experiment: stream the tile, skip the solve
            if (MQ_TRIVIAL_SOLVE == 1) {
                for (int t = a + lane; t < b; t += G) {
                    const double xn = ldx(t) + 1e-300 * su[t];
                    st.x[e0 + t] = xn;
                    __stcs(st.xbar + e0 + t, av.wold * ldxb(t) + av.wnew * xn);
                    if (kScatter) st_keep(st.xc + stp[t], xn, pkeep);
                    if (kBucket) st_keep(bslot + stp[t], xn, pkeep);
                    if (kAtomic && xn > 0.0) fixed_colsum_add(mk, st, scol[t], xn);
                }
            }
            if (false) {
#else
            if (kRegPer > 0 && __all_sync(MQ_FULL, b - a <= kRegPer * G)) {
#endif
                // ---- row in registers
                constexpr int RP = kRegPer > 0 ? kRegPer : 1;
                MQ_TS(tq0);
                MQ_TA(9, tc1, tq0);
                double c[RP], u[RP];
                uint32_t fb = 0;  // entries whose x^k was nonzero (sparse iterate)
                // every load of the pair is issued before any is consumed: the
                // price gathers and the flagged x loads overlap in one round trip
                double pv[RP], xv[RP];
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    const bool in = t < b;
                    pv[e] = (in && NGW == 0) ? ld_price(st.p + scol[t]) : 0.0;
                    bool f = false;
                    if (kSparse) f = in && sfl[t];
                    if (f) fb |= 1u << e;
                    xv[e] = NGW > 0 ? 0.0
                            : kSparse ? (f ? __ldcg(st.x + e0 + t) : 0.0)
                                      : (in ? ldx(t) : 0.0);
                    u[e] = in ? su[t] : 0.0;
                }
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    c[e] = t < b ? (NGW > 0 ? sc[t] : xv[e] - tau * pv[e]) : 0.0;
                }
                if (x_prev_out && NGW == 0) {
#pragma unroll
                    for (int e = 0; e < RP; ++e) {
                        const int t = a + lane + e * G;
                        if (t < b) x_prev_out[e0 + t] = xv[e];
                    }
                }
                const double s0 = has ? ss[r] : 0.0;
                MQ_TS(tq1);
                const uint32_t gmask = G == 32 ? MQ_FULL : (((1u << G) - 1u) << (gsub * G));
#ifdef MQ_U_SMEM
                // utilities re-read from the stage (fewer live registers per pair)
                const uint32_t su_l = smem_addr(su + a + lane);
                const int n_l = b - a - lane > 0 ? (b - a - lane + G - 1) / G : 0;
                auto uf = [&](int e) -> double { return e < n_l ? lds_f64(su_l + e * G * 8) : 0.0; };
#else
                auto uf = [&](int e) -> double { return u[e]; };
#endif
                const double sr = row_root_warm<G, RP>(c, uf, tw, s0, has, gmask, &nsw, &ok);
                if (has && lane == 0) st.srow[r0 + r] = sr;
                const double inv_s = 1.0 / sr;
                MQ_TS(tq2);
                constexpr int XP = (kXBDirect && !kSparse) ? RP : 1;  // direct xbar: loads first
                double xb[XP];
                if (kXBDirect && !kSparse) {
#pragma unroll
                    for (int e = 0; e < XP; ++e) {
                        const int t = a + lane + e * G;
                        xb[e] = t < b ? ldxb(t) : 0.0;
                    }
                }
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    if (t < b) {
#ifdef MQ_U_SMEM
                        const double xn = fmax(c[e] + tw * su[t] * inv_s, 0.0);
#else
                        const double xn = fmax(c[e] + tw * u[e] * inv_s, 0.0);
#endif
                        put_x(t, xn, (fb >> e) & 1u, false);
                        if (!kSparse)
                            __stcs(st.xbar + e0 + t,
                                   av.wold * (kXBDirect ? xb[e % XP] : ldxb(t)) + av.wnew * xn);
                        if (kScatter) st_keep(st.xc + stp[t], xn, pkeep);
                    if (kBucket) st_keep(bslot + stp[t], xn, pkeep);
                    if (kAtomic && xn > 0.0) fixed_colsum_add(mk, st, scol[t], xn);
                    }
                }
                MQ_TS(tq3);
                MQ_TA(5, tq0, tq1);
                MQ_TA(6, tq1, tq2);
                MQ_TA(7, tq2, tq3);
            } else if (!kTrivial) {
                // ---- longer rows: stream the row from shared memory
                double s0p = 0.0, ap = 0.0, bp = 0.0;
                // batches of 8 entries per lane: all loads of a batch in flight
                // before its c values are stored over x (the stores could alias
                // the next loads, which would serialize every gather)
#ifndef MQ_LB
#define MQ_LB 8
#endif
                constexpr int LB = MQ_LB;
                for (int t0 = a + lane; t0 < b; t0 += LB * G) {
                    double pv[LB], xv[LB];
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const int t = t0 + q * G;
                        const bool in = t < b;
                        pv[q] = (in && NGW == 0) ? ld_price(st.p + scol[t]) : 0.0;
                        xv[q] = (!in || NGW > 0) ? 0.0
                                : kSparse ? (sfl[t] ? __ldcg(st.x + e0 + t) : 0.0) : ldx(t);
                    }
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const int t = t0 + q * G;
                        if (t < b) {
                            const double ue = su[t], xe = xv[q];
                            double ce;
                            if (NGW > 0) {
                                ce = sc[t];
                            } else {
                                ce = xe - tau * pv[q];
                                if (x_prev_out) x_prev_out[e0 + t] = xe;
                                sc[t] = ce;  // over x (stage or global): this lane's entry only
                            }
                            s0p += ue * xe;
                            ap += ue * ce;
                            bp += ue * ue;
                        }
                    }
                }
                // with gather warps x is gone from the stage: warm start from srow
                const double s0 = NGW > 0 ? (has ? ss[r] : 0.0) : group_sum<G>(s0p);
                const double A = group_sum<G>(ap);
                const double B = group_sum<G>(bp);
                const double sr =
                    row_root_exact<G>(su, sc, a, b, lane, tw, s0, A, B, has, &nsw, &ok);
                if (has && lane == 0) st.srow[r0 + r] = sr;
                const double inv_s = 1.0 / sr;
                for (int t0 = a + lane; t0 < b; t0 += LB * G) {
                    double cv[LB];
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const int t = t0 + q * G;
                        cv[q] = t < b ? sc[t] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const int t = t0 + q * G;
                        if (t < b) {
                            const double xn = fmax(cv[q] + tw * su[t] * inv_s, 0.0);
                            // x held c during the sweeps (direct mode): rewrite every entry
                            put_x(t, xn, true, kXDirect);
                            if (!kSparse)
                                __stcs(st.xbar + e0 + t, av.wold * ldxb(t) + av.wnew * xn);
                            if (kScatter) st_keep(st.xc + stp[t], xn, pkeep);
                            if (kBucket) st_keep(bslot + stp[t], xn, pkeep);
                            if (kAtomic && xn > 0.0) fixed_colsum_add(mk, st, scol[t], xn);
                        }
                    }
                }
                // c was written over x in this stage: order those generic-proxy
                // writes before the producer's next bulk copy into the stage
                if (NGW == 0 && !kXDirect) fence_proxy_async();
            }
            if (has && b > a && lane == 0) {
                my_sweeps += nsw;
                if (!ok) ++my_faults;
            }
        }
        MQ_TS(te0);
        __syncwarp();
        if (wl == 0) {
            // the last solver warp out of the tile publishes it (one gpu-scope
            // fence per tile, off the producer's path)
            int prior = 0;
            if (!kAtomic)  // only the block publication below needs the count
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(prior) : "r"(smem_addr(&claim[NSTAGE + s])) : "memory");
#ifndef MQ_NO_PUBLISH
            if (!kSplit && !kScatter && !kPhased && !kAtomic && prior == NSW - 1) {
                __threadfence();
                atomicAdd(&st.blk_done[k / tpb_all], 1);
            }
#endif
            mbar_arrive(&empty[s]);
        }
        {
            MQ_TS(te1);
            MQ_TA(10, te0, te1);
        }
    }
    if (kPhased && write_cs) {
#pragma unroll
        for (int q = 0; q < PQ; ++q) {
            const int jl = tid + q * NP;
            if (jl < ph_nc) st.cs[ph_lo + jl] = ph_acc[q];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_sweeps += __shfl_xor_sync(MQ_FULL, my_sweeps, o);
        my_faults += __shfl_xor_sync(MQ_FULL, my_faults, o);
    }
    if (wl == 0 && my_sweeps)
        atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)my_sweeps);
    if (wl == 0 && my_faults)
        atomicAdd((unsigned long long *)st.faults, (unsigned long long)my_faults);
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

__global__ void __launch_bounds__(256)
primal_long_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out) {
    __shared__ double sm[96];
    const double tau = st.steps[0];
    const Avg av = avg_weights(st.navg, it);
    int64_t my_sweeps = 0;
    int my_faults = 0;
    for (int64_t r = blockIdx.x; r < mk.nlong; r += gridDim.x) {
        const int64_t i = mk.long_rows[r];
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
            if (kSparse) {
                st.xflag[t] = xn > 0.0;
                if (xn > 0.0) st.xsum[t] += xn;
            } else {
                st.xbar[t] = av.wold * st.xbar[t] + av.wnew * xn;
            }
            if (kScatter) st.xc[mk.tpos[t]] = xn;
            if (kAtomic && xn > 0.0) fixed_colsum_add(mk, st, mk.col[t], xn);
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
// Generic / long-row column sums over the blocked schedule: one thread per
// good walking blocks [b_lo, b_hi) in order (ascending rows), 4 gathers in
// flight.  acc_in (may be NULL) is the running sum to continue from.
__global__ void __launch_bounds__(256)
colsum_blocks_kernel(int64_t m, const int32_t *__restrict__ bptr, const int32_t *__restrict__ bperm,
                     int64_t b_lo, int64_t b_hi, const double *__restrict__ v,
                     const double *__restrict__ acc_in, double *__restrict__ out,
                     double *__restrict__ csbar, const int64_t *__restrict__ navg, int it) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    double acc = acc_in ? acc_in[j] : 0.0;
    for (int64_t b = b_lo; b < b_hi; ++b) {
        int64_t t = bptr[b * m + j];
        const int64_t end = bptr[b * m + j + 1];
        for (; t + 4 <= end; t += 4) {
            const double v0 = v[bperm[t]], v1 = v[bperm[t + 1]];
            const double v2 = v[bperm[t + 2]], v3 = v[bperm[t + 3]];
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; t < end; ++t) acc += v[bperm[t]];
    }
    out[j] = acc;
    if (csbar) {
        const Avg av = avg_weights(navg, it);
        csbar[j] = av.wold * csbar[j] + av.wnew * acc;
    }
}

// Scatter mode: xc holds x in column-major order, so a good's entries are
// contiguous: one warp per good streams them (coalesced, 4 loads in flight
// per lane, fixed butterfly => deterministic).
__global__ void __launch_bounds__(256)
colsum_xc_kernel(int64_t m, const int64_t *__restrict__ tptr, const double *__restrict__ xc,
                 double *__restrict__ out, double *__restrict__ csbar,
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
            const double v0 = __ldcs(xc + t), v1 = __ldcs(xc + t + 32);
            const double v2 = __ldcs(xc + t + 64), v3 = __ldcs(xc + t + 96);
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; t < end; t += 32) acc += __ldcs(xc + t);
        acc = group_sum<32>(acc);
        if (lane == 0) {
            out[j] = acc;
            if (csbar) csbar[j] = av.wold * csbar[j] + av.wnew * acc;
        }
    }
}

// Split mode: column sums of one block of tiles right after its primal
// launch, while its x is L2-resident: one warp per good, lanes stride the
// good's segment (coalesced bperm, independent gathers), fixed butterfly;
// blocks are added into cs in order (deterministic).
__global__ void __launch_bounds__(256)
colsum_seg_kernel(int64_t m, const int32_t *__restrict__ bptr, const int32_t *__restrict__ bperm,
                  int64_t b, const double *__restrict__ x, double *__restrict__ cs) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t row0 = b * m;
    for (int64_t j = warp_id; j < m; j += nwarps) {
        const int64_t beg = bptr[row0 + j], end = bptr[row0 + j + 1];
        double acc = 0.0;
        int64_t t = beg + lane;
        for (; t + 96 < end; t += 128) {
            const int32_t k0 = __ldcs(bperm + t), k1 = __ldcs(bperm + t + 32);
            const int32_t k2 = __ldcs(bperm + t + 64), k3 = __ldcs(bperm + t + 96);
            const double v0 = __ldcg(x + k0), v1 = __ldcg(x + k1);
            const double v2 = __ldcg(x + k2), v3 = __ldcg(x + k3);
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; t < end; t += 32) acc += __ldcg(x + __ldcs(bperm + t));
        acc = group_sum<32>(acc);
        if (lane == 0) cs[j] = b == 0 ? acc : cs[j] + acc;
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

// xbar = S / count (sparse iterate): the running average of kernels.py:138-142
// from the running sum, once per chunk
__global__ void avg_materialize_kernel(int64_t nnz, const double *__restrict__ xsum,
                                       double *__restrict__ xbar, const int64_t *__restrict__ navg) {
    const double count = (double)*navg;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        xbar[e] = count > 0.0 ? xsum[e] / count : xbar[e];
}

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

constexpr int kG = MQ_G, kNSW = MQ_NSW, kNGW = MQ_NGW, kNCW = MQ_NCW, kStages = MQ_STAGES;
constexpr int kEtile = MQ_ETILE;
#ifdef MQ_CS_PERWARP
constexpr int kQMax = (kWCols + 31) / 32;  // goods per column-sum lane
#else
constexpr int kQMax = kNCW > 0 ? (1152 + kNCW * 32 - 1) / (kNCW * 32) : 1;  // goods per thread
#endif
using PrimalLayout = TileLayout<kEtile, MQ_TILE_ROWS, (kNGW > 0 && kXDirect)>;

constexpr int kPrimalSmem = MQ_SMEM_PAD + kStages * PrimalLayout::kStage + 7 * kStages * 8 + 4 * kStages * 4 + 128 +
                            (kPhased ? kPhChunk * 8 : (kScatter || kSplit) ? 0 :
#ifdef MQ_CS_PERWARP
                             kNCW * (((2 * (kCsChunk + 8) + 2 * (kWCols + 8)) * 4 + kCsChunk * 8 +
                                      8 * 8 + 2 * 8 + 127) / 128 * 128)
#else
                             kAtomic ? 0
                             : kBucket ? (kCsCols + 8) * 4 + 2 * (kBkChunk + 4) * 8 + 3 * 8 + 16
                                       : (kCsCap + kCsCols + 8) * 4 + 4 * 8 + 16
#endif
                            );

int primal_launch(const mq_market *mk, const mq_state *st, int it, double *xprev, cudaStream_t s) {
    static bool configured = false;
    auto kern = primal_fused_kernel<kG, kNSW, kNGW, kNCW, kEtile, MQ_TILE_ROWS, kStages, kQMax>;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kPrimalSmem);
        if (e != cudaSuccess) return set_error(e, "mq_primal_step: smem attribute");
        configured = true;
    }
    const int nthr = (kNSW + kNGW + kNCW + 1 + kPF) * 32;
    if (mk->ntiles > 0 && kSplit) {
        // per block of tiles: the primal sweep, then the block's column sums
        // while its x is still in L2
        cudaMemsetAsync(st->blk_done, 0, sizeof(int32_t) * ((size_t)mk->nblk + 1), s);
        const int cgrid = grid_for(mk->m, 8, sm_count() * 8);
        for (int64_t b = 0; b < mk->nblk; ++b) {
            const int64_t lo = b * mk->tiles_per_block;
            const int64_t hi = lo + mk->tiles_per_block < mk->ntiles ? lo + mk->tiles_per_block
                                                                     : mk->ntiles;
            const int grid = (int)(hi - lo < mk->prim_grid ? hi - lo : mk->prim_grid);
            kern<<<grid, nthr, kPrimalSmem, s>>>(*mk, *st, it, xprev, 0, lo, hi, st->blk_done + b);
            colsum_seg_kernel<<<cgrid, 256, 0, s>>>(mk->m, mk->bptr, mk->bperm, b, st->x, st->cs);
        }
    } else if (mk->ntiles > 0 && kPhased) {
        if ((mk->m + mk->prim_grid - 1) / mk->prim_grid > 2048)
            return set_error(cudaErrorInvalidValue, "mq_primal_step: too many goods per CTA");
        cudaMemsetAsync(st->blk_done, 0, sizeof(int32_t) * (2 * (size_t)mk->nblk + 1), s);
        kern<<<mk->prim_grid, nthr, kPrimalSmem, s>>>(*mk, *st, it, xprev, 1, 0, mk->ntiles,
                                                      st->blk_done);
    } else if (mk->ntiles > 0) {
        if ((mk->m + mk->prim_grid - 1) / mk->prim_grid > (int64_t)kCsCols)
            return set_error(cudaErrorInvalidValue, "mq_primal_step: too many goods per CTA");
        cudaMemsetAsync(st->blk_done, 0, sizeof(int32_t) * (2 * (size_t)mk->nblk + 1), s);
        kern<<<mk->prim_grid, nthr, kPrimalSmem, s>>>(*mk, *st, it, xprev, 1, 0, mk->ntiles,
                                                      st->blk_done + 2 * mk->nblk);
    } else {
        cudaMemsetAsync(st->cs, 0, sizeof(double) * (size_t)mk->m, s);
    }
    if (mk->nlong > 0) {
        const int grid = grid_for(mk->nlong, 1, sm_count() * 8);
        primal_long_kernel<<<grid, 256, 0, s>>>(*mk, *st, it, xprev);
    }
    return check_launch("mq_primal_step");
}

// adds the long rows (pseudo-block nblk) to cs; csbar update when finalize
__global__ void cs_from_fixed_kernel(int64_t m, unsigned long long *__restrict__ fix,
                                     double *__restrict__ cs, double *__restrict__ csbar,
                                     const int64_t *__restrict__ navg, int it, double inv_scale) {
    const Avg av = avg_weights(navg, it);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double c = (double)fix[j] * inv_scale;  // exact for sums < 2^53 units
        cs[j] = c;
        fix[j] = 0ull;
        if (csbar) csbar[j] = av.wold * csbar[j] + av.wnew * c;
    }
}

int colsum_rest_launch(const mq_market *mk, const mq_state *st, int it, int finalize,
                       cudaStream_t s) {
    if (kAtomic) {  // every entry (tiles and long rows) went through the atomics
        cs_from_fixed_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(
            mk->m, reinterpret_cast<unsigned long long *>(st->bucket), st->cs,
            finalize ? st->csbar : nullptr, st->navg, it, 1.0 / mk->cs_scale);
        return check_launch("mq_colsum_step");
    }
    if (kScatter) {
        colsum_xc_kernel<<<grid_for(mk->m, 8, sm_count() * 8), 256, 0, s>>>(
            mk->m, mk->tptr, st->xc, st->cs, finalize ? st->csbar : nullptr, st->navg, it);
        return check_launch("mq_colsum_step");
    }
    const int grid = (int)((mk->m + 255) / 256);
    if (mk->nlong > 0) {
        colsum_blocks_kernel<<<grid, 256, 0, s>>>(mk->m, mk->bptr, mk->bperm, mk->nblk,
                                                  mk->nblk + 1, st->x, st->cs, st->cs,
                                                  finalize ? st->csbar : nullptr, st->navg, it);
    } else if (finalize) {
        colsum_finalize_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(
            mk->m, st->cs, st->csbar, st->navg, it);
    }
    return check_launch("mq_colsum_step");
}

// shared with the lifted PDHG step (lifted.cu)
int launch_dual(const mq_market *mk, double *p, double *pbar, double *cs, double *cs_prev,
                const double *steps, const int64_t *navg, int it, cudaStream_t s) {
    dual_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(mk->m, p, pbar, cs, cs_prev,
                                                                     steps, navg, it);
    return check_launch("mq_dual_step");
}
int launch_cs_from_fixed(const mq_market *mk, unsigned long long *fix, double *cs, double *csbar,
                         const int64_t *navg, int it, cudaStream_t s) {
    cs_from_fixed_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(
        mk->m, fix, cs, csbar, navg, it, 1.0 / mk->cs_scale);
    return check_launch("mq_colsum_step");
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
    return colsum_rest_launch(mk, st, it, finalize, (cudaStream_t)stream);
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
        if ((rc = colsum_rest_launch(mk, st, it, 1, s))) return rc;
    }
    if ((rc = mq_chunk_end(st, iters, stream))) return rc;
    return mq_avg_materialize(mk, st, stream);
}

// debug: read and reset the wait-cycle counters (zeros unless built with
// -DMQ_PROFILE_WAITS); not part of the public header
int mq_debug_counters(unsigned long long *out_host) {
    cudaError_t e = cudaMemcpyFromSymbol(out_host, g_wait_cycles, sizeof(g_wait_cycles));
    if (e != cudaSuccess) return set_error(e, "mq_debug_counters");
    unsigned long long z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_wait_cycles, z, sizeof(z));
    return e == cudaSuccess ? 0 : set_error(e, "mq_debug_counters");
}

int mq_tile_entries(void) { return kEtile; }

int mq_colsum_mode(void) {
    return kScatter ? 1 : (kSplit ? 2 : (kPhased ? 3 : (kBucket ? 4 : (kAtomic ? 5 : 0))));
}

int mq_bucket_slots(void) { return kBucket ? (int)kLag : 0; }
int mq_x_sparse(void) { return kSparse ? 1 : 0; }

int mq_avg_materialize(const mq_market *mk, const mq_state *st, void *stream) {
    if (!kSparse) return 0;
    if (!mk || !st) return set_error(cudaErrorInvalidValue, "mq_avg_materialize: null argument");
    avg_materialize_kernel<<<grid_for(mk->nnz, 256, sm_count() * 16), 256, 0, (cudaStream_t)stream>>>(
        mk->nnz, st->xsum, st->xbar, st->navg);
    return check_launch("mq_avg_materialize");
}
int mq_fixed_colsum(void) { return kAtomic ? 1 : 0; }

int mq_colsum(const mq_market *mk, const double *v, double *out, void *stream) {
    const int grid = (int)((mk->m + 255) / 256);
    colsum_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        mk->m, mk->bptr, mk->bperm, 0, mk->nblk + 1, v, nullptr, out, nullptr, nullptr, 0);
    return check_launch("mq_colsum");
}

}  // extern "C"
