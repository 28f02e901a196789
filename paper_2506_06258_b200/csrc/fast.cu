// Fast PDHCG iteration for sm_100a: exact warm-started per-buyer prox, sparse
// iterate, fixed-point column sums, price step.  One iteration =
// mq_dual_step + mq_primal_step + mq_colsum_step; all scalars (tau, sigma,
// navg) are device-resident so a chunk is captured once as a CUDA graph.
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
// The iterate is ~99 % zero after the first iteration (each buyer buys a few
// goods), which shapes the data flow:
//  * x is never streamed: a byte flag per entry (x > 0) is staged instead,
//    x is loaded only where flagged, written only where it is or was nonzero;
//  * the running average is a running sum S = sum of x since the restart,
//    updated with atomics on nonzero x only, xbar = S / count once per chunk;
//  * column sums add round(x * 2^k) of the nonzero entries into u64
//    accumulators: integer addition is associative, so they are bitwise
//    deterministic in any order (no transpose, no cross-CTA synchronisation).
//
// One persistent, warp-specialized kernel per iteration (primal_fused_kernel):
//  * a TMA producer warp streams each tile (whole rows, <= MQ_TILE_ENTRIES
//    entries: u, col, flags, row offsets, budgets, warm starts) into a
//    4-stage shared-memory ring with cp.async.bulk + mbarrier transaction
//    counts, claiming tiles dynamically from a global counter;
//  * 19 solver warps claim row pairs of the current tile (two 16-lane groups
//    per warp) and solve them, rows of <= 128 entries in registers.
// Skewed markets add two kernels after it: tile rows of 129-1024 entries
// (skipped by the tile kernel, so no stage waits on one slow row) are solved
// one warp per row (primal_med_kernel), rows > 1024 entries one CTA per row
// with the row's first MQ_LONG_CAP entries held in shared memory across the
// sweeps (primal_long_kernel).
// Variants measured along the way (dense iterate with gathered / bucketed /
// scattered column sums, gather warps, software pipelining, ...) are listed
// with their numbers in DESIGN.md §11.
#include <math_constants.h>

#include "mq_common.cuh"
#include "mq_tma.cuh"

// ---- compile-time configuration (tuning variants override with -D) ----
#ifndef MQ_G
#define MQ_G 16  // lanes per row
#endif
#ifndef MQ_NSW
#define MQ_NSW 19  // solver warps: 20 warps per CTA at 96 registers
#endif
#ifndef MQ_ETILE
#define MQ_ETILE MQ_TILE_ENTRIES
#endif
// Shared memory is sized so that the unified L1 keeps ~92 KB: random gathers
// (p[col]) need L1 lines to track their misses, and their throughput halves
// when the carveout leaves ~28 KB (tools/micro/gather_l1.cu).
#ifndef MQ_STAGES
#define MQ_STAGES 4  // 4 x 2560-entry stages: 158 KB (carveout 164 KB, 92 KB of L1)
#endif
#ifndef MQ_REG_PER
#define MQ_REG_PER 8  // entries per lane kept in registers (rows <= MQ_G * MQ_REG_PER)
#endif
#ifndef MQ_CLAIM
#define MQ_CLAIM 2  // tiles claimed per global atomic by a producer
#endif
#ifndef MQ_LB
#define MQ_LB 8  // entries per lane batched ahead of the stores (longer rows)
#endif
#ifndef MQ_LONG_THREADS
#define MQ_LONG_THREADS 256  // threads per CTA of the long-row kernel (one row per CTA)
#endif
#ifndef MQ_LONG_PER_SM
#define MQ_LONG_PER_SM 4  // resident long-row CTAs per SM (one row each)
#endif
#ifndef MQ_LONG_LB
#define MQ_LONG_LB 4  // entries per thread batched ahead of the stores (long rows)
#endif
#ifndef MQ_MED_CAP
#define MQ_MED_CAP 128  // working-set pool of a medium row > MQ_WS_MAX_ROW (4 per lane)
#endif
#ifndef MQ_LONG_WCAP
#define MQ_LONG_WCAP 128  // long-row pools up to this size are solved by a warp (primal_long_ws_kernel)
#endif
#ifndef MQ_LONG_CAP
#define MQ_LONG_CAP 1536  // entries of a long row kept in shared memory (32 KB, 4 CTAs/SM:
                          // the rest of the carveout stays L1 for the price gathers)
#endif

namespace mq {

constexpr int kMaxSweeps = 4096;

// cycle counters of the fused kernel (mq_debug_counters, tools/waits.py):
// 0 solver waiting for a tile, 2 producer waiting for a free stage, 5 solver
// loads + c, 6 row root, 7 stores, 8 claim, 9 row metadata, 10 tile end,
// 12 row pairs, 13 tile visits
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

// The fire-and-forget stores below carry no "memory" clobber: nothing in the
// kernel reads these addresses after writing them, and without the compiler
// barrier the loads around them (staged columns, utilities) can be scheduled
// freely.
__device__ __forceinline__ void st_flag(uint8_t *p, bool v) {
    asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"((int)v));
}
// float add (one writer per address and iteration: the plain rounded sum)
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}
// Column sums as fixed-point integers: x_e * cs_scale rounded to u64, added
// with fire-and-forget atomics only for the entries with x_e > 0.  cs_scale =
// 2^k is chosen per market so that no column can overflow while every x_e <
// cs_xmax (a larger x_e is counted as a fault; device.py fixed_point_scale).
__device__ __forceinline__ void fixed_colsum_add(const mq_market &mk, const mq_state &st, int j,
                                                 double xe) {
    MQ_CHECK(j >= 0 && j < mk.m);
    if (xe < mk.cs_xmax) {
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(reinterpret_cast<unsigned long long *>(
                         st.bucket) + j),
                     "l"(__double2ull_rn(xe * mk.cs_scale)));
    } else {  // out of the fixed-point range: faults[1] (engine raises FixedPointRangeError)
        atomicAdd(reinterpret_cast<unsigned long long *>(st.faults) + 1, 1ull);
    }
}

// the new x of an entry: its flag, its value where it is or was nonzero (so
// the dense array stays exact), the running sum and the column sum
__device__ __forceinline__ void put_x(const mq_market &mk, const mq_state &st, int64_t e, int j,
                                      double xn, bool write_x) {
    MQ_CHECK(e >= 0 && e < mk.nnz);
    const bool nz = xn > 0.0;
    st_flag(st.xflag + e, nz);
    if (nz || write_x) st.x[e] = xn;
    if (nz) {
        red_add_f64(st.xsum + e, xn);
        fixed_colsum_add(mk, st, j, xn);
    }
}

// ------------------------------------------------------------ price step
// drift (may be NULL): drift[1] = max_j (p_j^old - p_j^new)_+ rounded up, an
// order-free max on the bit patterns (the working set's certificate)
__global__ void dual_kernel(int64_t m, double *__restrict__ p, double *__restrict__ pbar,
                            double *__restrict__ cs, double *__restrict__ cs_prev,
                            const double *__restrict__ steps, const int64_t *__restrict__ navg,
                            int it, double *__restrict__ drift) {
    const double sigma = steps[1];
    const Avg w = avg_weights(navg, it);
    double dec = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double c = cs[j];
        const double acc = 2.0 * c - cs_prev[j];  // colsum(2 x^k - x^{k-1})
        const double pold = p[j];
        const double pj = pold + sigma * (acc - 1.0);
        p[j] = pj;
        pbar[j] = w.wold * pbar[j] + w.wnew * pj;
        cs_prev[j] = c;
        dec = fmax(dec, __dsub_ru(pold, pj));
    }
    if (drift) {
        dec = group_max<32>(dec);
        if ((threadIdx.x & 31) == 0) atomic_max_nonneg(drift + 1, dec);
    }
}

// ------------------------------------------------------------ row solves
// Rows of up to MQ_LONG_ROW entries that do not fit the registers: c is kept
// in global memory (the row's x slots) across the sweeps; count-based test.
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
    // the previous utility s0 is usually next to the new root
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

// Rows held in registers (PER entries per lane), warm-started from the
// row's utility after the previous prox s0 (srow; <= 0: none).  The first
// sweep evaluates the active set at s0: if g(s0) >= s0, s0 is below the root
// and the root of that set (or s0) is the next lower bound; otherwise g(s0)
// < s0 is itself a lower bound (g is nonincreasing).  Later sweeps compare
// each lane's active mask with the previous one (a ballot, no reduction) and
// reduce A, B only when the set changed, so a row whose set is already right
// costs one reduction.
template <int G, int PER>
__device__ __forceinline__ double row_root_warm(const double (&c)[PER], const double (&u)[PER],
                                                double tw, double s0, bool active_row,
                                                uint32_t gmask, int *sweeps, bool *ok) {
    auto amask = [&](double q) -> uint32_t {
        uint32_t msk = 0;
#pragma unroll
        for (int e = 0; e < PER; ++e)
            if (u[e] > 0.0 && fma(c[e], q, tw * u[e]) > 0.0) msk |= 1u << e;
        return msk;
    };
    auto sums = [&](uint32_t msk, double &As, double &Bs) {
        double a_ = 0.0, b_ = 0.0;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            if ((msk >> e) & 1u) {
                a_ += u[e] * c[e];
                b_ += u[e] * u[e];
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
            } else if (fma(A0, s0, tw * B0) >= s0 * s0) {  // g(s0) >= s0, no division
                s = fmax(active_root(A0, B0, tw), s0);
                prev = msk;
            } else {
                s = A0 + tw * B0 / s0;  // g(s0): a lower bound, active set unknown
                force = true;
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

// ------------------------------------------------------------ working sets
// Safe screening of the row solve (include/market_eq_b200.h
// mq_state.ws_*).  A zero entry stays zero through the prox iff
// c s + tau w u <= 0 with c = -tau p, i.e. p s >= w u: inactive entries never
// enter the root (masked) nor change.  A row whose zero entries satisfy that
// with margin at the row's root can therefore be solved over the rest —
// its working set: the nonzero entries plus the zero entries within a factor
// gamma of the threshold — and gives exactly the full row's active set,
// root and allocation.  The certificate needs no look at the screened
// entries: their prices have dropped by at most D (drift) since the working
// set was built, so p_j s >= (p_j^ref - D) s >= theta (1 - D / P) s with
// theta = min p^ref / u and P = min p^ref over them.  On C4 the working sets
// hold ~2.5 % of the entries and the certificate holds for all but ~1,600 of
// the 10^7 rows per iteration (tools/ws_waste.py, tools/ws_stats.py): one
// price gather in ~40 instead of every entry's.
// The factor is per row (mq_state.ws_lvl): a row whose certificate failed
// is rebuilt one level wider, a row with more working entries than slots one
// level narrower, and every row one level narrower when all working sets
// are rebuilt (after a restart).  Narrow sets are cheap; rows whose prices
// move fast widen theirs instead of failing every few iterations.
#ifndef MQ_WS_G0
#define MQ_WS_G0 1.001
#endif
#ifndef MQ_WS_G1
#define MQ_WS_G1 1.005
#endif
#ifndef MQ_WS_G2
#define MQ_WS_G2 1.02
#endif
#ifndef MQ_WS_G3
#define MQ_WS_G3 1.06
#endif
#ifndef MQ_WS_POOL_GAMMA
#define MQ_WS_POOL_GAMMA 1.03  // the medium / long rows' pools
#endif
__device__ __forceinline__ double ws_gamma(int lvl) {
    return lvl <= 0 ? MQ_WS_G0 : lvl == 1 ? MQ_WS_G1 : lvl == 2 ? MQ_WS_G2 : MQ_WS_G3;
}
__device__ __forceinline__ int ws_level(const mq_state &st, int64_t i) {
    return st.ws_lvl ? (int)st.ws_lvl[i] : 2;
}
#ifndef MQ_WS_MARGIN
#define MQ_WS_MARGIN 1e-12
#endif

// slot k of row i: a warp's 32 consecutive rows read slot k as one run
__device__ __forceinline__ int64_t ws_at(int64_t i, int k) {
    MQ_CHECK(i >= 0 && k >= 0 && k < MQ_WS_SLOTS);
    return (((i >> 5) * MQ_WS_SLOTS + k) << 5) + (i & 31);
}

// Append `row` to this iteration's full-solve list (warp-aggregated).  The
// list order is irrelevant to the results: rows are independent and the
// column sums are order-free.
__device__ __forceinline__ void ws_push(const mq_state &st, bool push, int64_t row) {
    const uint32_t b = __ballot_sync(MQ_FULL, push);
    if (!b) return;
    const int wl = threadIdx.x & 31;
    const int leader = __ffs(b) - 1;
    int base = 0;
    if (wl == leader) base = atomicAdd(st.blk_done + 3, __popc(b));
    base = __shfl_sync(MQ_FULL, base, leader);
    if (push) {
        MQ_CHECK(row >= 0 && base >= 0);
        st.ws_list[base + __popc(b & ((1u << wl) - 1u))] = (int32_t)row;
    }
}

// price-decrease bound of this iteration: C + dec, rounded up (the value the
// column-sum kernel stores as the next C)
__device__ __forceinline__ double drift_now(const mq_state &st) {
    return __dadd_ru(st.drift[0], st.drift[1]);
}

// Backoff of a pooled (medium / long) row, in its mq_state.ws_lvl byte
// (unused by those rows otherwise): low 5 bits = iterations left to solve
// the row in full without a pool (no screened attempt, no rebuild: the
// pool is marked missing), high 3 bits = level L.  A failed certificate or
// an overfull rebuild raises L (at most 5) and skips the next 2^L - 1
// iterations; a passing certificate lowers L.  Where the pools do not pay
// (prices oscillating in an exchange's late inner solves, or more working
// entries than the pool holds) the attempt and the rebuild — which
// re-gathers every entry's price — are overhead on top of the full solve.
__device__ __forceinline__ bool pool_attempt(const mq_state &st, int64_t i) {
    return !st.ws_lvl || (st.ws_lvl[i] & 31u) == 0;
}
__device__ __forceinline__ void pool_skipped(const mq_state &st, int64_t i) {
    if (st.ws_lvl) st.ws_lvl[i] = (uint8_t)(st.ws_lvl[i] - 1u);  // countdown > 0
}
// returns the iterations the row now skips (0: rebuild at once, as before
// any backoff: a first failure costs nothing extra)
__device__ __forceinline__ int pool_outcome(const mq_state &st, int64_t i, bool pass) {
    if (!st.ws_lvl) return 0;
    int lv = st.ws_lvl[i] >> 5;
    if (pass) {
        if (lv) st.ws_lvl[i] = (uint8_t)((lv - 1) << 5);
        return 0;
    }
#ifndef MQ_POOL_LSTEP
#define MQ_POOL_LSTEP 1
#endif
    lv = lv + MQ_POOL_LSTEP < 6 ? lv + MQ_POOL_LSTEP : 6;
    const int skip = lv > 1 ? (1 << (lv - 1)) - 1 : 0;  // 0, 1, 3, 7, 15, 31
    st.ws_lvl[i] = (uint8_t)((lv << 5) | skip);
    return skip;
}

// Rebuild row i's working set after its full solve (G lanes, entry t = lane
// + G e in register e): the nonzero entries and the zero entries near the
// threshold (p s < gamma w u) take slots in ascending entry order; theta =
// min p / u and P = min p over the rest, C = the drift now.  More than
// MQ_WS_SLOTS working entries: h = -2 (solved in full next time).
template <int G, int RP>
__device__ __forceinline__ void ws_build(const mq_state &st, int64_t i, int lane, int gsub,
                                         bool build, int len, double w, double s, double cnow,
                                         const double (&u)[RP], const double (&pv)[RP],
                                         const double (&xn)[RP], const int (&jc)[RP],
                                         double gamma) {
    constexpr int K = MQ_WS_SLOTS;
    const double gw = gamma * w;
    int before = 0, rank[RP];
    uint32_t hot = 0;
    // smallest p / u over the screened entries: the pair is picked by
    // cross-multiplication and divided once (rounded down, less 2 ulp); a
    // pick off by an ulp is far inside the certificate's 1e-12 margin
    double bp = CUDART_INF, bu = 1.0, pm = CUDART_INF;
#pragma unroll
    for (int e = 0; e < RP; ++e) {
        const int t = lane + e * G;
        const bool in = build && t < len;
        const bool hb = in && (xn[e] > 0.0 || pv[e] * s < gw * u[e]);
        if (hb) hot |= 1u << e;
        if (in && !hb) {
            if (pv[e] * bu < bp * u[e]) {
                bp = pv[e];
                bu = u[e];
            }
            pm = fmin(pm, pv[e]);
        }
        const uint32_t bal = G == 32 ? __ballot_sync(MQ_FULL, hb)
                                     : (__ballot_sync(MQ_FULL, hb) >> (gsub * G)) & ((1u << (G & 31)) - 1u);
        rank[e] = before + __popc(bal & ((1u << lane) - 1u));
        before += __popc(bal);
    }
    double th = bp == CUDART_INF ? CUDART_INF : __ddiv_rd(bp, bu) * (1.0 - 4e-16);
    th = group_min<G>(th);
    pm = group_min<G>(pm);
    if (!build) return;
    if (before <= K) {
#pragma unroll
        for (int e = 0; e < RP; ++e) {
            if ((hot >> e) & 1u) {
                MQ_CHECK(rank[e] < before && lane + e * G < len);
                const int64_t at = ws_at(i, rank[e]);
                st.ws_u[at] = u[e];
                st.ws_x[at] = xn[e];
                st.ws_col[at] = jc[e];
                st.ws_pos[at] = (uint8_t)(lane + e * G);
            }
        }
        if (lane == 0) {
            reinterpret_cast<int4 *>(st.ws_hdr)[i] =
                make_int4(before, __float_as_int(__double2float_rd(th)),
                          __float_as_int(__double2float_rd(pm)),
                          __float_as_int(__double2float_rd(cnow)));
            atomicMax(st.ws_kmax + (i >> 5), before);
        }
    } else if (lane == 0) {
        st.ws_hdr[4 * i] = -2;
    }
}

// ------------------------------------------------------------ primal (fused)
template <int ETILE, int RTILE>
struct TileLayout {
    // one stage (every region 16-byte aligned for the bulk copies):
    // u f64 [ETILE+2] | col i32 [ETILE+4] | row_ptr i64 [RTILE+4] | w f64 [RTILE+2]
    // | srow f64 [RTILE+2] | x > 0 flags u8 [ETILE+32]
    static constexpr int kU = 0;
    static constexpr int kCol = kU + (ETILE + 2) * 8;
    static constexpr int kRp = kCol + (ETILE + 4) * 4;
    static constexpr int kW = kRp + (RTILE + 4) * 8;
    static constexpr int kS = kW + (RTILE + 2) * 8;
    static constexpr int kF = kS + (RTILE + 2) * 8;
    static constexpr int kStage = (kF + ETILE + 32 + 127) / 128 * 128;
    static_assert(kCol % 16 == 0 && kRp % 16 == 0 && kW % 16 == 0 && kS % 16 == 0 && kF % 16 == 0,
                  "bulk-copy destinations must be 16-byte aligned");
};

// Warps 0..NSW-1 solve rows, warp NSW produces (TMA).  full[s]: stage s has
// landed; empty[s]: every solver warp is done with it.  Solver warps claim
// row pairs from a shared counter, so no solver waits for another inside a
// tile.
template <int G, int NSW, int ETILE, int RTILE, int NSTAGE, bool BUILD>
__global__ void __launch_bounds__((NSW + 1) * 32, 1)
primal_fused_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out,
                    int64_t tile_lo, int64_t tile_hi, int *tile_ctr) {
    using L = TileLayout<ETILE, RTILE>;
    MQ_PROF_DECL();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NSTAGE * L::kStage);
    uint64_t *empty = full + NSTAGE;
    int64_t *stile = reinterpret_cast<int64_t *>(empty + NSTAGE);  // tile held by each stage
    int64_t *smeta = stile + NSTAGE;                               // its r0, r1, e0 per stage
    int *claim = reinterpret_cast<int *>(smeta + 3 * NSTAGE);
    constexpr int GPW = 32 / G;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, wl = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NSW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == NSW) {  // ---------------------------------------- producer
        if (wl == 0) {
            const uint64_t pol = policy_evict_first();
            // tiles are claimed dynamically (global counter, MQ_CLAIM at a
            // time); the next tile's claim and metadata are fetched one step
            // ahead so the producer never waits on a dependent global load
            int64_t batch = tile_lo + atomicAdd(tile_ctr, MQ_CLAIM);
            int bpos = 0;
            auto next_tile = [&]() -> int64_t {
                if (bpos == MQ_CLAIM) {
                    batch = tile_lo + atomicAdd(tile_ctr, MQ_CLAIM);
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
            for (int64_t j = 0;; ++j) {
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
                if (k >= tile_hi) {  // sentinel: consumers leave
                    stile[s] = -1;
                    mbar_expect_tx(&full[s], 0);
                    break;
                }
                const int64_t r0 = m01.x, r1 = m01.y, e0 = m23.x, cnt = m23.y - m23.x;
                stile[s] = k;
                smeta[3 * s] = r0;
                smeta[3 * s + 1] = r1;
                smeta[3 * s + 2] = e0;
                unsigned char *base = smem + s * L::kStage;
                const unsigned char *src_rp, *src_w, *src_s, *src_u, *src_c, *src_f;
                uint32_t brp, bw, b8 = 0, b4 = 0, b1 = 0;
                aligned_span<8>(mk.row_ptr, r0, r1 - r0 + 1, &src_rp, &brp);
                aligned_span<8>(mk.w, r0, r1 - r0, &src_w, &bw);
                aligned_span<8>(st.srow, r0, r1 - r0, &src_s, &bw);
                aligned_span<8>(mk.u, e0, cnt, &src_u, &b8);
                aligned_span<4>(mk.col, e0, cnt, &src_c, &b4);
                aligned_span<1>(st.xflag, e0, cnt, &src_f, &b1);
                mbar_expect_tx(&full[s], brp + 2 * bw + (cnt > 0 ? b8 + b4 + b1 : 0));
                bulk_g2s(base + L::kRp, src_rp, brp, &full[s]);
                bulk_g2s(base + L::kW, src_w, bw, &full[s]);
                bulk_g2s(base + L::kS, src_s, bw, &full[s]);
                if (cnt > 0) {
                    bulk_g2s_hint(base + L::kU, src_u, b8, &full[s], pol);
                    bulk_g2s_hint(base + L::kCol, src_c, b4, &full[s], pol);
                    bulk_g2s_hint(base + L::kF, src_f, b1, &full[s], pol);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------- solvers
    const double tau = st.steps[0];
    const int lane = tid & (G - 1);
    const int gsub = wl / G;
    int my_sweeps = 0;  // per warp and launch: < 2^31
    int my_faults = 0;
    for (int64_t j = 0;; ++j) {
        const int s = (int)(j % NSTAGE);
        {
            MQ_T0();
            mbar_wait(&full[s], (uint32_t)((j / NSTAGE) & 1));
            if (wl == 0) MQ_T1(0);
        }
        if (stile[s] < 0) break;  // sentinel
        const int64_t r0 = smeta[3 * s], r1 = smeta[3 * s + 1];
        const int nrows = (int)(r1 - r0);
        unsigned char *base = smem + s * L::kStage;
        const int lr = (int)(((r0 * 8) & 15) >> 3);
        const int64_t *srp = reinterpret_cast<const int64_t *>(base + L::kRp) + lr;
        const double *sw = reinterpret_cast<const double *>(base + L::kW) + lr;
        const double *ss = reinterpret_cast<const double *>(base + L::kS) + lr;
        const int64_t e0 = srp[0];
        const double *su =
            reinterpret_cast<const double *>(base + L::kU) + (int)(((e0 * 8) & 15) >> 3);
        const int32_t *scol =
            reinterpret_cast<const int32_t *>(base + L::kCol) + (int)(((e0 * 4) & 15) >> 2);
        const uint8_t *sfl = reinterpret_cast<const uint8_t *>(base + L::kF) + (int)(e0 & 15);

        MQ_TA(13, 0, 1);  // tile visits
        for (;;) {
            MQ_TS(tc0);
            int rb = 0;
            if (wl == 0) rb = atomicAdd(&claim[s], GPW);
            rb = __shfl_sync(MQ_FULL, rb, 0);
            MQ_TS(tc1);
            MQ_TA(8, tc0, tc1);
            if (rb >= nrows) break;  // warp-uniform
            MQ_TA(12, 0, 1);         // row pairs
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
            if (__all_sync(MQ_FULL, b - a <= MQ_REG_PER * G)) {
                // ---- row in registers
                constexpr int RP = MQ_REG_PER;
                MQ_TS(tq0);
                MQ_TA(9, tc1, tq0);
                double c[RP], u[RP];
                uint32_t fb = 0;  // entries whose x^k was nonzero
                // every load of the pair is issued before any is consumed: the
                // price gathers and the flagged x loads overlap in one round trip
                double pv[RP], xv[RP];
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    const bool in = t < b;
                    pv[e] = in ? __ldg(st.p + scol[t]) : 0.0;
                    const bool f = in && sfl[t];
                    if (f) fb |= 1u << e;
                    xv[e] = f ? __ldcg(st.x + e0 + t) : 0.0;
                    u[e] = in ? su[t] : 0.0;
                }
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    c[e] = t < b ? xv[e] - tau * pv[e] : 0.0;
                }
                if (x_prev_out) {
#pragma unroll
                    for (int e = 0; e < RP; ++e) {
                        const int t = a + lane + e * G;
                        if (t < b) x_prev_out[e0 + t] = xv[e];
                    }
                }
                const double s0 = has ? ss[r] : 0.0;
                MQ_TS(tq1);
                const uint32_t gmask = G == 32 ? MQ_FULL : (((1u << G) - 1u) << (gsub * G));
                const double sr = row_root_warm<G, RP>(c, u, tw, s0, has, gmask, &nsw, &ok);
                if (has && lane == 0) st.srow[r0 + r] = sr;
                const double inv_s = 1.0 / sr;
                MQ_TS(tq2);
                double xn[RP];
                int jc[RP];
#pragma unroll
                for (int e = 0; e < RP; ++e) {
                    const int t = a + lane + e * G;
                    xn[e] = t < b ? fmax(c[e] + tw * u[e] * inv_s, 0.0) : 0.0;
                    jc[e] = t < b ? scol[t] : 0;
                    if (t < b) put_x(mk, st, e0 + t, jc[e], xn[e], (fb >> e) & 1u);
                }
                if (BUILD) {  // the working sets of every row, rebuilt at once, one level narrower
                    int lvl = has ? ws_level(st, r0 + r) : 0;
                    if (lvl > 0) {
                        --lvl;
                        if (lane == 0 && st.ws_lvl) st.ws_lvl[r0 + r] = (uint8_t)lvl;
                    }
                    ws_build<G, RP>(st, r0 + r, lane, gsub, has, b - a, has ? sw[r] : 0.0, sr,
                                    drift_now(st), u, pv, xn, jc, ws_gamma(lvl));
                }
                MQ_TS(tq3);
                MQ_TA(5, tq0, tq1);
                MQ_TA(6, tq1, tq2);
                MQ_TA(7, tq2, tq3);
            } else {
                // ---- a pair with a medium row (longer than the registers
                // hold): primal_med_kernel solves that row (one slow row here
                // would hold the stage); a short partner row is solved here
                // with c kept in its x slots across the sweeps; batches of
                // MQ_LB entries per lane keep all loads of a batch in flight
                // before its c values are stored over x (the stores could
                // alias the next loads, which would serialize them)
                const bool med = b - a > MQ_REG_PER * G;
                if (med) b = a;
                double *sc = st.x + e0;
                double s0p = 0.0, ap = 0.0, bp = 0.0;
                for (int t0 = a + lane; t0 < b; t0 += MQ_LB * G) {
                    double pv[MQ_LB], xv[MQ_LB];
#pragma unroll
                    for (int q = 0; q < MQ_LB; ++q) {
                        const int t = t0 + q * G;
                        const bool in = t < b;
                        pv[q] = in ? __ldg(st.p + scol[t]) : 0.0;
                        xv[q] = (in && sfl[t]) ? __ldcg(st.x + e0 + t) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < MQ_LB; ++q) {
                        const int t = t0 + q * G;
                        if (t < b) {
                            const double ue = su[t], xe = xv[q];
                            const double ce = xe - tau * pv[q];
                            if (x_prev_out) x_prev_out[e0 + t] = xe;
                            sc[t] = ce;  // this lane's entry only
                            s0p += ue * xe;
                            ap += ue * ce;
                            bp += ue * ue;
                        }
                    }
                }
                const double s0 = group_sum<G>(s0p);
                const double A = group_sum<G>(ap);
                const double B = group_sum<G>(bp);
                const double sr =
                    row_root_exact<G>(su, sc, a, b, lane, tw, s0, A, B, has, &nsw, &ok);
                if (has && !med && lane == 0) {
                    st.srow[r0 + r] = sr;
                    if (BUILD) st.ws_hdr[4 * (r0 + r)] = -1;  // full solve next time
                }
                const double inv_s = 1.0 / sr;
                for (int t0 = a + lane; t0 < b; t0 += MQ_LB * G) {
                    double cv[MQ_LB];
#pragma unroll
                    for (int q = 0; q < MQ_LB; ++q) {
                        const int t = t0 + q * G;
                        cv[q] = t < b ? sc[t] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < MQ_LB; ++q) {
                        const int t = t0 + q * G;
                        if (t < b)  // x held c: rewrite every entry
                            put_x(mk, st, e0 + t, scol[t], fmax(cv[q] + tw * su[t] * inv_s, 0.0),
                                  true);
                    }
                }
            }
            if (has && b > a && lane == 0) {
                my_sweeps += nsw;
                if (!ok) ++my_faults;
            }
        }
        MQ_TS(te0);
        __syncwarp();
        if (wl == 0) mbar_arrive(&empty[s]);
        {
            MQ_TS(te1);
            MQ_TA(10, te0, te1);
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

// Sums of three values over the CTA, every thread gets the totals.  Two
// slot buffers alternate (phase), so one barrier per call suffices: a
// buffer is rewritten two calls later, after every thread has passed the
// barrier of the call in between.
__device__ __forceinline__ void block_sum3(double &a, double &b, double &c, double *sm /*[192]*/,
                                           int &phase) {
    a = group_sum<32>(a);
    b = group_sum<32>(b);
    c = group_sum<32>(c);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    double *buf = sm + 96 * (phase & 1);
    ++phase;
    if (lane == 0) {
        buf[warp] = a;
        buf[32 + warp] = b;
        buf[64 + warp] = c;
    }
    __syncthreads();
    double ra = 0.0, rb = 0.0, rc = 0.0;
    if (lane < nw) {
        ra = buf[lane];
        rb = buf[32 + lane];
        rc = buf[64 + lane];
    }
    a = group_sum<32>(ra);
    b = group_sum<32>(rb);
    c = group_sum<32>(rc);
}

// Maxima of three values over the CTA (block_sum3's pattern).
__device__ __forceinline__ void block_max3(double &a, double &b, double &c, double *sm /*[192]*/,
                                           int &phase) {
    a = group_max<32>(a);
    b = group_max<32>(b);
    c = group_max<32>(c);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    double *buf = sm + 96 * (phase & 1);
    ++phase;
    if (lane == 0) {
        buf[warp] = a;
        buf[32 + warp] = b;
        buf[64 + warp] = c;
    }
    __syncthreads();
    double ra = -CUDART_INF, rb = -CUDART_INF, rc = -CUDART_INF;
    if (lane < nw) {
        ra = buf[lane];
        rb = buf[32 + lane];
        rc = buf[64 + lane];
    }
    a = group_max<32>(ra);
    b = group_max<32>(rb);
    c = group_max<32>(rc);
}

// One CTA per long row (rows claimed longest first from a global counter).
// The row's first MQ_LONG_CAP entries stay in shared memory across the
// sweeps (u, c = x - tau p[col], col, was-nonzero flag: 21 bytes per entry),
// so a long row streams its u / col / flags once and its x only where
// flagged, like a tile row; entries past the cap keep c in their x slots.
// Entry k of the row belongs to thread k mod MQ_LONG_THREADS in every pass,
// so each thread re-reads only what it wrote.
template <int T, int CAP>
struct LongSmem {
    static constexpr int kU = 0, kC = CAP * 8, kJ = 2 * CAP * 8, kP = kJ + CAP * 4;
    static constexpr int kF = kP + CAP * 4;
    static constexpr int kBytes = kF + CAP;
};

template <int T, int CAP>
__global__ void __launch_bounds__(T, MQ_LONG_PER_SM)
primal_long_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out,
                   int listed) {
    using L = LongSmem<T, CAP>;
    extern __shared__ __align__(16) unsigned char lsm[];
    double *s_u = reinterpret_cast<double *>(lsm + L::kU);
    double *s_c = reinterpret_cast<double *>(lsm + L::kC);
    int32_t *s_j = reinterpret_cast<int32_t *>(lsm + L::kJ);
    int32_t *s_p = reinterpret_cast<int32_t *>(lsm + L::kP);  // working-set positions
    uint8_t *s_f = lsm + L::kF;
    __shared__ double sm[192];
    __shared__ int64_t claimed;
    __shared__ int s_attempt;  // the row's pool backoff, read once for the block
    __shared__ int s_skip;     // the iterations a failed attempt now skips
    __shared__ int wtot[T / 32 + 1];  // per-warp counts of a working-set rebuild chunk
    const double cnow = st.pl_hdr ? drift_now(st) : 0.0;
    int phase = 0;
    const double tau = st.steps[0];
    const int tid = threadIdx.x;
    int64_t my_sweeps = 0;
    int my_faults = 0;
    constexpr int LB = MQ_LONG_LB;
    for (;;) {
        __syncthreads();  // the previous row's shared-memory reads are done
        if (tid == 0) {
            claimed = atomicAdd(st.blk_done + 1, 1);
            const int64_t nr = listed ? *(volatile int32_t *)(st.blk_done + 7) : mk.nlong;
            s_attempt = claimed < nr
                            ? (int)pool_attempt(st, mk.long_rows[listed ? (int64_t)st.pl_list[claimed]
                                                                        : claimed])
                            : 1;
        }
        __syncthreads();
        // listed: only the rows primal_long_ws_kernel left (pool too large
        // for a warp, missing, or its certificate failed)
        const int64_t nrows = listed ? *(volatile int32_t *)(st.blk_done + 7) : mk.nlong;
        if (claimed >= nrows) break;
        const int64_t r = listed ? (int64_t)st.pl_list[claimed] : claimed;
        MQ_CHECK(r >= 0 && r < mk.nlong);
        const int64_t i = mk.long_rows[r];
        MQ_CHECK(i >= 0 && i < mk.n);
        const int64_t a = mk.row_ptr[i];
        const int len = (int)(mk.row_ptr[i + 1] - a);
        MQ_CHECK(a >= 0 && a + len <= mk.nnz);
        const int ns = len < CAP ? len : CAP;
        const double wi = mk.w[i];
        const double tw = tau * wi;
        double *__restrict__ gx = st.x + a;
        bool failed_here = false;  // a screened attempt failed this iteration (block-uniform)
        // ---- screened solve over the row's working set (pool r): the same
        // certificate as the short rows'
        if (st.pl_hdr && !x_prev_out) {
            const int4 hd = reinterpret_cast<const int4 *>(st.pl_hdr)[r];
            const int h = hd.x;
            MQ_CHECK(h >= -2 && h <= CAP);
            // a pool the warp pass could hold already failed there (or was
            // skipped by its backoff, which this kernel applies itself to
            // the larger pools)
            // (the backoff countdown is the warp pass's to advance when listed)
            const bool attempt = !(listed && h <= MQ_LONG_WCAP) && s_attempt;
            if (h >= 0 && attempt) {
                const int64_t po = r * (int64_t)CAP;
                double s0w = 0.0, Aw = 0.0, Bw = 0.0;
                for (int k = tid; k < h; k += T) {
                    const double ue = st.pl_u[po + k], xe = st.pl_x[po + k];
                    const int j = st.pl_col[po + k];
                    MQ_CHECK(j >= 0 && j < mk.m && st.pl_pos[po + k] < len);
                    const double ce = xe - tau * __ldg(st.p + j);
                    s_u[k] = ue;
                    s_c[k] = ce;
                    s_j[k] = j;
                    s_p[k] = st.pl_pos[po + k];
                    s_f[k] = xe > 0.0;
                    s0w += ue * xe;
                    Aw += ue * ce;
                    Bw += ue * ue;
                }
                block_sum3(s0w, Aw, Bw, sm, phase);
                double sw = active_root(Aw, Bw, tw);
                int prev = h, nsw = 0;
                bool ok = false;
                auto wsweep = [&](double q, double &As, double &Bs, double &cnt) {
                    As = Bs = cnt = 0.0;
                    for (int k = tid; k < h; k += T) {
                        const double ue = s_u[k], ce = s_c[k];
                        if (fma(ce, q, tw * ue) > 0.0) {
                            As += ue * ce;
                            Bs += ue * ue;
                            cnt += 1.0;
                        }
                    }
                    block_sum3(As, Bs, cnt, sm, phase);
                };
                if (s0w > sw) {
                    double A0, B0, k0;
                    wsweep(s0w, A0, B0, k0);
                    ++nsw;
                    const double g0 = A0 + tw * B0 / s0w;
                    if (g0 >= s0w) {
                        sw = fmax(active_root(A0, B0, tw), s0w);
                        prev = (int)k0;
                    } else if (g0 > sw) {
                        sw = g0;
                        prev = -1;
                    }
                }
                for (int k = 0; k < kMaxSweeps && !ok; ++k) {
                    double As, Bs, kc;
                    wsweep(sw, As, Bs, kc);
                    ++nsw;
                    const int cnt = (int)kc;
                    if (cnt == prev || cnt == 0) {
                        ok = cnt != 0 || h == 0;
                        break;
                    }
                    sw = fmax(active_root(As, Bs, tw), sw);
                    prev = cnt;
                }
                bool pass = false;
                if (ok && h > 0) {
                    const double th = (double)__int_as_float(hd.y), pm = (double)__int_as_float(hd.z);
                    const double D = fmax(__dsub_ru(cnow, (double)__int_as_float(hd.w)), 0.0);
                    const double lhs = __dmul_rd(__dmul_rd(th, sw), __dsub_rd(pm, D));
                    const double rhs = __dmul_ru(__dmul_ru(wi, pm), 1.0 + MQ_WS_MARGIN);
                    pass = lhs >= rhs && pm > D;
                }
                if (pass) {  // block-uniform
                    const double inv_s = 1.0 / sw;
                    for (int k = tid; k < h; k += T) {
                        const double xn = fmax(s_c[k] + tw * s_u[k] * inv_s, 0.0);
                        if (xn > 0.0 || s_f[k]) st.pl_x[po + k] = xn;
                        put_x(mk, st, a + s_p[k], s_j[k], xn, s_f[k]);
                    }
                    if (tid == 0) {
                        my_sweeps += nsw;
                        st.srow[i] = sw;
                        pool_outcome(st, i, true);
                    }
                    continue;  // the next row (the loop head syncs)
                }
                if (tid == 0) s_skip = h > 0 ? pool_outcome(st, i, false) : 0;
                __syncthreads();  // the full solve below reuses the shared arrays
                failed_here = s_skip > 0;  // backing off from now on (block-uniform)
            }
        }
        double s0 = 0.0, A = 0.0, B = 0.0;
        for (int k0 = tid; k0 < len; k0 += LB * T) {
            int jv[LB];
            bool fv[LB];
            double uv[LB], pv[LB], xv[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {  // every load of the batch before any store
                const int k = k0 + q * T;
                const bool in = k < len;
                jv[q] = in ? __ldg(mk.col + a + k) : 0;
                fv[q] = in && __ldg(st.xflag + a + k);
                uv[q] = in ? __ldg(mk.u + a + k) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int k = k0 + q * T;
                pv[q] = k < len ? __ldg(st.p + jv[q]) : 0.0;
                // past the cap the x slots carry c: read them whole
                xv[q] = (fv[q] || (k >= CAP && k < len)) ? __ldcg(gx + k) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int k = k0 + q * T;
                if (k < len) {
                    const double ce = xv[q] - tau * pv[q];
                    if (x_prev_out) x_prev_out[a + k] = xv[q];
                    if (k < CAP) {
                        s_u[k] = uv[q];
                        s_c[k] = ce;
                        s_j[k] = jv[q];
                        s_f[k] = fv[q];
                    } else {
                        gx[k] = ce;
                    }
                    s0 += uv[q] * xv[q];
                    A += uv[q] * ce;
                    B += uv[q] * uv[q];
                }
            }
        }
        block_sum3(s0, A, B, sm, phase);
        double s = active_root(A, B, tw);
        int prev_cnt = len;
        int sweeps = 0;
        bool done = false;
        auto sweep = [&](double q, double &As, double &Bs, double &cnt) {
            As = 0.0;
            Bs = 0.0;
            cnt = 0.0;
            for (int k = tid; k < ns; k += T) {
                const double ue = s_u[k], ce = s_c[k];
                if (fma(ce, q, tw * ue) > 0.0) {
                    As += ue * ce;
                    Bs += ue * ue;
                    cnt += 1.0;
                }
            }
            for (int k = CAP + tid; k < len; k += T) {
                const double ue = __ldg(mk.u + a + k), ce = gx[k];
                if (fma(ce, q, tw * ue) > 0.0) {
                    As += ue * ce;
                    Bs += ue * ue;
                    cnt += 1.0;
                }
            }
            block_sum3(As, Bs, cnt, sm, phase);
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
        if (tid == 0) {
            my_sweeps += sweeps;
            if (!done) ++my_faults;
            st.srow[i] = s;
        }
        const double inv_s = 1.0 / s;
        if (st.pl_hdr && (!s_attempt || failed_here)) {  // backing off: pool missing
            if (tid == 0) {
                if (!listed && !s_attempt) pool_skipped(st, i);
                st.pl_hdr[4 * r] = -1;
            }
        }
        if (st.pl_hdr && s_attempt && !failed_here) {
            // write-back fused with the working-set rebuild, chunk by chunk of
            // T entries so the block scan ranks working entries in ascending
            // position: nonzero entries and zero entries near the threshold
            const int64_t po = r * (int64_t)CAP;
            const double gw = MQ_WS_POOL_GAMMA * wi;
            const int lane = tid & 31, warp = tid >> 5;
            int base = 0;
            double bp = CUDART_INF, bu = 1.0, pmn = CUDART_INF;
            for (int k0 = 0; k0 < len; k0 += T) {
                const int k = k0 + tid;
                bool hot = false;
                double ue = 0.0, xn = 0.0, pj = 0.0;
                int j = 0;
                if (k < len) {
                    double ce;
                    bool was;
                    if (k < CAP) {
                        ue = s_u[k];
                        ce = s_c[k];
                        j = s_j[k];
                        was = s_f[k];
                    } else {
                        ue = __ldg(mk.u + a + k);
                        ce = gx[k];
                        j = __ldg(mk.col + a + k);
                        was = true;  // the x slot held c: rewrite it
                    }
                    xn = fmax(ce + tw * ue * inv_s, 0.0);
                    put_x(mk, st, a + k, j, xn, was);
                    pj = __ldg(st.p + j);
                    hot = xn > 0.0 || pj * s < gw * ue;
                    if (!hot) {
                        if (pj * bu < bp * ue) {
                            bp = pj;
                            bu = ue;
                        }
                        pmn = fmin(pmn, pj);
                    }
                }
                const uint32_t bal = __ballot_sync(MQ_FULL, hot);
                if (lane == 0) wtot[warp] = __popc(bal);
                __syncthreads();
                int before = 0, total = 0;
                for (int q = 0; q < T / 32; ++q) {
                    if (q < warp) before += wtot[q];
                    total += wtot[q];
                }
                const int rank = base + before + __popc(bal & ((1u << lane) - 1u));
                if (hot && rank < CAP) {
                    st.pl_u[po + rank] = ue;
                    st.pl_x[po + rank] = xn;
                    st.pl_col[po + rank] = j;
                    st.pl_pos[po + rank] = k;
                }
                base += total;
                __syncthreads();  // wtot is rewritten by the next chunk
            }
            double th = bp == CUDART_INF ? CUDART_INF : __ddiv_rd(bp, bu) * (1.0 - 4e-16);
            double dummy = 0.0;
            th = -th;
            pmn = -pmn;  // block max of the negatives = block min (fixed order)
            block_max3(th, pmn, dummy, sm, phase);
            th = -th;
            pmn = -pmn;
            if (tid == 0) {
                reinterpret_cast<int4 *>(st.pl_hdr)[r] =
                    base <= CAP ? make_int4(base, __float_as_int(__double2float_rd(th)),
                                            __float_as_int(__double2float_rd(pmn)),
                                            __float_as_int(__double2float_rd(cnow)))
                                : make_int4(-2, 0, 0, 0);
                if (base > CAP) pool_outcome(st, i, false);
            }
            continue;
        }
        for (int k = tid; k < ns; k += T)
            put_x(mk, st, a + k, s_j[k], fmax(s_c[k] + tw * s_u[k] * inv_s, 0.0), s_f[k]);
        for (int k0 = CAP + tid; k0 < len; k0 += LB * T) {
            double cv[LB], uv[LB];
            int jv[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int k = k0 + q * T;
                const bool in = k < len;
                cv[q] = in ? gx[k] : 0.0;
                uv[q] = in ? __ldg(mk.u + a + k) : 0.0;
                jv[q] = in ? __ldg(mk.col + a + k) : 0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int k = k0 + q * T;
                if (k < len)  // the x slot held c: rewrite it
                    put_x(mk, st, a + k, jv[q], fmax(cv[q] + tw * uv[q] * inv_s, 0.0), true);
            }
        }
    }
    __shared__ int64_t red[32];
    const int64_t tot = block_sum_i64(my_sweeps, red);
    if (tid == 0 && tot) atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)tot);
    const int64_t fl = block_sum_i64((int64_t)my_faults, red);
    if (tid == 0 && fl) atomicAdd((unsigned long long *)st.faults, (unsigned long long)fl);
}

// Long rows' screened pass, a warp per row: a pool of up to MQ_LONG_WCAP
// entries is solved in registers (MQ_LONG_WCAP / 32 per lane) with the
// certificate of the short rows; every other row (no pool, a larger one, a
// failed certificate) is listed for primal_long_kernel.  Most long rows
// work over a few dozen entries: a whole CTA per row idles on them.
static_assert(MQ_LONG_WCAP % 32 == 0 && MQ_LONG_WCAP <= MQ_LONG_CAP, "warp pool cap");
__global__ void __launch_bounds__(256)
primal_long_ws_kernel(const mq_market mk, const mq_state st, int it) {
    constexpr int G = 32, PC = MQ_LONG_WCAP / 32;
    const double tau = st.steps[0];
    const int lane = threadIdx.x & 31;
    const double cnow = drift_now(st);
    int my_sweeps = 0;
    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(st.blk_done + 6, 1);
        r = __shfl_sync(MQ_FULL, r, 0);
        if (r >= mk.nlong) break;  // warp-uniform
        const int64_t i = mk.long_rows[r];
        MQ_CHECK(i >= 0 && i < mk.n);
        const int64_t e0 = mk.row_ptr[i];
        const int len = (int)(mk.row_ptr[i + 1] - e0);
        const double wi = mk.w[i];
        const double tw = tau * wi;
        const int4 hd = reinterpret_cast<const int4 *>(st.pl_hdr)[r];
        const int h = hd.x;
        MQ_CHECK(h >= -2 && h <= MQ_LONG_CAP);
        bool solved = false;
        const bool attempt = __shfl_sync(MQ_FULL, (int)pool_attempt(st, i), 0) != 0;
        if (!attempt && lane == 0) pool_skipped(st, i);
        if (attempt && h > 0 && h <= MQ_LONG_WCAP) {  // warp-uniform
            const int64_t po = r * (int64_t)MQ_LONG_CAP;
            double c[PC], u[PC], xk[PC];
            int jc[PC], ps[PC];
#pragma unroll
            for (int e = 0; e < PC; ++e) {
                const int k = lane + e * G;
                const bool in = k < h;
                u[e] = in ? __ldcg(st.pl_u + po + k) : 0.0;
                xk[e] = in ? __ldcg(st.pl_x + po + k) : 0.0;
                jc[e] = in ? __ldcg(st.pl_col + po + k) : 0;
                ps[e] = in ? __ldcg(st.pl_pos + po + k) : 0;
                MQ_CHECK(!in || (jc[e] >= 0 && jc[e] < mk.m && ps[e] >= 0 && ps[e] < len));
            }
#pragma unroll
            for (int e = 0; e < PC; ++e)
                c[e] = xk[e] - tau * (lane + e * G < h ? __ldg(st.p + jc[e]) : 0.0);
            int nsw = 0;
            bool ok = true;
            const double sw = row_root_warm<G, PC>(c, u, tw, st.srow[i], true, MQ_FULL, &nsw, &ok);
            const double th = (double)__int_as_float(hd.y), pm = (double)__int_as_float(hd.z);
            const double D = fmax(__dsub_ru(cnow, (double)__int_as_float(hd.w)), 0.0);
            const double lhs = __dmul_rd(__dmul_rd(th, sw), __dsub_rd(pm, D));
            const double rhs = __dmul_ru(__dmul_ru(wi, pm), 1.0 + MQ_WS_MARGIN);
            if (ok && lhs >= rhs && pm > D) {  // warp-uniform
                const double inv_s = 1.0 / sw;
#pragma unroll
                for (int e = 0; e < PC; ++e) {
                    const int k = lane + e * G;
                    if (k < h) {
                        const double xn = fmax(c[e] + tw * u[e] * inv_s, 0.0);
                        const bool was = xk[e] > 0.0;
                        if (xn > 0.0 || was) st.pl_x[po + k] = xn;
                        put_x(mk, st, e0 + ps[e], jc[e], xn, was);
                    }
                }
                if (lane == 0) {
                    st.srow[i] = sw;
                    my_sweeps += nsw;
                    pool_outcome(st, i, true);
                }
                solved = true;
            } else if (lane == 0) {
                pool_outcome(st, i, false);
            }
        }
        if (!solved && lane == 0) st.pl_list[atomicAdd(st.blk_done + 7, 1)] = r;
    }
    if (lane == 0 && my_sweeps)
        atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)my_sweeps);
}

// Medium rows (MQ_REG_ROW < length <= MQ_LONG_ROW, listed longest first in
// mk.med_rows): one warp per row, rows claimed from a global counter.  c is
// kept in the row's x slots across the sweeps (each lane re-reads only the
// entries it wrote); u, col and the flags are read straight from global
// memory, MQ_LB entries per lane in flight.
#ifndef MQ_MED_LB
#define MQ_MED_LB MQ_LB  // entries per lane batched ahead of the stores (medium rows)
#endif
#ifdef MQ_MED_MINB  // tuning: resident 256-thread CTAs per SM to build for
__global__ void __launch_bounds__(256, MQ_MED_MINB)
#else
__global__ void __launch_bounds__(256)
#endif
primal_med_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out,
                  int64_t nrows) {
    constexpr int G = 32, LB = MQ_MED_LB, PC = MQ_MED_CAP / G;
    const double tau = st.steps[0];
    const int lane = threadIdx.x & 31;
    const double cnow = st.pm_hdr ? drift_now(st) : 0.0;
    int my_sweeps = 0, my_faults = 0;
    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(st.blk_done + 2, 1);
        r = __shfl_sync(MQ_FULL, r, 0);
        if (r >= nrows) break;  // warp-uniform
        const int64_t i = mk.med_rows[r];
        MQ_CHECK(i >= 0 && i < mk.n);
        const int64_t e0 = mk.row_ptr[i];
        const int len = (int)(mk.row_ptr[i + 1] - e0);
        MQ_CHECK(e0 >= 0 && e0 + len <= mk.nnz);
        const double wi = mk.w[i];
        const double tw = tau * wi;
        const double *__restrict__ su = mk.u + e0;
        const int32_t *__restrict__ cl = mk.col + e0;
        const uint8_t *__restrict__ fl = st.xflag + e0;
        double *sc = st.x + e0;
        // rows longer than MQ_WS_MAX_ROW have a pool (the leading nmed_long)
        const bool pooled = st.pm_hdr != nullptr && r < mk.nmed_long;
        const int64_t po = r * (int64_t)MQ_MED_CAP;
        const bool fresh =  // lane 0's read for the whole warp (lane 0 writes it below)
            __shfl_sync(MQ_FULL, (int)(pooled && pool_attempt(st, i)), 0) != 0;
        const bool attempt = fresh && !x_prev_out;
        if (pooled && !fresh && lane == 0) {  // backing off: solved in full, pool missing
            pool_skipped(st, i);
            st.pm_hdr[4 * r] = -1;
        }
        bool failed = false;  // this iteration's certificate failed: back off now
        if (attempt) {
            // screened solve over the pool, in registers; the certificate of
            // the short rows
            const int4 hd = reinterpret_cast<const int4 *>(st.pm_hdr)[r];
            const int h = hd.x;
            MQ_CHECK(h >= -2 && h <= MQ_MED_CAP);
            if (h > 0) {
                double c[PC], u[PC], xk[PC];
                int jc[PC], ps[PC];
#pragma unroll
                for (int e = 0; e < PC; ++e) {
                    const int k = lane + e * G;
                    const bool in = k < h;
                    u[e] = in ? __ldcg(st.pm_u + po + k) : 0.0;
                    xk[e] = in ? __ldcg(st.pm_x + po + k) : 0.0;
                    jc[e] = in ? __ldcg(st.pm_col + po + k) : 0;
                    ps[e] = in ? __ldcg(st.pm_pos + po + k) : 0;
                    MQ_CHECK(!in || (jc[e] >= 0 && jc[e] < mk.m && ps[e] >= 0 && ps[e] < len));
                }
#pragma unroll
                for (int e = 0; e < PC; ++e)
                    c[e] = xk[e] - tau * (lane + e * G < h ? __ldg(st.p + jc[e]) : 0.0);
                int nsw = 0;
                bool ok = true;
                const double sw = row_root_warm<G, PC>(c, u, tw, st.srow[i], true, MQ_FULL, &nsw, &ok);
                const double th = (double)__int_as_float(hd.y), pm = (double)__int_as_float(hd.z);
                const double D = fmax(__dsub_ru(cnow, (double)__int_as_float(hd.w)), 0.0);
                const double lhs = __dmul_rd(__dmul_rd(th, sw), __dsub_rd(pm, D));
                const double rhs = __dmul_ru(__dmul_ru(wi, pm), 1.0 + MQ_WS_MARGIN);
                if (ok && lhs >= rhs && pm > D) {  // warp-uniform
                    const double inv_s = 1.0 / sw;
#pragma unroll
                    for (int e = 0; e < PC; ++e) {
                        const int k = lane + e * G;
                        if (k < h) {
                            const double xn = fmax(c[e] + tw * u[e] * inv_s, 0.0);
                            const bool was = xk[e] > 0.0;
                            if (xn > 0.0 || was) st.pm_x[po + k] = xn;
                            put_x(mk, st, e0 + ps[e], jc[e], xn, was);
                        }
                    }
                    if (lane == 0) {
                        st.srow[i] = sw;
                        my_sweeps += nsw;
                        pool_outcome(st, i, true);
                    }
                    continue;
                }
                int skip = 0;
                if (lane == 0) skip = pool_outcome(st, i, false);
                failed = __shfl_sync(MQ_FULL, skip, 0) > 0;  // backing off from now on
            }
        }
        if (failed && lane == 0) st.pm_hdr[4 * r] = -1;  // no rebuild while backing off
        double s0p = 0.0, ap = 0.0, bp = 0.0;
        for (int t0 = lane; t0 < len; t0 += LB * G) {
            double pv[LB], xv[LB], uv[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {  // all loads of the batch before its stores
                const int t = t0 + q * G;
                const bool in = t < len;
                pv[q] = in ? __ldg(st.p + __ldg(cl + t)) : 0.0;
                xv[q] = (in && __ldg(fl + t)) ? __ldcg(sc + t) : 0.0;
                uv[q] = in ? __ldg(su + t) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int t = t0 + q * G;
                if (t < len) {
                    const double ce = xv[q] - tau * pv[q];
                    if (x_prev_out) x_prev_out[e0 + t] = xv[q];
                    sc[t] = ce;  // this lane's entry only
                    s0p += uv[q] * xv[q];
                    ap += uv[q] * ce;
                    bp += uv[q] * uv[q];
                }
            }
        }
        const double s0 = group_sum<G>(s0p);
        const double A = group_sum<G>(ap);
        const double B = group_sum<G>(bp);
        int nsw = 0;
        bool ok = true;
        const double sr = row_root_exact<G>(su, sc, 0, len, lane, tw, s0, A, B, true, &nsw, &ok);
        if (lane == 0) {
            st.srow[i] = sr;
            my_sweeps += nsw;
            if (!ok) ++my_faults;
        }
        const double inv_s = 1.0 / sr;
        if (pooled && fresh && !failed) {
            // write-back fused with the pool rebuild: warp-wide chunks of 32
            // entries in ascending position, ballots rank the working entries
            // (nonzero, or zero with p_j s < gamma w u_j)
            const double gw = MQ_WS_POOL_GAMMA * wi;
            int base = 0;
            double bp = CUDART_INF, bu = 1.0, pmn = CUDART_INF;
            for (int b0 = 0; b0 < len; b0 += LB * G) {  // warp-uniform bounds
                double cv[LB], uv[LB], pv[LB];
                int jv[LB];
#pragma unroll
                for (int q = 0; q < LB; ++q) {
                    const int t = b0 + q * G + lane;
                    const bool in = t < len;
                    cv[q] = in ? sc[t] : 0.0;
                    uv[q] = in ? __ldg(su + t) : 0.0;
                    jv[q] = in ? __ldg(cl + t) : 0;
                }
#pragma unroll
                for (int q = 0; q < LB; ++q)
                    pv[q] = b0 + q * G + lane < len ? __ldg(st.p + jv[q]) : 0.0;
#pragma unroll
                for (int q = 0; q < LB; ++q) {
                    const int t = b0 + q * G + lane;
                    const bool in = t < len;
                    const double xn = in ? fmax(cv[q] + tw * uv[q] * inv_s, 0.0) : 0.0;
                    if (in) put_x(mk, st, e0 + t, jv[q], xn, true);  // x held c
                    const bool hot = in && (xn > 0.0 || pv[q] * sr < gw * uv[q]);
                    if (in && !hot) {
                        if (pv[q] * bu < bp * uv[q]) {
                            bp = pv[q];
                            bu = uv[q];
                        }
                        pmn = fmin(pmn, pv[q]);
                    }
                    const uint32_t bal = __ballot_sync(MQ_FULL, hot);
                    const int rank = base + __popc(bal & ((1u << lane) - 1u));
                    if (hot && rank < MQ_MED_CAP) {
                        st.pm_u[po + rank] = uv[q];
                        st.pm_x[po + rank] = xn;
                        st.pm_col[po + rank] = jv[q];
                        st.pm_pos[po + rank] = t;
                    }
                    base += __popc(bal);
                }
            }
            double th = bp == CUDART_INF ? CUDART_INF : __ddiv_rd(bp, bu) * (1.0 - 4e-16);
            th = group_min<32>(th);
            pmn = group_min<32>(pmn);
            if (lane == 0) {
                reinterpret_cast<int4 *>(st.pm_hdr)[r] =
                    base <= MQ_MED_CAP ? make_int4(base, __float_as_int(__double2float_rd(th)),
                                                   __float_as_int(__double2float_rd(pmn)),
                                                   __float_as_int(__double2float_rd(cnow)))
                                       : make_int4(-2, 0, 0, 0);
                if (base > MQ_MED_CAP) pool_outcome(st, i, false);
            }
            continue;
        }
        for (int t0 = lane; t0 < len; t0 += LB * G) {
            double cv[LB], uv[LB];
            int jv[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int t = t0 + q * G;
                const bool in = t < len;
                cv[q] = in ? sc[t] : 0.0;
                uv[q] = in ? __ldg(su + t) : 0.0;
                jv[q] = in ? __ldg(cl + t) : 0;
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int t = t0 + q * G;
                if (t < len)  // x held c: rewrite every entry
                    put_x(mk, st, e0 + t, jv[q], fmax(cv[q] + tw * uv[q] * inv_s, 0.0), true);
            }
        }
    }
    if (lane == 0 && my_sweeps)
        atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)my_sweeps);
    if (lane == 0 && my_faults)
        atomicAdd((unsigned long long *)st.faults, (unsigned long long)my_faults);
}

// Screened solve over 32-row blocks, one thread per row, fed by a TMA
// producer warp.  The producer claims batches of MQ_WS_SB consecutive blocks
// and bulk-copies each into a shared-memory stage: the rows' headers (h,
// theta, P, C), budgets, warm starts and row offsets, and each block's slots
// 0..kmax-1 (u, x, column, position: one contiguous run per array).  MQ_WS_NC consumer warps claim
// blocks of the current stage and solve one row per thread: the only round
// trip left in a row's chain is the price gather of its working entries.
// The root is the monotone active-set iteration of row_root_warm run
// serially on the thread's row (no shuffles); the certificate
// theta s (P - D) >= w P (1 + margin) is evaluated in directed rounding
// (left side down, right side up).  Rows without a working set, or whose
// certificate fails, go to the full-solve list untouched.
#ifndef MQ_WS_NC
#define MQ_WS_NC 11  // consumer warps per CTA (one CTA per SM; 12 warps: <= 168 registers)
#endif
#ifndef MQ_WS_SB
#define MQ_WS_SB 8  // 32-row blocks per stage
#endif
#ifndef MQ_WS_NST
#define MQ_WS_NST 2  // stages
#endif
template <int K, int SB>
struct WsStage {
    int4 hdr[SB * 32];  // h, theta, P, C (float bits)
    double w[SB * 32];
    double srow[SB * 32];
    long long rp[SB * 32];  // row offsets
    // slots of the stage's SB blocks, block e's slot k of row l at
    // (e * K + k) * 32 + l (the global layout); block e's slots 0..kmax-1
    // arrive with one copy per array
    double u[SB * K * 32];
    double x[SB * K * 32];
    int32_t col[SB * K * 32];
    uint8_t pos[SB * K * 32];
};
using WsStageT = WsStage<MQ_WS_SLOTS, MQ_WS_SB>;
constexpr int kWsSmem =
    MQ_WS_NST * (int)sizeof(WsStageT) + MQ_WS_NST * (2 * 8 + 8 + 4) + 64;
static_assert(sizeof(WsStageT) % 16 == 0, "stage must keep 16-byte alignment");

__global__ void __launch_bounds__((MQ_WS_NC + 1) * 32, 1)
ws_kernel(const mq_market mk, const mq_state st, int it, int force_full) {
    constexpr int K = MQ_WS_SLOTS, SB = MQ_WS_SB, NST = MQ_WS_NST, NC = MQ_WS_NC;
    static_assert(SB <= NC, "every warp takes at most one block per stage visit");
    extern __shared__ __align__(128) unsigned char wsm[];
    WsStageT *stg = reinterpret_cast<WsStageT *>(wsm);
    uint64_t *full = reinterpret_cast<uint64_t *>(wsm + NST * sizeof(WsStageT));
    uint64_t *empty = full + NST;
    int64_t *sblk = reinterpret_cast<int64_t *>(empty + NST);  // first block of each stage
    int *claim = reinterpret_cast<int *>(sblk + NST);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < NST; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], NC);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t nblk = (mk.n + 31) >> 5;
    const int64_t nbatch = (nblk + SB - 1) / SB;

    if (warp == NC) {  // ------------------------------------------- producer
        if (lane == 0) {
            // batches claimed from a global counter one step ahead (dynamic
            // claims balance the CTAs), with their blocks' kmax
            const uint64_t pol = policy_evict_first();
            int *ctr = st.blk_done + 5;
            auto load_km = [&](int64_t bt, int (&km)[SB]) {
                for (int e = 0; e < SB; ++e)
                    km[e] = (bt < nbatch && bt * SB + e < nblk) ? __ldcg(st.ws_kmax + bt * SB + e)
                                                                 : 0;
            };
            int64_t bnx = atomicAdd(ctr, 1);
            int kmn[SB];
            load_km(bnx, kmn);
            for (int64_t j = 0;; ++j) {
                const int q = (int)(j % NST);
                const int64_t bt = bnx;
                int km[SB];
                for (int e = 0; e < SB; ++e) km[e] = kmn[e];
                if (bt < nbatch) {
                    bnx = atomicAdd(ctr, 1);
                    load_km(bnx, kmn);
                }
                if (j >= NST) mbar_wait(&empty[q], (uint32_t)(((j / NST) - 1) & 1));
                claim[q] = 0;
                if (bt >= nbatch) {  // sentinel: the consumers leave
                    sblk[q] = -1;
                    mbar_arrive(&full[q]);
                    break;
                }
                WsStageT &d = stg[q];
                const int64_t b0 = bt * SB, r0 = b0 * 32;
                const int64_t rows = mk.n - r0 < SB * 32 ? mk.n - r0 : SB * 32;
                const int nb = (int)(nblk - b0 < SB ? nblk - b0 : SB);
                sblk[q] = b0;
                const uint32_t b16 = (uint32_t)rows * 16u;
                const uint32_t b8 = ((uint32_t)rows * 8u + 15u) & ~15u;
                uint32_t tx = b16 + 3 * b8;
                for (int e = 0; e < nb; ++e) tx += (uint32_t)km[e] * 32u * (8u + 8u + 4u + 1u);
                mbar_expect_tx(&full[q], tx);
                bulk_g2s(d.hdr, st.ws_hdr + 4 * r0, b16, &full[q]);
                bulk_g2s(d.w, mk.w + r0, b8, &full[q]);
                bulk_g2s(d.srow, st.srow + r0, b8, &full[q]);
                bulk_g2s(d.rp, mk.row_ptr + r0, b8, &full[q]);
                for (int e = 0; e < nb; ++e) {
                    if (!km[e]) continue;
                    const int64_t o = (b0 + e) * K * 32;
                    const int so = e * K * 32;
                    const uint32_t ns = (uint32_t)km[e] * 32u;
#ifndef MQ_WS_HINT
#define MQ_WS_HINT 1  // bit 0: u, bit 1: x, bit 2: col and pos copied evict-first
#endif
                    if (MQ_WS_HINT & 1) bulk_g2s_hint(d.u + so, st.ws_u + o, ns * 8u, &full[q], pol);
                    else bulk_g2s(d.u + so, st.ws_u + o, ns * 8u, &full[q]);
                    if (MQ_WS_HINT & 2) bulk_g2s_hint(d.x + so, st.ws_x + o, ns * 8u, &full[q], pol);
                    else bulk_g2s(d.x + so, st.ws_x + o, ns * 8u, &full[q]);
                    if (MQ_WS_HINT & 4) {
                        bulk_g2s_hint(d.col + so, st.ws_col + o, ns * 4u, &full[q], pol);
                        bulk_g2s_hint(d.pos + so, st.ws_pos + o, ns, &full[q], pol);
                    } else {  // re-read by the write-back: keep them in L2
                        bulk_g2s(d.col + so, st.ws_col + o, ns * 4u, &full[q]);
                        bulk_g2s(d.pos + so, st.ws_pos + o, ns, &full[q]);
                    }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    // A consumer copies its block's rows into registers and releases the
    // stage at once (at most one block per stage and warp: the stage is back
    // with the producer after a shared-memory read, not after the solve);
    // the price gathers and the solve then run from registers.
    const double tau = st.steps[0];
    const double cnow = drift_now(st);
    int my_sweeps = 0;
    for (int64_t j = 0;; ++j) {
        const int q = (int)(j % NST);
        mbar_wait(&full[q], (uint32_t)((j / NST) & 1));
        const int64_t b0 = sblk[q];
        if (b0 < 0) break;
        const WsStageT &d = stg[q];
        int e = 0;
        if (lane == 0) e = atomicAdd(&claim[q], 1);
        e = __shfl_sync(MQ_FULL, e, 0);
        const bool mine = e < SB && b0 + e < nblk;  // warp-uniform
        const int rl = mine ? e * 32 + lane : 0;
        const int so = mine ? e * K * 32 + lane : 0;
        const int64_t i = (b0 + (mine ? e : 0)) * 32 + lane;
        const bool has = mine && i < mk.n;
        int4 hd = make_int4(-3, 0, 0, 0);
        double w = 0.0, s0 = 0.0, u[K], c[K], pv[K];
        int64_t e0 = 0;
        if (mine) {
            hd = d.hdr[rl];
            w = d.w[rl];
            s0 = d.srow[rl];
            e0 = d.rp[rl];
        }
        int h = has ? hd.x : -3;
        MQ_CHECK(h >= -3 && h <= K);
        if (force_full && h != -3) h = -1;
        uint32_t was = 0;  // slots whose x was nonzero
#pragma unroll
        for (int k = 0; k < K; ++k) {  // the price gathers leave before the release
            u[k] = 0.0;
            c[k] = 0.0;  // holds x until the gathers return
            pv[k] = 0.0;
            if (k < h) {
                u[k] = d.u[so + k * 32];
                c[k] = d.x[so + k * 32];
                MQ_CHECK(d.col[so + k * 32] >= 0 && d.col[so + k * 32] < mk.m);
                pv[k] = __ldg(st.p + d.col[so + k * 32]);
                if (c[k] > 0.0) was |= 1u << k;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[q]);
        if (!mine) continue;
        ws_push(st, h == -1 || h == -2, i);
        const bool act = h >= 0;
#pragma unroll
        for (int k = 0; k < K; ++k) c[k] -= tau * pv[k];
        const double tw = tau * w;
        // ---- exact root over the working set (row_root_warm, one thread)
        auto amask = [&](double z) -> uint32_t {
            uint32_t msk = 0;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (u[k] > 0.0 && fma(c[k], z, tw * u[k]) > 0.0) msk |= 1u << k;
            return msk;
        };
        auto sums = [&](uint32_t msk, double &A, double &B) {
            A = 0.0;
            B = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if ((msk >> k) & 1u) {
                    A += u[k] * c[k];
                    B += u[k] * u[k];
                }
        };
        double sr = 1.0;
        int nsw = 0;
        bool ok = act;
        if (act) {
            const bool warm = s0 > 0.0;
            uint32_t prev = amask(warm ? s0 : 0.0);
            double A, B;
            sums(prev, A, B);
            ++nsw;
            bool force = false, done = false;
            if (!warm) {
                if (prev) sr = active_root(A, B, tw);
                done = prev == 0u;
                ok = prev != 0u;
            } else if (fma(A, s0, tw * B) >= s0 * s0) {  // g(s0) >= s0
                sr = fmax(active_root(A, B, tw), s0);
            } else {
                sr = A + tw * B / s0;  // g(s0): a lower bound, active set unknown
                force = true;
            }
            for (int sw = 0; sw < kMaxSweeps && !done; ++sw) {
                const uint32_t msk = amask(sr);
                ++nsw;
                if ((msk == prev && !force) || msk == 0u) {
                    done = true;
                    if (msk == 0u) ok = false;
                } else {
                    sums(msk, A, B);
                    sr = fmax(active_root(A, B, tw), sr);
                    prev = msk;
                    force = false;
                }
            }
            ok = ok && done;
        }
        bool pass = false;
        if (ok) {
            const double th = (double)__int_as_float(hd.y), pm = (double)__int_as_float(hd.z);
            const double D = fmax(__dsub_ru(cnow, (double)__int_as_float(hd.w)), 0.0);
            const double lhs = __dmul_rd(__dmul_rd(th, sr), __dsub_rd(pm, D));
            const double rhs = __dmul_ru(__dmul_ru(w, pm), 1.0 + MQ_WS_MARGIN);
            pass = lhs >= rhs && pm > D;
        }
        ws_push(st, act && !pass, i);
        if (pass) {
            const double inv_s = 1.0 / sr;
            // entries that are or were nonzero: their positions and goods are
            // fetched together (one round trip), then written
            uint32_t wm = was;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k < h && c[k] + tw * u[k] * inv_s > 0.0) wm |= 1u << k;
            int pos[K], jc[K];
            const int64_t wb = ws_at(i, 0);  // slot k at wb + 32 k
#pragma unroll
            for (int k = 0; k < K; ++k) {
                pos[k] = 0;
                jc[k] = 0;
                if ((wm >> k) & 1u) {
                    const int64_t at = wb + (k << 5);
                    pos[k] = __ldcg(st.ws_pos + at);
                    jc[k] = __ldcg(st.ws_col + at);
                    MQ_CHECK(e0 + pos[k] < mk.nnz && jc[k] >= 0 && jc[k] < mk.m);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if ((wm >> k) & 1u) {
                    // the slot is authoritative; x and its flag are written
                    // back once per chunk (ws_flush_kernel)
                    const double xn = fmax(c[k] + tw * u[k] * inv_s, 0.0);
                    st.ws_x[wb + (k << 5)] = xn;
                    if (xn > 0.0) {
                        red_add_f64(st.xsum + e0 + pos[k], xn);
                        fixed_colsum_add(mk, st, jc[k], xn);
                    }
                }
            }
            st.srow[i] = sr;
            my_sweeps += nsw;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_sweeps += __shfl_xor_sync(MQ_FULL, my_sweeps, o);
    if (lane == 0 && my_sweeps)
        atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)my_sweeps);
}

// Full solve of the listed rows (no working set, a failed certificate, more
// than MQ_WS_SLOTS working entries, or x_prev_out requested), a warp per row,
// the row (<= MQ_WS_MAX_ROW entries) in registers, then the working set rebuilt:
// slots in ascending entry order, theta / P over the screened entries, C.
#ifndef MQ_WSF_MINB
#define MQ_WSF_MINB 2  // resident 256-thread CTAs per SM of the full solve
#endif
__global__ void __launch_bounds__(256, MQ_WSF_MINB)
ws_full_kernel(const mq_market mk, const mq_state st, int it, double *__restrict__ x_prev_out) {
    constexpr int G = 32, RP = MQ_WS_MAX_ROW / 32;  // a warp per row, rows <= 256 entries
    const double tau = st.steps[0];
    const double cnow = drift_now(st);
    const int wl = threadIdx.x & 31, lane = wl, gsub = 0;
    const uint32_t gmask = MQ_FULL;
    const int count = *(volatile int32_t *)(st.blk_done + 3);
    int my_sweeps = 0, my_faults = 0;
    for (;;) {
        int rb = 0;
        if (wl == 0) rb = atomicAdd(st.blk_done + 4, 1);
        rb = __shfl_sync(MQ_FULL, rb, 0);
        if (rb >= count) break;  // warp-uniform
        const int r = rb + gsub;
        const bool has = r < count;
        const int64_t i = has ? st.ws_list[r] : 0;
        MQ_CHECK(count <= mk.n && i >= 0 && i < mk.n);
        int64_t a = 0;
        int len = 0;
        double w = 0.0, s0 = 0.0;
        int hold = -3;
        if (has) {
            a = __ldg(mk.row_ptr + i);
            len = (int)(__ldg(mk.row_ptr + i + 1) - a);
            w = __ldg(mk.w + i);
            s0 = st.srow[i];
            hold = __ldcg(st.ws_hdr + 4 * i);
            MQ_CHECK(len <= RP * G && hold >= -2 && hold <= MQ_WS_SLOTS);
        }
        double c[RP], u[RP], pv[RP], xv[RP];
        int jc[RP];
        uint32_t fb = 0;  // x > 0 flags as stored
#pragma unroll
        for (int e = 0; e < RP; ++e) {
            const int t = lane + e * G;
            const bool in = t < len;
            jc[e] = in ? __ldg(mk.col + a + t) : 0;
            u[e] = in ? __ldg(mk.u + a + t) : 0.0;
            if (in && __ldcg(st.xflag + a + t)) fb |= 1u << e;
        }
        uint32_t was = fb;  // entries whose x^k is nonzero
        if (hold >= 0) {
            // a row solved over its working set so far this chunk: x^k lives
            // in its slots (x and the flags are written back at chunk end);
            // every other entry of the row is zero
            was = 0;
#pragma unroll
            for (int e = 0; e < RP; ++e) xv[e] = 0.0;
            for (int k = 0; k < hold; ++k) {
                const int64_t at = ws_at(i, k);
                const int ps = __ldcg(st.ws_pos + at);
                if ((ps & (G - 1)) == lane) {
                    const double xk = __ldcg(st.ws_x + at);
#pragma unroll
                    for (int e = 0; e < RP; ++e)
                        if (e == ps / G) {
                            xv[e] = xk;
                            if (xk > 0.0) was |= 1u << e;
                        }
                }
            }
#pragma unroll
            for (int e = 0; e < RP; ++e) {
                const int t = lane + e * G;
                pv[e] = t < len ? __ldg(st.p + jc[e]) : 0.0;
            }
        } else {
#pragma unroll
            for (int e = 0; e < RP; ++e) {
                const int t = lane + e * G;
                pv[e] = t < len ? __ldg(st.p + jc[e]) : 0.0;
                xv[e] = ((fb >> e) & 1u) ? __ldcg(st.x + a + t) : 0.0;
            }
        }
        const double tw = tau * w;
#pragma unroll
        for (int e = 0; e < RP; ++e) {
            c[e] = xv[e] - tau * pv[e];
            const int t = lane + e * G;
            if (x_prev_out && t < len) x_prev_out[a + t] = xv[e];
        }
        int nsw = 0;
        bool ok = true;
        const double s = row_root_warm<G, RP>(c, u, tw, s0, has, gmask, &nsw, &ok);
        const double inv_s = 1.0 / s;
        double xn[RP];
#pragma unroll
        for (int e = 0; e < RP; ++e) {
            const int t = lane + e * G;
            xn[e] = t < len ? fmax(c[e] + tw * u[e] * inv_s, 0.0) : 0.0;
            if (t < len) {
                const bool nz = xn[e] > 0.0, fl = (fb >> e) & 1u;
                const int64_t g = a + t;
                if (nz != fl) st_flag(st.xflag + g, nz);
                if (nz || fl || ((was >> e) & 1u)) st.x[g] = xn[e];
                if (nz) {
                    red_add_f64(st.xsum + g, xn[e]);
                    fixed_colsum_add(mk, st, jc[e], xn[e]);
                }
            }
        }
        // a failed certificate widens the row's set, an overfull one narrows it
        int lvl = has ? ws_level(st, i) : 0;
        const int nl = hold >= 0 ? (lvl < 3 ? lvl + 1 : 3) : hold == -2 ? (lvl > 0 ? lvl - 1 : 0) : lvl;
        if (has && hold != -3 && nl != lvl && lane == 0 && st.ws_lvl) st.ws_lvl[i] = (uint8_t)nl;
        ws_build<G, RP>(st, i, lane, gsub, has && hold != -3, len, w, s, cnow, u, pv, xn, jc,
                        ws_gamma(nl));
        if (has && lane == 0) {
            st.srow[i] = s;
            my_sweeps += nsw;
            if (!ok) ++my_faults;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_sweeps += __shfl_xor_sync(MQ_FULL, my_sweeps, o);
        my_faults += __shfl_xor_sync(MQ_FULL, my_faults, o);
    }
    if (wl == 0 && my_sweeps)
        atomicAdd((unsigned long long *)(st.pass_out + it), (unsigned long long)my_sweeps);
    if (wl == 0 && my_faults) atomicAdd((unsigned long long *)st.faults, (unsigned long long)my_faults);
}

// ------------------------------------------------------------ column sums
// Deterministic fp64 column sums over the blocked schedule (residual checks,
// restarts: the reference's column_sums order): one thread per good walking
// blocks [b_lo, b_hi) in order (ascending rows), 4 gathers in flight.
__global__ void __launch_bounds__(256)
colsum_blocks_kernel(int64_t m, const int32_t *__restrict__ bptr, const int32_t *__restrict__ bperm,
                     int64_t b_lo, int64_t b_hi, const double *__restrict__ v,
                     double *__restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    double acc = 0.0;
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
}

// fixed-point column sums -> cs (and csbar), accumulators zeroed for the next
// iteration
__global__ void cs_from_fixed_kernel(int64_t m, unsigned long long *__restrict__ fix,
                                     double *__restrict__ cs, double *__restrict__ csbar,
                                     const int64_t *__restrict__ navg, int it, double inv_scale,
                                     double *__restrict__ drift) {
    const Avg av = avg_weights(navg, it);
    if (drift && blockIdx.x == 0 && threadIdx.x == 0) {
        // the primal kernels' C + dec, stored: the price-decrease bound so far
        drift[0] = __dadd_ru(drift[0], drift[1]);
        drift[1] = 0.0;
    }
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double c = (double)fix[j] * inv_scale;  // exact for sums < 2^53 units
        cs[j] = c;
        fix[j] = 0ull;
        if (csbar) csbar[j] = av.wold * csbar[j] + av.wnew * c;
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

// xbar = S / count: the running average of kernels.py:138-142 from the
// running sum, once per chunk
__global__ void avg_materialize_kernel(int64_t nnz, const double *__restrict__ xsum,
                                       double *__restrict__ xbar, const int64_t *__restrict__ navg) {
    const double count = (double)*navg;
    if (count <= 0.0) return;
    const double inv = 1.0 / count;  // one division, not one per entry
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x)
        xbar[e] = xsum[e] * inv;
}

// End of a chunk: x and its flags of every row with a working set, from the
// slots (inside a chunk the screened solve writes only the slots)
__global__ void ws_flush_kernel(int64_t n, const int64_t *__restrict__ row_ptr, mq_state st) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int h = st.ws_hdr[4 * i];
        if (h <= 0) continue;
        const int64_t e0 = row_ptr[i];
        for (int k = 0; k < h; ++k) {
            const int64_t at = ws_at(i, k);
            const int64_t g = e0 + st.ws_pos[at];
            MQ_CHECK(g < row_ptr[i + 1]);
            const double x = st.ws_x[at];
            const bool nz = x > 0.0;
            const uint8_t f = st.xflag[g];  // x > 0 as of the last write-back
            if (nz || f) {  // a zero that stayed zero needs no write
                st.x[g] = x;
                if (nz != (f != 0)) st.xflag[g] = nz;
            }
        }
    }
}

// ------------------------------------------------------------ launchers
// per-device caches: a process may solve on several GPUs (SolveConfig.device)
static int sm_count() {
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

// opt in to `bytes` of dynamic shared memory for `kern` once per device
template <typename F>
static int ensure_smem(F kern, int bytes, unsigned long long *done, const char *what) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (*done & bit) return 0;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return set_error(e, what);
    *done |= bit;
    return 0;
}

using PrimalLayout = TileLayout<MQ_ETILE, MQ_TILE_ROWS>;
constexpr int kPrimalSmem = MQ_STAGES * PrimalLayout::kStage + 6 * MQ_STAGES * 8 + MQ_STAGES * 4;

template <bool BUILD>
static int tile_launch(const mq_market *mk, const mq_state *st, int it, double *xprev,
                       cudaStream_t s) {
    static unsigned long long configured = 0;
    auto kern = primal_fused_kernel<MQ_G, MQ_NSW, MQ_ETILE, MQ_TILE_ROWS, MQ_STAGES, BUILD>;
    if (int rc = ensure_smem(kern, kPrimalSmem, &configured, "mq_primal_step: smem attribute"))
        return rc;
    // the dynamic tile counter lives in blk_done[0]
    kern<<<mk->prim_grid, (MQ_NSW + 1) * 32, kPrimalSmem, s>>>(*mk, *st, it, xprev, 0, mk->ntiles,
                                                               st->blk_done);
    return 0;
}

int primal_launch(const mq_market *mk, const mq_state *st, int it, double *xprev, cudaStream_t s) {
    int rc = 0;
    // every dynamic work counter (tiles, long rows, medium rows, full-solve
    // list and its claims, screened batches) restarts at 0
    cudaMemsetAsync(st->blk_done, 0, 8 * sizeof(int32_t), s);
    if (st->ws_hdr && !st->ws_rebuild) {  // screened solve, then the full-solve list
        static unsigned long long wconfigured = 0;
        if (int rc2 = ensure_smem(ws_kernel, kWsSmem, &wconfigured,
                                  "mq_primal_step: ws smem attribute"))
            return rc2;
        ws_kernel<<<sm_count(), (MQ_WS_NC + 1) * 32, kWsSmem, s>>>(*mk, *st, it,
                                                                   xprev != nullptr);
        ws_full_kernel<<<sm_count() * MQ_WSF_MINB, 256, 0, s>>>(*mk, *st, it, xprev);
    } else if (mk->ntiles > 0) {
        rc = (st->ws_hdr && st->ws_rebuild) ? tile_launch<true>(mk, st, it, xprev, s)
                                            : tile_launch<false>(mk, st, it, xprev, s);
        if (rc) return rc;
    }
    if (mk->nlong > 0) {
        using LS = LongSmem<MQ_LONG_THREADS, MQ_LONG_CAP>;
        auto lk = primal_long_kernel<MQ_LONG_THREADS, MQ_LONG_CAP>;
        static unsigned long long lconfigured = 0;
        if (int rc2 = ensure_smem(lk, LS::kBytes, &lconfigured,
                                  "mq_primal_step: long-row smem attribute"))
            return rc2;
        const int per_sm = MQ_LONG_PER_SM;
        const int grid = grid_for(mk->nlong, 1, sm_count() * per_sm);
        // with pools: the warp pass first, the CTA kernel on the rows it left
        const int listed = st->pl_hdr && st->pl_list && !xprev;
        if (listed)
            primal_long_ws_kernel<<<grid_for(mk->nlong, 8, sm_count() * 8), 256, 0, s>>>(*mk, *st, it);
        lk<<<grid, MQ_LONG_THREADS, LS::kBytes, s>>>(*mk, *st, it, xprev, listed);
    }
    // with working sets, medium rows up to MQ_WS_MAX_ROW entries are
    // screened / fully solved above; the leading (longest) nmed_long stay here
    const int64_t nmed = (st->ws_hdr && !st->ws_rebuild) ? mk->nmed_long : mk->nmed;
    if (nmed > 0) {
        const int grid = grid_for(nmed, 8, sm_count() * 8);
        primal_med_kernel<<<grid, 256, 0, s>>>(*mk, *st, it, xprev, nmed);
    }
    return check_launch("mq_primal_step");
}

// shared with the lifted PDHG step (lifted.cu)
int launch_dual(const mq_market *mk, double *p, double *pbar, double *cs, double *cs_prev,
                const double *steps, const int64_t *navg, int it, cudaStream_t s,
                double *drift) {
    dual_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(mk->m, p, pbar, cs, cs_prev,
                                                                     steps, navg, it, drift);
    return check_launch("mq_dual_step");
}
int launch_cs_from_fixed(const mq_market *mk, unsigned long long *fix, double *cs, double *csbar,
                         const int64_t *navg, int it, cudaStream_t s, double *drift) {
    cs_from_fixed_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, s>>>(
        mk->m, fix, cs, csbar, navg, it, 1.0 / mk->cs_scale, drift);
    return check_launch("mq_colsum_step");
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_dual_step(const mq_market *mk, const mq_state *st, int it, void *stream) {
    return launch_dual(mk, st->p, st->pbar, st->cs, st->cs_prev, st->steps, st->navg, it,
                       (cudaStream_t)stream, st->ws_hdr ? st->drift : nullptr);
}

int mq_primal_step(const mq_market *mk, const mq_state *st, int it, double *x_prev_out,
                   void *stream) {
    return primal_launch(mk, st, it, x_prev_out, (cudaStream_t)stream);
}

// every entry (tiles and long rows) went through the fixed-point atomics
int mq_colsum_step(const mq_market *mk, const mq_state *st, int it, int finalize, void *stream) {
    return launch_cs_from_fixed(mk, reinterpret_cast<unsigned long long *>(st->bucket), st->cs,
                                finalize ? st->csbar : nullptr, st->navg, it,
                                (cudaStream_t)stream, st->ws_hdr ? st->drift : nullptr);
}

int mq_colsum_finalize(const mq_market *mk, const mq_state *st, int it, void *stream) {
    colsum_finalize_kernel<<<grid_for(mk->m, 256, sm_count() * 8), 256, 0, (cudaStream_t)stream>>>(
        mk->m, st->cs, st->csbar, st->navg, it);
    return check_launch("mq_colsum_finalize");
}

int mq_chunk_end(const mq_state *st, int iters, void *stream) {
    chunk_end_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(st->navg, iters);
    return check_launch("mq_chunk_end");
}

int mq_ws_flush(const mq_market *mk, const mq_state *st, void *stream) {
    if (!mk || !st) return set_error(cudaErrorInvalidValue, "mq_ws_flush: null argument");
    if (st->ws_hdr)  // the screened rows' x and flags, from their slots
        ws_flush_kernel<<<grid_for(mk->n, 256, sm_count() * 16), 256, 0, (cudaStream_t)stream>>>(
            mk->n, mk->row_ptr, *st);
    return check_launch("mq_ws_flush");
}

int mq_avg_xbar(const mq_market *mk, const mq_state *st, void *stream) {
    if (!mk || !st) return set_error(cudaErrorInvalidValue, "mq_avg_xbar: null argument");
    avg_materialize_kernel<<<grid_for(mk->nnz, 256, sm_count() * 16), 256, 0,
                             (cudaStream_t)stream>>>(mk->nnz, st->xsum, st->xbar, st->navg);
    return check_launch("mq_avg_xbar");
}

int mq_avg_materialize(const mq_market *mk, const mq_state *st, void *stream) {
    if (int rc = mq_ws_flush(mk, st, stream)) return rc;
    return mq_avg_xbar(mk, st, stream);
}

int mq_fast_chunk(const mq_market *mk, const mq_state *st, int iters, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    for (int it = 0; it < iters; ++it) {
        if ((rc = mq_dual_step(mk, st, it, stream))) return rc;
        if ((rc = primal_launch(mk, st, it, nullptr, s))) return rc;
        if ((rc = mq_colsum_step(mk, st, it, 1, stream))) return rc;
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

int mq_tile_entries(void) { return MQ_ETILE; }
int mq_reg_row(void) { return MQ_REG_PER * MQ_G; }
int mq_colsum_mode(void) { return 5; }   // fixed-point sparse column sums
int mq_bucket_slots(void) { return 0; }  // no bucket mode in this build
int mq_x_sparse(void) { return 1; }
int mq_fixed_colsum(void) { return 1; }
int mq_ws_slots(void) { return MQ_WS_SLOTS; }
int mq_long_cap(void) { return MQ_LONG_CAP; }
int mq_med_cap(void) { return MQ_MED_CAP; }
int mq_market_bytes(void) { return (int)sizeof(mq_market); }
int mq_state_bytes(void) { return (int)sizeof(mq_state); }

int mq_colsum(const mq_market *mk, const double *v, double *out, void *stream) {
    const int grid = (int)((mk->m + 255) / 256);
    colsum_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(mk->m, mk->bptr, mk->bperm, 0,
                                                                 mk->nblk + 1, v, out);
    return check_launch("mq_colsum");
}

}  // extern "C"
