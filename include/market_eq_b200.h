/*
 * market_eq_b200 — C ABI of the B200-native PDHCG hot path.
 *
 * Drop-in boundary for the reference's fused iteration kernel
 * (/root/reference/pkg/src/market_eq/kernels.py:99-145, called from
 * driver._CompactRun.run_chunk, driver.py:134-145) plus the device-side
 * reductions the reference's solve loop runs between chunks (kkt.py:29-87,
 * driver.py:123-132, 156-162) and the Arrow-Debreu budget map
 * (exchange.py:75-93 -> sparse.py:147-153).
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless the parameter name ends in
 *    `_host`.  Buffers are owned by the caller (PyTorch in the Python
 *    package); the library allocates nothing that outlives a call.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    and graph-capturable, except mq_pdhcg_chunk, which mirrors the
 *    reference's synchronous return of (navg, faults).
 *  - Return value: 0 on success, < 0 on a CUDA error (mq_last_error() has the
 *    message), > 0 only from mq_pdhcg_chunk (= number of faulted rows, which
 *    the caller turns into SubproblemError exactly as driver.py:142-144).
 *  - No C++ exception crosses this boundary.
 *  - Index layout: row offsets int64 [n+1]; column indices int32 [nnz];
 *    transpose schedule tperm int32 [nnz] / tptr int64 [m+1] (the stable
 *    column grouping of sparse.py:130-145); values float64.
 */
#ifndef MARKET_EQ_B200_H
#define MARKET_EQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MQ_ABI_VERSION 12
#define MQ_TILE_ENTRIES 2560 /* entries staged per shared-memory tile (default build) */
#define MQ_LONG_ROW 1024      /* rows longer than this use the CTA-per-row path */
#define MQ_TILE_ROWS 256      /* rows per tile                                */
#define MQ_REG_ROW 128        /* tile rows longer than this (medium rows) are
                                 solved by the warp-per-row path          */
#ifndef MQ_WS_SLOTS
#define MQ_WS_SLOTS 10        /* working-set slots per row (screened solve)  */
#endif
#define MQ_WS_MAX_ROW 256     /* rows up to this length have working sets    */

/* Read-only market description (device pointers, borrowed).  Arrays marked
 * [pad] must have 16 readable bytes past their last element (TMA bulk copies
 * move 16-byte-aligned ranges). */
typedef struct mq_market {
    int64_t n, m, nnz;
    const int64_t *row_ptr;  /* [n+1] [pad]                                    */
    const int32_t *col;      /* [nnz] [pad] strictly increasing within a row   */
    const double *u;         /* [nnz] [pad] normalized utilities (row max 1),
                                instance.py:118-138                             */
    const double *u_orig;    /* [nnz] original utilities (residuals, kkt.py)    */
    const double *w;         /* [n] [pad] budgets                               */
    /* row tiles of the primal kernel: tile k = rows [tiles[4k], tiles[4k+1])
       = entries [tiles[4k+2], tiles[4k+3]), at most MQ_TILE_ENTRIES entries
       and MQ_TILE_ROWS rows, no row longer than MQ_LONG_ROW (32-byte aligned) */
    const int64_t *tiles;
    int64_t ntiles;
    const int32_t *long_rows; /* rows longer than MQ_LONG_ROW, longest first    */
    int64_t nlong;
    /* medium rows: tile rows longer than MQ_REG_ROW, longest first; the tile
       kernel skips them (their entries are still staged) and the warp-per-row
       kernel solves them, so no tile stage waits on one slow row             */
    const int32_t *med_rows;
    int64_t nmed;
    /* the leading med_rows longer than MQ_WS_MAX_ROW: with working sets on,
       the warp-per-row kernel solves only these (shorter rows have working
       sets); without, or in a rebuild step, all nmed                       */
    int64_t nmed_long;
    /* tile-blocked transpose schedule of the deterministic fp64 column sums
       (mq_colsum: residual checks, restarts): the tiles are grouped in blocks
       of tiles_per_block consecutive tiles; bperm lists, block by block and
       column by column, the entry positions of each block (ascending inside
       a column), bptr[b*m + j] where (block b, good j) starts; pseudo-block
       nblk holds the long rows' entries.                                     */
    const int32_t *bperm;    /* [nnz]                                           */
    const int32_t *bptr;     /* [(nblk+1)*m + 1]                                */
    int64_t nblk, tiles_per_block;
    int32_t prim_grid;       /* CTAs of the persistent primal kernel            */
    int64_t row_begin;       /* first global row of this shard (0 on 1 GPU)    */
    /* fixed-point column sums of the price step: x_e is
       added to its good's u64 accumulator as round(x_e * cs_scale) when
       0 < x_e < cs_xmax (larger values count as faults); cs_scale = 2^k with
       cs_xmax * cs_scale * (max entries of a good) <= 2^62                    */
    double cs_scale, cs_xmax;
} mq_market;

/* Mutable iterate of the fast (graph-captured) path.  cs / cs_prev / csbar are
 * the column sums of x^k, x^{k-1} and xbar: the price step of kernels.py:111-116
 * needs colsum(2x^k - x^{k-1}) = 2 cs - cs_prev, so x^{k-1} itself is never
 * stored. */
typedef struct mq_state {
    double *x;        /* [nnz] [pad] current allocation x^k (updated in place) */
    double *xbar;     /* [nnz] [pad] running average                           */
    double *p;        /* [m]   prices                                          */
    double *pbar;     /* [m]   running average of prices                       */
    double *cs;       /* [m]   colsum(x^k)                                     */
    double *cs_prev;  /* [m]   colsum(x^{k-1})                                 */
    double *csbar;    /* [m]   colsum(xbar)                                    */
    int32_t *blk_done;/* [8] the primal kernels' dynamic work counters (tiles,
                         long rows, medium rows, full-solve list length, its
                         claim counter, screened-solve batches), zeroed by
                         mq_primal_step                                      */
    const double *steps; /* [2] tau, sigma (device-resident: one graph serves
                            every step size)                                   */
    int64_t *navg;    /* [1]  inner iterations since the last restart          */
    int64_t *pass_out;/* [iters] per-iteration row-solver work counter         */
    int64_t *faults;  /* [1]  rows whose solver failed                         */
    double *bucket;   /* [m] u64 fixed-point column-sum accumulators (zero
                         between iterations)                                   */
    double *srow;     /* [n] [pad] per-buyer utility after the last prox: the
                         row solve's warm start (<= 0: none; any value is
                         correct, a close one saves sweeps)                    */
    /* sparse iterate: xflag[e] = (x[e] > 0) is staged
       instead of x (x is read only where flagged and stays exact); xsum =
       sum of x since the last restart, xbar = xsum / navg is written by
       mq_avg_materialize.  The host sets xflag = 1 and xsum = navg * xbar
       whenever it writes x, xbar or navg itself.                            */
    uint8_t *xflag;   /* [nnz] [pad]                                          */
    double *xsum;     /* [nnz]                                                */
    /* Working set of the screened row solve; ws_hdr == NULL
       selects the unscreened tile kernel.  For a zero entry x_ij = 0, the
       prox keeps it at zero iff p_j s_i >= w_i u_ij (s_i = the row's root),
       so a row is solved over its working set only — nonzero and "near"
       entries, at most MQ_WS_SLOTS, held in slots — and the result is the
       full row's when the certificate
           theta_i s (P_i - D) >= w_i P_i (1 + 1e-12)
       holds, theta_i = min p_j / u_ij and P_i = min p_j over the screened
       entries at the working set's last rebuild and D the accumulated price
       decrease since (drift); otherwise (and when h < 0) the row is solved in
       full and its working set rebuilt.  Rows are grouped in blocks of 32
       (block b = rows 32b..32b+31), the unit of the screened kernel's
       bulk copies.  The host writes h = -1 (keeping -3) and kmax = 0
       whenever it writes x or p itself.                                   */
    int32_t *ws_hdr;  /* [4 npad] per row: h = slots in use (>= 0), -1 none,
                         -2 more than MQ_WS_SLOTS (solved in full every
                         iteration), -3 not a tile row (medium / long
                         kernels); then theta, P, C at the rebuild as float
                         bit patterns, each rounded down                     */
    int32_t *ws_kmax; /* [npad / 32] upper bound of h over each block of 32
                         rows (the screened kernel copies slots 0..kmax-1) */
    /* slots, ascending entry order within a row; slot k of row i at
       ((i / 32) * MQ_WS_SLOTS + k) * 32 + i % 32 (a block's slots 0..k are
       one contiguous run); arrays of npad * MQ_WS_SLOTS, npad = n rounded
       up to 32                                                             */
    double *ws_u;     /* normalized utility of the slot's entry              */
    double *ws_x;     /* its current x (the slot is authoritative)           */
    int32_t *ws_col;  /* its good                                            */
    uint8_t *ws_pos;  /* its offset in the row (tile rows <= MQ_REG_ROW)     */
    int32_t *ws_list; /* [n] rows solved in full this iteration               */
    double *drift;    /* [2] C = accumulated bound on the largest price
                         decrease (rounded up), this iteration's decrease
                         (bit pattern, order-free max)                      */
    /* working sets of the long rows (> MQ_LONG_ROW entries, the CTA-per-row
       kernel; pl_hdr == NULL: none), one pool of MQ_LONG_CAP entries per row
       in mk.long_rows order: row r's working entries (ascending position) at
       r * MQ_LONG_CAP + k, k < h; the header and certificate as ws_hdr's    */
    int32_t *pl_hdr;  /* [4 nlong] h (-1 none, -2 more than MQ_LONG_CAP), theta,
                         P, C (float bits, rounded down)                     */
    double *pl_u;     /* [nlong MQ_LONG_CAP] normalized utility              */
    double *pl_x;     /* its x (a long row's canonical x and flags are also
                         written every iteration)                           */
    int32_t *pl_col;  /* its good                                            */
    int32_t *pl_pos;  /* its offset in the row                               */
    /* working sets of the medium rows longer than MQ_WS_MAX_ROW (the first
       mk.nmed_long of mk.med_rows, the warp-per-row kernel; pm_hdr == NULL:
       none), one pool of MQ_MED_CAP entries per row, laid out as pl_*      */
    int32_t *pm_hdr;  /* [4 nmed_long] h (-1 none, -2 more than MQ_MED_CAP),
                         theta, P, C                                        */
    double *pm_u;     /* [nmed_long MQ_MED_CAP] normalized utility           */
    double *pm_x;     /* its x (canonical x and flags also written)          */
    int32_t *pm_col;  /* its good                                            */
    int32_t *pm_pos;  /* its offset in the row                               */
    int32_t ws_rebuild; /* nonzero: this step runs the unscreened tile kernel
                           over every tile row and rebuilds all working sets
                           (after the host invalidated them; cheaper than
                           the per-row full solves when every row needs one) */
    int32_t xbar_lazy;  /* nonzero: xbar is stale (the host skipped
                           mq_avg_xbar after the last chunk);
                           mq_resid_rows_pair reads the average as
                           xsum / navg instead                               */
    uint8_t *ws_lvl;    /* [n] per row: the working-set width level (gamma =
                           1.001, 1.005, 1.02, 1.06 for 0..3; +1 after a
                           failed certificate, -1 after an overfull set or
                           a rebuild of all sets); NULL: level 2             */
    int32_t *pl_list;   /* [nlong] long rows left for the CTA-per-row kernel
                           after the warp-per-row screened pass (count in
                           blk_done[7]); used when pl_hdr is set             */
} mq_state;

/* Mutable iterate of the lifted PDHG path (algo="pdhg", kernels.py:146-197):
 * x (nnz), t and y (n), p (m), their running averages, and the row sums
 * ru = u.x^k, ru_prev = u.x^{k-1} (normalized utilities) that stand in for the
 * reference's x_prev in the y step. */
typedef struct mq_lstate {
    double *x, *xbar;                        /* [nnz]                          */
    double *t, *t_prev, *tbar, *y, *ybar;    /* [n]                            */
    double *ru, *ru_prev;                    /* [n]                            */
    double *p, *pbar, *cs, *cs_prev, *csbar; /* [m]                            */
    unsigned long long *fix;                 /* [m] fixed-point column sums,
                                                zero between iterations        */
    const double *steps;                     /* [2] tau, sigma                 */
    int64_t *navg;                           /* [1]                            */
    int64_t *faults;                         /* [1] x beyond cs_xmax           */
} mq_lstate;

/* ---- faithful drop-in ------------------------------------------------------
 * Replaces kernels.pdhcg_chunk (kernels.py:99-145) argument for argument:
 * same in-place semantics for x, x_prev, p, xbar, pbar, c_buf and
 * pass_out[iters]; the literal k-section row search of _row_root
 * (kernels.py:33-96) with `sections` and `subtol`; fixed-order serial sums.
 * Bit-identical to the reference on the same inputs.  Synchronous: returns the
 * fault count (>= 0) and writes the new navg to *navg_out_host. */
int mq_pdhcg_chunk(int64_t n, int64_t m, const int64_t *indptr, const int32_t *colind,
                   const double *uval, const int32_t *tperm, const int64_t *tindptr,
                   const double *w, double *x, double *x_prev, double *p, double *xbar,
                   double *pbar, int64_t navg, double tau, double sigma, int sections,
                   double subtol, int iters, double *c_buf, int64_t *pass_out,
                   int64_t *navg_out_host, void *stream);

/* ---- fast path: one PDHCG iteration as three graph-capturable launches ----
 * it = index of the iteration inside the chunk (count = *navg + it + 1). */

/* Price step + price average (kernels.py:111-116, 143-144):
 * p += sigma (2 cs - cs_prev - 1); pbar <- avg; cs_prev <- cs. */
int mq_dual_step(const mq_market *mk, const mq_state *st, int it, void *stream);

/* Exact per-buyer proximal step fused with the running average and the
 * column sums (kernels.py:117-142 then the next iteration's 111-116): for
 * every row, the unique root s of s = sum_j u_j max(0, c_j + tau w u_j / s),
 * c = x - tau p[col], by the monotone active-set iteration (closed-form root
 * per active set, warm-started from srow), then x <- max(0, c + tau w u / s)
 * with its flag, the running sum xsum and the fixed-point column-sum atomics
 * of the nonzero entries.  x_prev_out (may be NULL) receives the pre-step x
 * (the reference's x_prev copy).  pass_out[it] += number of sweeps. */
int mq_primal_step(const mq_market *mk, const mq_state *st, int it, double *x_prev_out,
                   void *stream);

/* cs = colsum(x) over this shard from the fixed-point accumulators (which it
 * zeroes).  With finalize != 0 also csbar <- avg(csbar, cs); multi-GPU callers
 * all-reduce the accumulators (int64) first and then call it with
 * finalize != 0; mq_colsum_finalize updates csbar alone. */
int mq_colsum_step(const mq_market *mk, const mq_state *st, int it, int finalize,
                   void *stream);
int mq_colsum_finalize(const mq_market *mk, const mq_state *st, int it, void *stream);

/* navg += iters (end of a captured chunk). */
int mq_chunk_end(const mq_state *st, int iters, void *stream);

/* Whole chunk on one GPU: `iters` x (dual, primal, colsum) + chunk_end +
 * mq_avg_materialize. */
int mq_fast_chunk(const mq_market *mk, const mq_state *st, int iters, void *stream);

/* Plain column sums out[j] = sum_{col j} v over this shard, one thread per
 * good walking the blocked schedule (ascending rows; deterministic). */
int mq_colsum(const mq_market *mk, const double *v, double *out, void *stream);

/* ---- residuals (kkt.py:29-87 specialised to the compact state) -----------
 * Row pass over this shard: t_i = u_orig_i . x_i, y_i = w_i / t_i, column
 * maxima colbest_j = max_i u_orig_ij y_i (order-free max, deterministic),
 * and the entry-wise gap maxima.  `use_norm` selects the normalized
 * utilities instead (driver.py:123-132 omega_0 norms).
 * row_out[8] (device): [0] max y, [1] gap numerator max x (p-uy)_+,
 * [2] max |x|, [3] max (p-uy)_+, [4] first row with t <= 0 (as double, or -1),
 * [5] sum_i w_i log t_i (fixed order), [6] rows with t <= 0, [7] unused.
 * t_out / y_out (may be NULL) receive t and y per local row.
 * colbest must be zero-initialised by the caller (values are positive).
 * work: 2m doubles of workspace (p and the running column maxima interleaved,
 * one random access per entry), or NULL for a stream-ordered temporary. */
int mq_resid_rows(const mq_market *mk, const double *x, const double *p, int use_norm,
                  double *colbest, double *work, double *t_out, double *y_out, double *row_out,
                  double *scratch, void *stream);
/* Both row passes of a check in one sweep (the fast path's state): the
 * last iterate (st->x with st->xflag, st->p) and the average (st->xbar,
 * st->pbar), original utilities; each side exactly as mq_resid_rows with
 * use_norm = 0 (bitwise the two separate calls).  work: 4m doubles. */
int mq_resid_rows_pair(const mq_market *mk, const mq_state *st, double *colbest_last,
                       double *colbest_avg, double *work, double *row_out_last,
                       double *row_out_avg, double *scratch_last, double *scratch_avg,
                       void *stream);
/* Column pass (replicated data): col_out[6] (device):
 * [0] max |cs - 1|, [1] max |cs|, [2] max (colbest - p)_+, [3] max (p - colbest)
 * (initial 0), [4] sum (cs - 1)^2, [5] sum min(p - colbest, 0)^2. */
int mq_resid_cols(int64_t m, const double *cs, const double *p, const double *colbest,
                  double *col_out, double *scratch, void *stream);

/* Restart moves (driver.py:156-162): out[4] (device):
 * [0] sum (xbar-x0)^2 over this shard, [1] sum (pbar-p0)^2,
 * [2] sum_j (csbar-cs0)_j (pbar-p0)_j, [3] unused. */
int mq_restart_moves(const mq_market *mk, const double *xbar, const double *x0,
                     const double *pbar, const double *p0, const double *csbar,
                     const double *cs0, double *out, double *scratch, void *stream);

/* ---- lifted PDHG (algo="pdhg") ------------------------------------------
 * One iteration (kernels.py:158-196): price step, per-buyer y/t update and the
 * entry-wise x update with the averages, fixed-point column sums of x. */
int mq_pdhg_step(const mq_market *mk, const mq_lstate *ls, int it, void *stream);
/* N ranks: mq_pdhg_step without the column-sum conversion; the host
 * all-reduces ls->fix (int64) and then calls mq_pdhg_finish_colsum. */
int mq_pdhg_colsum_only(const mq_market *mk, const mq_lstate *ls, int it, void *stream);
int mq_pdhg_finish_colsum(const mq_market *mk, const mq_lstate *ls, int it, void *stream);
int mq_pdhg_chunk_end(const mq_lstate *ls, int iters, void *stream);
/* out_i = u_i . x_i (use_norm: normalized utilities, else original). */
int mq_row_dot(const mq_market *mk, const double *x, int use_norm, double *out, void *stream);
/* residuals_lifted (kkt.py:29-76) row/entry part for (x, t*s, p, y/s), s =
 * scales (use_norm = 0) or 1 (normalized instance, use_norm = 1);
 * colbest[m] <- max_i u_ij y_i (signed, order-free); row_out[10]: [0] max
 * |t - u.x|, [1] max |w/t|, [2] max |y|, [3] max |w/t - y|, [4] max
 * x (p - uy)_+, [5] max |x|, [6] max (p - uy)_+, [7] rows with t <= 0,
 * [8] sum (t - u.x)^2, [9] sum (w/t - y)^2 (fixed order). */
int mq_pdhg_resid_rows(const mq_market *mk, const double *scales, const double *x,
                       const double *t, const double *y, const double *p, int use_norm,
                       double *colbest, double *row_out, double *scratch, void *stream);
/* restart moves, row part (driver.py:242-252): out[3] = sum dt^2, sum dy^2,
 * sum (dt - u.dx) dy over this shard. */
int mq_pdhg_moves(const mq_market *mk, const double *xbar, const double *x0, const double *tbar,
                  const double *t0, const double *ybar, const double *y0, double *out,
                  double *scratch, void *stream);
/* lifted operator power step (pdhg.py:157-161) given out_p = colsum(vx):
 * out_y = vt - u.vx, wx = out_p[col] - u out_y[row], sums[2] = sum wx^2,
 * sum out_y^2 (fixed order). */
int mq_pdhg_opnorm_step(const mq_market *mk, const double *vx, const double *vt,
                        const double *out_p, double *out_y, double *wx, double *sums,
                        double *scratch, void *stream);

/* ---- theory diagnostics (kkt.py:88-168) ---------------------------------
 * Scaled KKT residual, row/entry parts on the original utilities: out[4] =
 * sum (t y - w)^2, sum (x - [x - slack/xi]_+)^2, sum min(slack, 0)^2,
 * sum (t - u.x)^2 with slack = p_j - u_ij y_i (fixed order). */
int mq_scaled_kkt_rows(const mq_market *mk, const double *x, const double *t, const double *p,
                       const double *y, double xi, double *out, double *scratch, void *stream);
/* Smoothed gap, allocation part: out[0] = sum_i -w_i log(u_i.xh_i) + p.xh_i +
 * xi/2 |xh_i - xc_i|^2 with xh_i the exact row prox of (xc, p) at step 1/xi
 * (cbuf: nnz scratch); rows whose iteration did not settle add to *faults. */
int mq_smoothed_gap_rows(const mq_market *mk, const double *xc, const double *p, double xi,
                         double *cbuf, double *out, double *scratch, int64_t *faults,
                         void *stream);

/* Sparse matrix-vector product out = E p for a CSR matrix (Arrow-Debreu
 * budget map, exchange.py:89 -> sparse.py:147-153); fixed-order row sums. */
int mq_spmv(int64_t n_rows, const int64_t *row_ptr, const int32_t *col,
            const double *val, const double *v, double *out, void *stream);

/* Row normalization (instance.py:118-138): scales_i = max_j u_ij,
 * u_out = u / scales_i (IEEE division, bit-identical to the reference). */
int mq_normalize_rows(int64_t n, const int64_t *row_ptr, const double *u, double *u_out,
                      double *scales, void *stream);

/* ---- device instance generator (BASELINE configs 3-5) ----------------------
 * Rows [row0, row0+nrows) of an n x m market: Bernoulli(q_i) support per row
 * drawn by geometric skipping (q_mode 0: q_i = q; q_mode 1: q_i = d_i/m with a
 * truncated power-law degree d_i = dmin U^(-1/(alpha-1))), an empty draw
 * repaired with one uniform column, values and budgets U(0,1].  One Philox
 * subsequence per row: shards generate independently and identically.
 * Pass 1 writes per-row degrees; the caller scans them into row_ptr (local,
 * starting at 0); pass 2 fills columns (ascending), values and budgets (w may
 * be NULL). */
int mq_gen_degrees(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                   double dmin, unsigned long long seed, int64_t *deg, void *stream);
int mq_gen_fill(int64_t row0, int64_t nrows, int64_t m, int q_mode, double q, double alpha,
                double dmin, unsigned long long seed, const int64_t *row_ptr, int32_t *col,
                double *val, double *w, void *stream);

/* Entries per primal tile this build was compiled for (tiles must not exceed
 * it; MQ_TILE_ENTRIES by default). */
int mq_tile_entries(void);

/* Longest tile row the tile kernel solves itself (MQ_REG_ROW); longer tile
 * rows go in mq_market.med_rows. */
int mq_reg_row(void);

/* How this build computes the price step's column sums: 5 = fixed-point
 * atomics on the nonzero entries (the only mode of this build; the earlier
 * gathered / scattered / bucketed modes are described in DESIGN.md §11). */
int mq_colsum_mode(void);

/* Size in doubles of the `scratch` buffer the reduction calls need. */
int64_t mq_scratch_doubles(void);

const char *mq_last_error(void);
int mq_abi_version(void);
/* 1 if the build sums columns in fixed point (state.bucket = m u64) */
int mq_fixed_colsum(void);
/* working-set slots per row of this build (MQ_WS_SLOTS) */
int mq_ws_slots(void);
/* long-row working-set pool entries per row of this build (MQ_LONG_CAP) */
int mq_long_cap(void);
/* MQ_MED_CAP: entries of a medium row's working-set pool (mq_state.pm_*) */
int mq_med_cap(void);
/* sizeof(mq_market), sizeof(mq_state) of this build (binding layout checks) */
int mq_market_bytes(void);
int mq_state_bytes(void);
/* 1 if the build keeps the sparse iterate (xflag / xsum) */
int mq_x_sparse(void);
/* sparse iterate, after mq_chunk_end: the screened rows' x and flags from
 * their working-set slots (mq_ws_flush), then xbar = xsum / navg
 * (mq_avg_xbar); mq_avg_materialize runs both */
int mq_ws_flush(const mq_market *mk, const mq_state *st, void *stream);
int mq_avg_xbar(const mq_market *mk, const mq_state *st, void *stream);
int mq_avg_materialize(const mq_market *mk, const mq_state *st, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MARKET_EQ_B200_H */
