/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the Accel-GCN hot path
 * (arXiv 2308.11825).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path in paper_2308_11825_b200/.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.  Readings of ambiguous passages are
 * the Q-numbers of SURVEY.md section 8(c3), restated in DESIGN.md "Readings".
 *
 *   orc_spmm / orc_spmm_check   result oracle, the plain definition of Y = A.X in fp64
 *                               ("feature aggregation ... SpMM between A' and Y^l")
 *   orc_degree_sort             stable counting sort of rows by degree (P:295 steps 1-2)
 *   orc_sorted_csr              row-pointer / column update in the new order (P:295 step 3)
 *   orc_patterns                Algorithm 1 "Get partition patterns", step by step
 *   orc_block_partition         Algorithm 2 "Block-level partitioning"
 *   orc_warp_partition          warp-level partition metadata of Fig. 3(b)
 *   orc_shard_bounds            nnz-balanced row shards (BASELINE.json north_star; reading Q32)
 *
 * Pins (tests/test_oracle*.py): Fig. 3 worked example, closed forms, dense brute force,
 * invariants (identity, all-ones X, row permutation, linearity, integer exactness).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---------------------------------------------------------------- threading (rows only) */
typedef void (*orc_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { orc_fn fn; void* ctx; int64_t lo, hi; } orc_job;
static void* orc_job_run(void* p) { orc_job* j = (orc_job*)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }
/* Rows are split into contiguous ranges; each row is summed by exactly one thread in
   index order, so results are bitwise independent of the thread count. */
static void orc_parallel_rows(int64_t n, int nt, orc_fn fn, void* ctx) {
    if (nt <= 0) { long c = sysconf(_SC_NPROCESSORS_ONLN); nt = c > 0 ? (int)c : 1; }
    if (nt > 256) nt = 256;
    if (n < 1024 || nt == 1) { fn(ctx, 0, n); return; }
    pthread_t th[256]; orc_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].lo = n * t / nt; jobs[t].hi = n * (t + 1) / nt;
        pthread_create(&th[t], NULL, orc_job_run, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- result oracle */
/*
 * y[i][k] = sum_{p=rowptr[i]}^{rowptr[i+1]-1} vals[p] * X[colidx[p]][k]   (fp64)
 * s[i][k] = sum_p |vals[p] * X[colidx[p]][k]|                            (fp64)
 * rowptr may start at a nonzero base (row shard); colidx/vals are indexed by rowptr values.
 * X is n_cols x F row-major fp32 (ld = F).  y, s: n x F fp64 (s may be NULL).
 */
typedef struct {
    const int32_t* rowptr; const int32_t* colidx; const float* vals; const float* X;
    int64_t F; double* y; double* s;
} spmm_ctx;
static void spmm_rows(void* c, int64_t lo, int64_t hi) {
    spmm_ctx* u = (spmm_ctx*)c;
    for (int64_t i = lo; i < hi; ++i) {
        double* yi = u->y + i * u->F;
        double* si = u->s ? u->s + i * u->F : NULL;
        for (int64_t k = 0; k < u->F; ++k) { yi[k] = 0.0; if (si) si[k] = 0.0; }
        for (int64_t p = u->rowptr[i]; p < u->rowptr[i + 1]; ++p) {
            double a = (double)u->vals[p];
            const float* xj = u->X + (int64_t)u->colidx[p] * u->F;
            for (int64_t k = 0; k < u->F; ++k) {
                double t = a * (double)xj[k];
                yi[k] += t;
                if (si) si[k] += fabs(t);
            }
        }
    }
}
void orc_spmm(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* vals,
              const float* X, int64_t F, double* y, double* s, int nthreads) {
    spmm_ctx c = {rowptr, colidx, vals, X, F, y, s};
    orc_parallel_rows(n, nthreads, spmm_rows, &c);
}

/*
 * Streaming parity check (no n x F fp64 arrays; used at full BASELINE sizes).
 * For every row i in rows[0..nrows) (or every row 0..n-1 if rows == NULL) and k < F:
 *   r = |(double)Y[i][k] - y_ref[i][k]| / (rel * s[i][k] + abs_tol)
 * Returns max r in *max_ratio (NaN/Inf in Y -> +inf), worst (row, col) in worst[0..1],
 * and the number of failing elements (r > 1) as the function result.
 * Tolerance |y - y_ref| <= 1e-5 * sum|a x| + 1e-7 is BASELINE.json north_star's.
 */
typedef struct {
    const int32_t* rowptr; const int32_t* colidx; const float* vals; const float* X;
    int64_t F; const float* Y; const int64_t* rows; double rel, abs_tol;
    double max_r; int64_t wi, wk, nfail; pthread_mutex_t* mu;
} chk_ctx;
static void chk_rows(void* c, int64_t lo, int64_t hi) {
    chk_ctx* u = (chk_ctx*)c;
    double* y = (double*)malloc(sizeof(double) * (size_t)(u->F > 0 ? u->F : 1));
    double* s = (double*)malloc(sizeof(double) * (size_t)(u->F > 0 ? u->F : 1));
    double mr = 0.0; int64_t wi = -1, wk = -1, nf = 0;
    for (int64_t t = lo; t < hi; ++t) {
        int64_t i = u->rows ? u->rows[t] : t;
        for (int64_t k = 0; k < u->F; ++k) { y[k] = 0.0; s[k] = 0.0; }
        for (int64_t p = u->rowptr[i]; p < u->rowptr[i + 1]; ++p) {
            double a = (double)u->vals[p];
            const float* xj = u->X + (int64_t)u->colidx[p] * u->F;
            for (int64_t k = 0; k < u->F; ++k) { double v = a * (double)xj[k]; y[k] += v; s[k] += fabs(v); }
        }
        const float* yi = u->Y + (u->rows ? t : i) * u->F;
        for (int64_t k = 0; k < u->F; ++k) {
            double g = (double)yi[k];
            double r = (isfinite(g)) ? fabs(g - y[k]) / (u->rel * s[k] + u->abs_tol) : INFINITY;
            if (r > 1.0) nf++;
            if (wi < 0 || r > mr) { mr = r; wi = i; wk = k; }
        }
    }
    pthread_mutex_lock(u->mu);
    if (wi >= 0 && (u->wi < 0 || mr > u->max_r)) { u->max_r = mr; u->wi = wi; u->wk = wk; }
    u->nfail += nf;
    pthread_mutex_unlock(u->mu);
    free(y); free(s);
}
/* Y layout: if rows == NULL, Y is the full n x F output; else Y holds the nrows sampled
   rows contiguously (row t of Y = output row rows[t]). */
int64_t orc_spmm_check(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* vals,
                       const float* X, int64_t F, const float* Y, const int64_t* rows, int64_t nrows,
                       double rel, double abs_tol, double* max_ratio, int64_t* worst, int nthreads) {
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    chk_ctx c = {rowptr, colidx, vals, X, F, Y, rows, rel, abs_tol, 0.0, -1, -1, 0, &mu};
    orc_parallel_rows(rows ? nrows : n, nthreads, chk_rows, &c);
    *max_ratio = c.max_r; worst[0] = c.wi; worst[1] = c.wk;
    return c.nfail;
}

/* ---------------------------------------------------------------- degree sorting */
/*
 * P:295 "(1) computing each row's degree using the row pointer array ... (2) applying a
 * stable sorting algorithm to sort rows based on the degrees ... employing count sort".
 * Ascending order (Q1), ties keep the original row order (Q2), degree-0 rows first (Q16).
 * perm[k] = original row at sorted position k (sorted_to_orig).
 * Returns max degree, or -1 on a malformed rowptr (decreasing).
 */
int64_t orc_degree_sort(int64_t n, const int32_t* rowptr, int32_t* perm) {
    int64_t maxd = 0;
    for (int64_t i = 0; i < n; ++i) {                   /* (1) deg[i] = rowptr[i+1]-rowptr[i] */
        int64_t d = (int64_t)rowptr[i + 1] - rowptr[i];
        if (d < 0) return -1;
        if (d > maxd) maxd = d;
    }
    int64_t* cnt = (int64_t*)calloc((size_t)(maxd + 1), sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[rowptr[i + 1] - rowptr[i]]++;   /* histogram */
    int64_t run = 0;                                    /* exclusive scan -> bucket starts */
    for (int64_t d = 0; d <= maxd; ++d) { int64_t c = cnt[d]; cnt[d] = run; run += c; }
    for (int64_t i = 0; i < n; ++i) {                   /* (2) stable scatter, rows in order */
        int64_t d = rowptr[i + 1] - rowptr[i];
        perm[cnt[d]++] = (int32_t)i;
    }
    free(cnt);
    return maxd;
}

/*
 * P:295 "(3) updating the row pointer array to reflect the new row order".
 * sorted_rowptr[k] = sum of degrees of sorted rows < k (starts at 0);
 * sorted_colidx[sorted_rowptr[k] + j] = colidx[rowptr[perm[k]] + j] (columns NOT relabelled, Q3);
 * row_src_off[k] = rowptr[perm[k]] - rowptr[0]  (where the caller's vals of that row start).
 */
void orc_sorted_csr(int64_t n, const int32_t* rowptr, const int32_t* colidx, const int32_t* perm,
                    int32_t* sorted_rowptr, int32_t* sorted_colidx, int32_t* row_src_off) {
    sorted_rowptr[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
        int32_t r = perm[k];
        int32_t d = rowptr[r + 1] - rowptr[r];
        sorted_rowptr[k + 1] = sorted_rowptr[k] + d;
        row_src_off[k] = rowptr[r] - rowptr[0];
        for (int32_t j = 0; j < d; ++j) sorted_colidx[sorted_rowptr[k] + j] = colidx[rowptr[r] + j];
    }
}

/* ---------------------------------------------------------------- Algorithm 1 */
/*
 * Literal transcription of Algorithm 1 "Get partition patterns":
 *   deg_bound <- max_block_warps * max_warp_nzs;             (line 1)
 *   factors   <- all factors of max_block_warps (ascending);  (line 2, Q6)
 *   i <- 0; deg <- 1;                                         (line 3)
 *   while deg <= deg_bound:        (Q4: inclusive; Fig. 3 BP-2 uses deg = deg_bound = 4)
 *     if factors[i] * max_warp_nzs >= deg:                    (Q5: warp_max_nz == max_warp_nzs)
 *        block_rows <- max_block_warps / factors[i]; warp_nzs <- ceil(deg / factors[i]); deg++
 *     else i++                                                (index never reset, Q6)
 * Outputs indexed by degree: block_rows[deg], warp_nzs[deg] for deg in 1..deg_bound
 * (index 0 unused, set to 0).  Arrays must hold deg_bound + 1 entries.  Returns deg_bound.
 */
int64_t orc_patterns(int32_t max_block_warps, int32_t max_warp_nzs, int32_t* block_rows,
                     int32_t* warp_nzs) {
    int64_t deg_bound = (int64_t)max_block_warps * max_warp_nzs;
    int32_t factors[4096]; int nf = 0;
    for (int32_t f = 1; f <= max_block_warps && nf < 4096; ++f)
        if (max_block_warps % f == 0) factors[nf++] = f;
    int i = 0; int64_t deg = 1;
    block_rows[0] = 0; warp_nzs[0] = 0;
    while (deg <= deg_bound) {
        if ((int64_t)factors[i] * max_warp_nzs >= deg) {
            block_rows[deg] = max_block_warps / factors[i];
            warp_nzs[deg] = (int32_t)((deg + factors[i] - 1) / factors[i]);
            deg++;
        } else {
            i++;
        }
    }
    return deg_bound;
}

/* ---------------------------------------------------------------- Algorithm 2 */
/*
 * Algorithm 2 "Block-level partitioning" over the degree-sorted rows, with running cursors
 * row (sorted row position) and loc (offset in the degree-sorted nnz array) (Q9, Q12, Q13).
 * Emits one 128-bit descriptor per block, field order (deg, loc, row, info) as in the
 * worked example P:421 (Q10):
 *   deg <= deg_bound: for each degree present, full blocks of pattern[deg].block_rows rows
 *       info = warp_nzs << 16 | block_rows   (Q11: high = warp_nzs, low = rows)
 *     then the residual block info = warp_nzs << 16 | rows_remaining, skipped if 0 (Q8)
 *   deg >  deg_bound: per row (Q7) in sorted order, chunks of deg_bound nnz, info = deg_bound,
 *     then the residual chunk info = deg_remaining, skipped if 0 (Q8, Q14)
 * Degree-0 rows produce nothing (Q16).  sorted_deg[k] = degree of sorted row k (must be
 * non-decreasing).  desc: 4 * max_desc uint32 (NULL to count only).
 * Returns the descriptor count, -1 if the input is not degree-sorted, -2 on 16-bit field
 * overflow (block_rows or warp_nzs >= 2^16), -3 if max_desc is too small.
 */
int64_t orc_block_partition(int64_t n, const int32_t* sorted_deg, int32_t max_block_warps,
                            int32_t max_warp_nzs, uint32_t* desc, int64_t max_desc) {
    for (int64_t k = 1; k < n; ++k) if (sorted_deg[k] < sorted_deg[k - 1]) return -1;
    int64_t deg_bound = (int64_t)max_block_warps * max_warp_nzs;
    int32_t* br = (int32_t*)malloc(sizeof(int32_t) * (size_t)(deg_bound + 1));
    int32_t* wn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(deg_bound + 1));
    orc_patterns(max_block_warps, max_warp_nzs, br, wn);
    int64_t nd = 0, row = 0, loc = 0, k = 0;
#define EMIT(D, L, R, I)                                                        \
    do {                                                                        \
        if (desc) {                                                             \
            if (nd >= max_desc) { free(br); free(wn); return -3; }              \
            desc[4 * nd + 0] = (uint32_t)(D); desc[4 * nd + 1] = (uint32_t)(L); \
            desc[4 * nd + 2] = (uint32_t)(R); desc[4 * nd + 3] = (uint32_t)(I); \
        }                                                                       \
        nd++;                                                                   \
    } while (0)
    while (k < n && sorted_deg[k] == 0) { k++; row++; }   /* degree-0 rows: no descriptor */
    while (k < n) {                                        /* "for each deg" */
        int64_t deg = sorted_deg[k];
        if (deg <= deg_bound) {
            int64_t rows_remaining = 0;                    /* total number of rows of deg */
            while (k + rows_remaining < n && sorted_deg[k + rows_remaining] == deg) rows_remaining++;
            k += rows_remaining;
            int64_t brd = br[deg], wnd = wn[deg];
            if (brd >= 65536 || wnd >= 65536) { free(br); free(wn); return -2; }
            while (rows_remaining >= brd) {
                EMIT(deg, loc, row, (wnd << 16) | brd);
                row += brd; loc += brd * deg;
                rows_remaining -= brd;
            }
            if (rows_remaining > 0) {
                EMIT(deg, loc, row, (wnd << 16) | rows_remaining);
                row += rows_remaining; loc += rows_remaining * deg;
            }
        } else {                                           /* one oversized row */
            int64_t deg_remaining = deg;
            while (deg_remaining >= deg_bound) {
                EMIT(deg, loc, row, deg_bound);
                loc += deg_bound; deg_remaining -= deg_bound;
            }
            if (deg_remaining > 0) {
                EMIT(deg, loc, row, deg_remaining);
                loc += deg_remaining;
            }
            row += 1; k += 1;
        }
    }
#undef EMIT
    free(br); free(wn);
    return nd;
}

/* ---------------------------------------------------------------- warp-level partition */
/*
 * Fig. 3(b) / P:417: each warp manages at most max_warp_nzs nonzeros of one row; metadata
 * {row, col, len} (col = offset inside the row) padded to 128 bits with a zero word.
 * Rows in ORIGINAL order, no sort (Q19).  tasks: 4 * max_tasks uint32 (NULL to count).
 * Returns the task count, or -3 if max_tasks is too small.
 */
int64_t orc_warp_partition(int64_t n, const int32_t* rowptr, int32_t max_warp_nzs, uint32_t* tasks,
                           int64_t max_tasks) {
    int64_t nt = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t d = (int64_t)rowptr[i + 1] - rowptr[i];
        for (int64_t c = 0; c < d; c += max_warp_nzs) {
            int64_t len = d - c < max_warp_nzs ? d - c : max_warp_nzs;
            if (tasks) {
                if (nt >= max_tasks) return -3;
                tasks[4 * nt + 0] = (uint32_t)i; tasks[4 * nt + 1] = (uint32_t)c;
                tasks[4 * nt + 2] = (uint32_t)len; tasks[4 * nt + 3] = 0u;
            }
            nt++;
        }
    }
    return nt;
}

/* ---------------------------------------------------------------- row shards (Q32) */
/*
 * nnz-balanced contiguous row shards: b_0 = 0, b_P = n,
 * b_p = first row r with rowptr[r] - rowptr[0] >= floor(p * nnz / P)   (linear scan).
 */
void orc_shard_bounds(int64_t n, const int32_t* rowptr, int32_t nranks, int64_t* bounds) {
    int64_t nnz = (int64_t)rowptr[n] - rowptr[0];
    bounds[0] = 0;
    for (int32_t p = 1; p < nranks; ++p) {
        int64_t target = ((int64_t)p * nnz) / nranks, r = 0;
        while (r < n && (int64_t)rowptr[r] - rowptr[0] < target) r++;
        bounds[p] = r;
    }
    bounds[nranks] = n;
}
