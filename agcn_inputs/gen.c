/*
 * agcn_inputs/gen.c -- seeded synthetic INPUT generators (test + bench infrastructure).
 *
 * This module only manufactures inputs: CSR graphs shaped like the paper's benchmark
 * graphs (Table I) and dense / value arrays.  It contains none of the
 * method's arithmetic (no degree sort, no partitioning, no SpMM).  Both the CPU oracle
 * (oracle/) and the CUDA path (paper_2308_11825_b200/) consume its output; neither side
 * is imported here.  Recipes are stated in DESIGN.md section "Input recipe".
 *
 * Every random number is counter based (splitmix64 of (seed, stream, index)), so output is
 * bit-identical for any thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
/* counter-based generator: independent stream per (seed, stream), index = counter */
static inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t idx) {
    return splitmix64(splitmix64(seed * 0x632BE59BD9B4E019ull + stream) ^ (idx * 0xD1342543DE82EF95ull));
}
static inline double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

static int default_threads(int nt) {
    if (nt > 0) return nt;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } job_t;
static void* job_run(void* p) { job_t* j = (job_t*)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }
static void parallel_for(int64_t n, int nt, range_fn fn, void* ctx) {
    nt = default_threads(nt);
    if (nt > 64) nt = 64;
    if (n < 4096 || nt == 1) { fn(ctx, 0, n); return; }
    pthread_t th[64]; job_t jobs[64];
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = n * t / nt; jobs[t].hi = n * (t + 1) / nt;
        pthread_create(&th[t], NULL, job_run, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* ---------------------------------------------------------------- dense arrays */
typedef struct { uint64_t seed; float lo, hi; float* out; } unif_ctx;
static void unif_body(void* c, int64_t lo, int64_t hi) {
    unif_ctx* u = (unif_ctx*)c;
    for (int64_t i = lo; i < hi; ++i) {
        /* 24-bit uniform in [0,1): exactly representable in fp32 */
        float f = (float)(rng(u->seed, 1, (uint64_t)i) >> 40) * (1.0f / 16777216.0f);
        u->out[i] = u->lo + (u->hi - u->lo) * f;
    }
}
/* out[i] ~ U[lo, hi) fp32, counter-based on (seed, i). */
void gen_uniform_f32(uint64_t seed, int64_t count, float lo, float hi, float* out, int nt) {
    unif_ctx c = {seed, lo, hi, out};
    parallel_for(count, nt, unif_body, &c);
}

typedef struct { uint64_t seed; int lo, hi; float* out; } int_ctx;
static void int_body(void* c, int64_t lo, int64_t hi) {
    int_ctx* u = (int_ctx*)c;
    uint64_t span = (uint64_t)(u->hi - u->lo + 1);
    for (int64_t i = lo; i < hi; ++i)
        u->out[i] = (float)(u->lo + (int)(rng(u->seed, 2, (uint64_t)i) % span));
}
/* out[i] = uniform integer in [lo, hi] stored as fp32 (exactness tests). */
void gen_int_f32(uint64_t seed, int64_t count, int lo, int hi, float* out, int nt) {
    int_ctx c = {seed, lo, hi, out};
    parallel_for(count, nt, int_body, &c);
}

typedef struct { const int32_t* rowptr; const int32_t* colidx; int64_t n; float* out; } norm_ctx;
static void norm_body(void* c, int64_t lo, int64_t hi) {
    norm_ctx* u = (norm_ctx*)c;
    for (int64_t i = lo; i < hi; ++i) {
        int32_t di = u->rowptr[i + 1] - u->rowptr[i];
        double a = di > 1 ? (double)di : 1.0;
        for (int32_t p = u->rowptr[i]; p < u->rowptr[i + 1]; ++p) {
            int32_t j = u->colidx[p];
            int32_t dj = (j < u->n) ? u->rowptr[j + 1] - u->rowptr[j] : 1;
            double b = dj > 1 ? (double)dj : 1.0;
            u->out[p] = (float)(1.0 / sqrt(a * b));
        }
    }
}
/* GCN-normalisation-like benchmark values: 1/sqrt(max(1,d_i) max(1,d_j)) (d = row degree). */
void gen_gcn_vals(int64_t n, const int32_t* rowptr, const int32_t* colidx, float* out, int nt) {
    norm_ctx c = {rowptr, colidx, n, out};
    parallel_for(n, nt, norm_body, &c);
}

/* ---------------------------------------------------------------- permutations */
/* Seeded Fisher-Yates permutation of [0,n) (sequential, counter based). */
void gen_permutation(uint64_t seed, int64_t n, int32_t* perm) {
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    for (int64_t i = n - 1; i > 0; --i) {
        int64_t j = (int64_t)(rng(seed, 3, (uint64_t)i) % (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
}

/* ---------------------------------------------------------------- CSR helpers */
typedef struct { const int32_t* rowptr; int32_t* colidx; } sortrows_ctx;
static void sortrows_body(void* c, int64_t lo, int64_t hi) {
    sortrows_ctx* u = (sortrows_ctx*)c;
    for (int64_t i = lo; i < hi; ++i) {
        int32_t a = u->rowptr[i], b = u->rowptr[i + 1];
        if (b - a > 1) qsort(u->colidx + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
    }
}
static void sort_rows(int64_t n, const int32_t* rowptr, int32_t* colidx, int nt) {
    sortrows_ctx c = {rowptr, colidx};
    parallel_for(n, nt, sortrows_body, &c);
}

/* Relabel rows and columns of a CSR by perm (new id = perm[old]); columns re-sorted. */
static void relabel_csr(int64_t n, const int32_t* perm, const int32_t* rp_in, const int32_t* ci_in,
                        int32_t* rp_out, int32_t* ci_out, int nt) {
    int32_t* inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) inv[perm[i]] = (int32_t)i;
    rp_out[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        int32_t old = inv[r];
        rp_out[r + 1] = rp_out[r] + (rp_in[old + 1] - rp_in[old]);
    }
    for (int64_t r = 0; r < n; ++r) {
        int32_t old = inv[r];
        int32_t d = rp_in[old + 1] - rp_in[old];
        for (int32_t k = 0; k < d; ++k) ci_out[rp_out[r] + k] = perm[ci_in[rp_in[old] + k]];
    }
    free(inv);
    sort_rows(n, rp_out, ci_out, nt);
}

/* ---------------------------------------------------------------- Chung-Lu power law */
static double ratio_for_alpha(int64_t n, double alpha) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += pow((double)(i + 1), -alpha);
    return (double)n / s; /* max / mean of w_i = (i+1)^-alpha */
}
double gen_chung_lu_alpha(int64_t n, double max_over_mean) {
    double lo = 0.0, hi = 8.0;
    for (int it = 0; it < 100; ++it) {
        double mid = 0.5 * (lo + hi);
        if (ratio_for_alpha(n, mid) < max_over_mean) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

typedef struct { double frac; int64_t idx; } fr_t;
static int cmp_fr(const void* a, const void* b) {
    const fr_t* x = (const fr_t*)a; const fr_t* y = (const fr_t*)b;
    if (x->frac != y->frac) return x->frac > y->frac ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

typedef struct {
    int64_t n; const double* cdf; const int32_t* rowptr; int32_t* colidx; uint64_t seed;
} cl_ctx;
static void cl_body(void* c, int64_t lo, int64_t hi) {
    cl_ctx* u = (cl_ctx*)c;
    int64_t n = u->n;
    uint8_t* seen = (uint8_t*)calloc((size_t)n, 1);
    for (int64_t i = lo; i < hi; ++i) {
        int32_t a = u->rowptr[i], d = u->rowptr[i + 1] - a;
        uint64_t k = 0;
        if ((int64_t)d * 2 > n) {   /* near-dense row (tiny graphs only): unweighted subset */
            int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
            for (int64_t j = 0; j < n; ++j) tmp[j] = (int32_t)j;
            for (int32_t t = 0; t < d; ++t) {
                int64_t j = t + (int64_t)(rng(u->seed, 4 + (uint64_t)i, k++) % (uint64_t)(n - t));
                int32_t x = tmp[t]; tmp[t] = tmp[j]; tmp[j] = x;
                u->colidx[a + t] = tmp[t];
            }
            free(tmp);
            continue;
        }
        for (int32_t t = 0; t < d;) {
            double x = u01(rng(u->seed, 4 + (uint64_t)i, k++)) * u->cdf[n - 1];
            int64_t l = 0, h = n - 1;             /* first index with cdf > x */
            while (l < h) { int64_t m = (l + h) >> 1; if (u->cdf[m] > x) h = m; else l = m + 1; }
            if (seen[l]) continue;                 /* distinct columns: reject repeats */
            seen[l] = 1;
            u->colidx[a + t++] = (int32_t)l;
        }
        for (int32_t t = 0; t < d; ++t) seen[u->colidx[a + t]] = 0;
    }
    free(seen);
}

/*
 * Chung-Lu power-law CSR: n x n, exactly nnz entries, degrees proportional to
 * w_i = (i+1)^-alpha (alpha by bisection so that max/mean degree = max_over_mean,
 * PAPER.md:164 "degrees up to 66 times greater than the average"), integer degrees by
 * largest remainder (capped at n), distinct columns drawn proportional to w, then one
 * seeded relabel of rows and columns (if relabel != 0), columns sorted per row.
 * Returns alpha.
 */
double gen_chung_lu(int64_t n, int64_t nnz, double max_over_mean, uint64_t seed, int relabel,
                    int32_t* rowptr, int32_t* colidx, int nt) {
    double alpha = gen_chung_lu_alpha(n, max_over_mean);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)n);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { w[i] = pow((double)(i + 1), -alpha); s += w[i]; cdf[i] = s; }
    int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    fr_t* fr = (fr_t*)malloc(sizeof(fr_t) * (size_t)n);
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        double e = (double)nnz * w[i] / s;
        deg[i] = (int64_t)floor(e);
        if (deg[i] > n) deg[i] = n;
        fr[i].frac = e - floor(e); fr[i].idx = i;
        tot += deg[i];
    }
    qsort(fr, (size_t)n, sizeof(fr_t), cmp_fr);
    for (int64_t k = 0; tot < nnz; k = (k + 1) % n) {
        int64_t i = fr[k].idx;
        if (deg[i] < n) { deg[i]++; tot++; }
    }
    int32_t* rp = relabel ? (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1)) : rowptr;
    int32_t* ci = relabel ? (int32_t*)malloc(sizeof(int32_t) * (size_t)nnz) : colidx;
    rp[0] = 0;
    for (int64_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + (int32_t)deg[i];
    cl_ctx c = {n, cdf, rp, ci, seed};
    parallel_for(n, nt, cl_body, &c);
    if (relabel) {
        int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        gen_permutation(seed ^ 0x5EEDull, n, perm);
        relabel_csr(n, perm, rp, ci, rowptr, colidx, nt);
        free(perm); free(rp); free(ci);
    } else {
        sort_rows(n, rowptr, colidx, nt);
    }
    free(w); free(cdf); free(deg); free(fr);
    return alpha;
}

/* ---------------------------------------------------------------- R-MAT (Graph500) */
typedef struct {
    int scale; double a, b, c; uint64_t seed; int32_t* src; int32_t* dst;
} rmat_ctx;
static void rmat_body(void* cx, int64_t lo, int64_t hi) {
    rmat_ctx* u = (rmat_ctx*)cx;
    const double ab = u->a + u->b, abc = u->a + u->b + u->c;
    for (int64_t e = lo; e < hi; ++e) {
        uint32_t r = 0, col = 0;
        uint64_t word = 0;
        for (int l = 0; l < u->scale; ++l) {
            if (l % 3 == 0) word = rng(u->seed, 7, (uint64_t)e * 16 + (uint64_t)(l / 3));
            double x = (double)((word >> (21 * (l % 3))) & 0x1FFFFF) * (1.0 / 2097152.0);
            uint32_t bit = 1u << l;
            if (x < u->a) { }
            else if (x < ab) col |= bit;
            else if (x < abc) r |= bit;
            else { r |= bit; col |= bit; }
        }
        u->src[e] = (int32_t)r; u->dst[e] = (int32_t)col;
    }
}
/*
 * Graph500 Kronecker / R-MAT: 2^scale vertices, edge_factor * 2^scale directed edges,
 * quadrant probabilities (a, b, c, 1-a-b-c), no noise; self loops and duplicates kept
 * (so nnz is exact); one seeded vertex relabel; CSR with columns sorted per row.
 */
void gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
              int32_t* rowptr, int32_t* colidx, int nt) {
    int64_t n = (int64_t)1 << scale, m = n * edge_factor;
    int32_t* src = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    int32_t* dst = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    rmat_ctx cx = {scale, a, b, c, seed, src, dst};
    parallel_for(m, nt, rmat_body, &cx);
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    gen_permutation(seed ^ 0xA11CEull, n, perm);
    memset(rowptr, 0, sizeof(int32_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; ++e) rowptr[perm[src[e]] + 1]++;
    for (int64_t i = 0; i < n; ++i) rowptr[i + 1] += rowptr[i];
    int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(fill, rowptr, sizeof(int32_t) * (size_t)n);
    for (int64_t e = 0; e < m; ++e) colidx[fill[perm[src[e]]]++] = perm[dst[e]];
    sort_rows(n, rowptr, colidx, nt);
    free(src); free(dst); free(perm); free(fill);
}
