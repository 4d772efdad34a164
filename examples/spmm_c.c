/*
 * spmm_c.c -- the C ABI used from plain C (no Python, no torch): a small power-law CSR, its
 * plan (degree sort + Alg. 1/2, P:295 / P:314-382), one SpMM Y = A.X through
 * agcn_spmm, and the propagation on host buffers (agcn_propagate_host), each checked against a
 * straightforward double-precision loop.  Device memory comes from agcn_device_alloc.
 *
 * build: gcc -O2 -std=c11 examples/spmm_c.c -Iinclude -I/usr/local/cuda/include \
 *            -Lpaper_2308_11825_b200 -lagcn -L/usr/local/cuda/lib64 -lcudart -lm \
 *            -Wl,-rpath,$PWD/paper_2308_11825_b200:/usr/local/cuda/lib64 -o /tmp/spmm_c
 * run:   /tmp/spmm_c          (exit 0 and "ok" on success)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "agcn.h"

enum { H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost };

#define CHECK(x)                                                                     \
    do {                                                                             \
        agcn_status_t st__ = (x);                                                    \
        if (st__ != AGCN_OK) {                                                       \
            fprintf(stderr, "%s failed: %d %s\n", #x, (int)st__, agcn_last_error()); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static uint32_t next(void) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (uint32_t)(rng >> 11);
}

int main(void) {
    const int64_t n = 5000;
    const int32_t F = 64;
    int32_t* rowptr = malloc(sizeof(int32_t) * (n + 1));
    rowptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {                 /* heavy-tailed degrees, some zero rows */
        uint32_t r = next() % 1000;
        int32_t d = r < 300 ? 0 : r < 900 ? (int32_t)(1 + next() % 8) : r < 995 ? (int32_t)(1 + next() % 200)
                                                                               : (int32_t)(500 + next() % 3000);
        rowptr[i + 1] = rowptr[i] + d;
    }
    const int64_t nnz = rowptr[n];
    int32_t* colidx = malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
    float* vals = malloc(sizeof(float) * (size_t)(nnz ? nnz : 1));
    float* X = malloc(sizeof(float) * (size_t)n * F);
    float* Y = malloc(sizeof(float) * (size_t)n * F);
    for (int64_t k = 0; k < nnz; ++k) {
        colidx[k] = (int32_t)(next() % n);
        vals[k] = (float)((int32_t)(next() % 2001) - 1000) / 1000.f;
    }
    for (int64_t k = 0; k < n * F; ++k) X[k] = (float)((int32_t)(next() % 2001) - 1000) / 1000.f;

    /* device copies of the CSR and X; Y on the device */
    void *d_rp, *d_ci, *d_va, *d_X, *d_Y;
    CHECK(agcn_device_alloc(sizeof(int32_t) * (n + 1), &d_rp));
    CHECK(agcn_device_alloc(sizeof(int32_t) * (size_t)nnz, &d_ci));
    CHECK(agcn_device_alloc(sizeof(float) * (size_t)nnz, &d_va));
    CHECK(agcn_device_alloc(sizeof(float) * (size_t)n * F, &d_X));
    CHECK(agcn_device_alloc(sizeof(float) * (size_t)n * F, &d_Y));
    if (cudaMemcpy(d_rp, rowptr, sizeof(int32_t) * (n + 1), H2D) || cudaMemcpy(d_ci, colidx, sizeof(int32_t) * nnz, H2D) ||
        cudaMemcpy(d_va, vals, sizeof(float) * nnz, H2D) || cudaMemcpy(d_X, X, sizeof(float) * n * F, H2D)) {
        fprintf(stderr, "cudaMemcpy failed\n");
        return 1;
    }

    agcn_plan_t plan = agcn_plan(d_rp, d_ci, n, nnz);
    if (!plan) {
        fprintf(stderr, "agcn_plan failed: %s\n", agcn_last_error());
        return 1;
    }
    CHECK(agcn_device_free(d_ci));                  /* the plan copied colidx */
    d_ci = NULL;
    CHECK(agcn_spmm(plan, d_va, d_X, F, d_Y, NULL));
    if (cudaMemcpy(Y, d_Y, sizeof(float) * n * F, D2H)) return 1;
    agcn_plan_stats_t st;
    CHECK(agcn_plan_stats(plan, &st));

    /* check against the definition, per element |y - y_ref| <= 1e-5 sum|a x| + 1e-7 */
    int64_t fails = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int32_t k = 0; k < F; ++k) {
            double y = 0, s = 0;
            for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
                const double t = (double)vals[p] * (double)X[(int64_t)colidx[p] * F + k];
                y += t;
                s += fabs(t);
            }
            if (!(fabs((double)Y[i * F + k] - y) <= 1e-5 * s + 1e-7)) ++fails;
        }

    /* the same through agcn_propagate_host (host buffers end to end), one layer */
    float* Y2 = malloc(sizeof(float) * (size_t)n * F);
    CHECK(agcn_propagate_host(rowptr, colidx, vals, n, nnz, X, F, 1, Y2, NULL));
    const int same = memcmp(Y, Y2, sizeof(float) * (size_t)n * F) == 0;

    CHECK(agcn_plan_destroy(plan));
    agcn_device_free(d_rp);
    agcn_device_free(d_va);
    agcn_device_free(d_X);
    agcn_device_free(d_Y);
    printf("%s: n=%lld nnz=%lld nblocks=%lld oversized_rows=%lld fails=%lld propagate_host_equal=%d (%s)\n",
           fails == 0 && same ? "ok" : "FAIL", (long long)n, (long long)nnz, (long long)st.nblocks,
           (long long)st.n_oversized_rows, (long long)fails, same, agcn_version());
    return fails == 0 && same ? 0 : 1;
}
