// transpose.cu -- agcn_transpose / agcn_gather_vals: the CSR of A^T on the device, for the
// backward pass of a GCN layer (dX = A^T . dY).
//
// A stable counting sort of the nonzeros by column (the same stable LSD radix machinery as
// the degree sort of P:295, plan.cu): within a row of A^T (a column of A) the entries keep
// increasing original-row order.  Outputs the row pointer of A^T, its column indices (the
// original rows) and, per entry of A^T, the index of its entry in A (src), so that any values
// array of A maps to A^T with one gather (agcn_gather_vals) and one plan of A^T serves every
// backward step.
#include <algorithm>

#include "internal.h"

namespace agcn {
namespace {

// keys = colidx (the run starting at rowptr[0]), vals = entry index; column counts
__global__ void k_tr_init(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx_g, int64_t nnz,
                          int32_t* __restrict__ keys, int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
    const int32_t* __restrict__ colidx = colidx_g + __ldg(rowptr);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = __ldcs(colidx + q);
        keys[q] = c;
        idx[q] = (int32_t)q;
        atomicAdd(&cnt[c], 1);
    }
}

// row id of every entry of A (one warp per row)
__global__ void k_row_ids(const int32_t* __restrict__ rowptr, int64_t n, int32_t* __restrict__ rowid) {
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int32_t base = __ldg(rowptr);
    for (int64_t i = w0; i < n; i += W) {
        const int32_t a = rowptr[i] - base, b = rowptr[i + 1] - base;
        for (int32_t q = a + lane; q < b; q += 32) rowid[q] = (int32_t)i;
    }
}

__global__ void k_tr_cols(const int32_t* __restrict__ src, const int32_t* __restrict__ rowid, int64_t nnz,
                          int32_t* __restrict__ colidx_t) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        colidx_t[k] = rowid[src[k]];
}

__global__ void k_gather_vals(const float* __restrict__ vals, const int32_t* __restrict__ src, int64_t nnz,
                              float* __restrict__ out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        out[k] = __ldg(vals + __ldg(src + k));
}

inline unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void transpose_csr(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t n_cols, int64_t nnz,
                   int32_t* rowptr_t, int32_t* colidx_t, int32_t* src, cudaStream_t s) {
    AGCN_CHECK(rowptr && rowptr_t && n >= 0 && n_cols >= 0 && nnz >= 0, AGCN_ERR_INVALID_ARG, "bad argument");
    AGCN_CHECK(nnz == 0 || (colidx && colidx_t && src), AGCN_ERR_INVALID_ARG, "colidx / outputs are NULL");
    AGCN_CHECK(nnz < (1ll << 31) && n < (1ll << 31) && n_cols < (1ll << 31), AGCN_ERR_INVALID_ARG,
               "sizes must be < 2^31");
    Scratch tmp(s);
    int32_t* cnt = rowptr_t;  // column counts, scanned in place into the row pointer of A^T
    AGCN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_cols + 1), s));
    if (nnz > 0) {
        int32_t* ka = tmp.alloc<int32_t>(nnz);
        int32_t* kb = tmp.alloc<int32_t>(nnz);
        int32_t* vb = tmp.alloc<int32_t>(nnz);
        int32_t* va = src;   // the entry indices end up in src (copied if the sort ends in vb)
        k_tr_init<<<grid_for(nnz), 256, 0, s>>>(rowptr, colidx, nnz, ka, va, cnt);
        post_launch();
        radix_sort_pairs(ka, va, kb, vb, nnz, std::max<int64_t>(n_cols - 1, 0), s);
        if (va != src) AGCN_CUDA(cudaMemcpyAsync(src, va, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
        int32_t* rowid = kb == src ? ka : kb;  // a free nnz buffer (not src)
        if (n > 0) {
            k_row_ids<<<grid_for(n * 32), 256, 0, s>>>(rowptr, n, rowid);
            post_launch();
        }
        k_tr_cols<<<grid_for(nnz), 256, 0, s>>>(src, rowid, nnz, colidx_t);
        post_launch();
    }
    exclusive_scan_i32(cnt, rowptr_t, n_cols, s);
}

void gather_vals(const float* vals, const int32_t* src, int64_t nnz, float* out, cudaStream_t s) {
    AGCN_CHECK(nnz >= 0 && (nnz == 0 || (vals && src && out)), AGCN_ERR_INVALID_ARG, "bad argument");
    if (nnz == 0) return;
    k_gather_vals<<<grid_for(nnz), 256, 0, s>>>(vals, src, nnz, out);
    post_launch();
}

}  // namespace agcn
