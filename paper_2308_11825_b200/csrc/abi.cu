// abi.cu -- the extern "C" entry points of include/agcn.h: argument checks, error state,
// plan lifetime and introspection, row shards, and the host-buffer end-to-end call.
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "internal.h"

namespace agcn {

std::atomic<uint64_t> g_launches{0};

namespace {
thread_local agcn_status_t t_status = AGCN_OK;
thread_local std::string t_msg;
}  // namespace

void set_error(agcn_status_t code, const std::string& msg) {
    t_status = code;
    t_msg = msg;
}
void clear_error() {
    t_status = AGCN_OK;
    t_msg.clear();
}
agcn_status_t last_status() { return t_status; }
const char* last_message() { return t_msg.c_str(); }
agcn_status_t cuda_status(cudaError_t e) {
    return e == cudaErrorMemoryAllocation ? AGCN_ERR_OOM : AGCN_ERR_CUDA;
}

agcn_plan_s* build_plan(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz,
                        const agcn_opts_t& o);
void free_plan_arrays(agcn_plan_s* p);
void auto_partition(int64_t n, int64_t nnz, int32_t sms, int32_t* mbw, int32_t* mwn);
void plan_copy_sorted_colidx(agcn_plan_s* p, int32_t* host_dst);

namespace {

// nnz-balanced shard bounds: bounds[p] = first r with rowptr[r] - rowptr[0] >= floor(p nnz / P)
__global__ void k_shard_bounds(const int32_t* __restrict__ rowptr, int64_t n, int32_t P,
                               int64_t* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    const int64_t base = rowptr[0], nnz = (int64_t)rowptr[n] - base;
    if (p == 0) { out[0] = 0; return; }
    if (p == P) { out[P] = n; return; }
    const int64_t target = base + (p * nnz) / P;
    int64_t lo = 0, hi = n;  // first r in [0, n] with rowptr[r] >= target
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)rowptr[mid] < target) lo = mid + 1; else hi = mid;
    }
    out[p] = lo;
}

bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb) {
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

}  // namespace
}  // namespace agcn

using namespace agcn;

extern "C" {

void agcn_default_opts(agcn_opts_t* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->max_block_warps = 12;
    o->max_warp_nzs = 32;
    o->partition = AGCN_PARTITION_BLOCK;
    o->validate = 1;
    o->hot_rows = -1;
    o->small_plan = 1;
}

agcn_plan_t agcn_plan_ex(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz,
                         const agcn_opts_t* opts) {
    agcn_plan_t out = nullptr;
    guarded([&] {
        agcn_opts_t o;
        if (opts) o = *opts; else agcn_default_opts(&o);
        if (nnz < 0 && n >= 0 && rowptr) {  // "derive nnz": one readback of rowptr[0], rowptr[n]
            int32_t ends[2];
            cudaStream_t s = (cudaStream_t)o.stream;
            AGCN_CUDA(cudaMemcpyAsync(ends, rowptr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            AGCN_CUDA(cudaMemcpyAsync(ends + 1, rowptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            AGCN_CUDA(cudaStreamSynchronize(s));
            nnz = (int64_t)ends[1] - ends[0];
            AGCN_CHECK(nnz >= 0, AGCN_ERR_BAD_CSR, "rowptr[n] < rowptr[0]");
        }
        out = build_plan(rowptr, colidx, n, nnz, o);
    });
    return out;
}

agcn_plan_t agcn_plan(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz) {
    return agcn_plan_ex(rowptr, colidx, n, nnz, nullptr);
}

void agcn_default_spmm_opts(agcn_spmm_opts_t* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->kernel = AGCN_KERNEL_AUTO;
    o->l2_hint = AGCN_L2_AUTO;
    o->hot_mb = 0;
}

agcn_status_t agcn_spmm_ex(agcn_plan_t plan, const float* vals, const float* X, int32_t F, float* Y,
                           agcn_stream_t stream, const agcn_spmm_opts_t* opts) {
    return guarded([&] {
        AGCN_CHECK(plan != nullptr, AGCN_ERR_INVALID_ARG, "plan is NULL");
        AGCN_CHECK(F > 0, AGCN_ERR_INVALID_ARG, "F must be > 0");
        agcn_spmm_opts_t o;
        if (opts) o = *opts; else agcn_default_spmm_opts(&o);
        AGCN_CHECK(o.kernel >= AGCN_KERNEL_AUTO && o.kernel <= AGCN_KERNEL_WIDE, AGCN_ERR_INVALID_ARG,
                   "unknown kernel");
        AGCN_CHECK(o.l2_hint >= AGCN_L2_AUTO && o.l2_hint <= AGCN_L2_HOT_HINTS, AGCN_ERR_INVALID_ARG,
                   "l2_hint must be -1 .. 3 (agcn_l2_hint_t)");
        AGCN_CHECK(o.hot_mb >= 0, AGCN_ERR_INVALID_ARG, "hot_mb must be >= 0");
        AGCN_CHECK(o.chunk_shape == -1 || o.chunk_shape == 0 || o.chunk_shape == 3 || o.chunk_shape == 4 ||
                       o.chunk_shape == 6, AGCN_ERR_INVALID_ARG, "chunk_shape must be -1, 0, 3, 4 or 6");
        AGCN_CHECK(o.chunk_order == 0 || o.chunk_order == -1, AGCN_ERR_INVALID_ARG, "chunk_order must be 0 or -1");
        AGCN_CHECK(o.aggregation == AGCN_AGG_SUM || o.aggregation == AGCN_AGG_MEAN, AGCN_ERR_INVALID_ARG,
                   "unknown aggregation");
        AGCN_CHECK(o.self_scale == 0.f || o.self != nullptr, AGCN_ERR_INVALID_ARG,
                   "self_scale != 0 needs the self matrix");
        AGCN_CHECK(((reinterpret_cast<uintptr_t>(o.self) | reinterpret_cast<uintptr_t>(o.bias)) & 15u) == 0,
                   AGCN_ERR_INVALID_ARG, "self and bias must be 16-byte aligned");
        AGCN_CHECK(o.npeer >= 0 && o.npeer <= kMaxPeers, AGCN_ERR_INVALID_ARG, "npeer must be in [0, 8]");
        for (int q = 0; q < o.npeer; ++q)
            AGCN_CHECK(o.peer_out[q] && (reinterpret_cast<uintptr_t>(o.peer_out[q]) & 15u) == 0,
                       AGCN_ERR_INVALID_ARG, "peer_out pointers must be non-NULL and 16-byte aligned");
        if (plan->n == 0) return;
        AGCN_CHECK(Y != nullptr, AGCN_ERR_INVALID_ARG, "Y is NULL");
        AGCN_CHECK(plan->nnz == 0 || (vals != nullptr && X != nullptr), AGCN_ERR_INVALID_ARG,
                   "vals / X is NULL");
        AGCN_CHECK((int64_t)F * std::max<int64_t>(plan->n, plan->x_rows) < (1ll << 40),
                   AGCN_ERR_INVALID_ARG, "F too large");
        AGCN_CHECK(X == nullptr || X != Y, AGCN_ERR_INVALID_ARG, "X and Y must not alias");
        if (X) {
            const size_t nx = sizeof(float) * (size_t)plan->x_rows * F;
            const size_t ny = sizeof(float) * (size_t)plan->n * F;
            AGCN_CHECK(!ranges_overlap(X, nx, Y, ny), AGCN_ERR_INVALID_ARG, "X and Y overlap");
        }
        spmm_launch(plan, vals, X, F, Y, (cudaStream_t)stream, o);
    });
}

agcn_status_t agcn_spmm(agcn_plan_t plan, const float* vals, const float* X, int32_t F, float* Y,
                        agcn_stream_t stream) {
    return agcn_spmm_ex(plan, vals, X, F, Y, stream, nullptr);
}

agcn_status_t agcn_plan_destroy(agcn_plan_t plan) {
    return guarded([&] {
        if (!plan) return;
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != plan->device) cudaSetDevice(plan->device);
        free_plan_arrays(plan);  // stream-ordered: no host synchronisation
        if (cur != plan->device) cudaSetDevice(cur);
        delete plan;
    });
}

agcn_status_t agcn_plan_stats(agcn_plan_t plan, agcn_plan_stats_t* out) {
    return guarded([&] {
        AGCN_CHECK(plan && out, AGCN_ERR_INVALID_ARG, "NULL argument");
        std::memset(out, 0, sizeof(*out));
        out->n = plan->n;
        out->n_cols = plan->n_cols;
        out->nnz = plan->nnz;
        out->nblocks = plan->nblocks;
        out->ntasks = plan->ntasks;
        out->deg_bound = plan->deg_bound;
        out->max_deg = plan->max_deg;
        out->n_zero_rows = plan->n_zero;
        out->n_oversized_rows = plan->n_ov;
        out->n_oversized_blocks = plan->ov_chunks;
        out->max_block_warps = plan->mbw;
        out->max_warp_nzs = plan->mwn;
        out->partition = plan->partition;
        out->device_bytes = plan->device_bytes + plan->ov_partial_floats * sizeof(float) +
                            plan->xhot_floats * sizeof(float);
        out->hot_rows = plan->n_hot;
    });
}

agcn_status_t agcn_plan_copy(agcn_plan_t plan, int32_t field, void* host_dst, size_t bytes) {
    return guarded([&] {
        AGCN_CHECK(plan && host_dst, AGCN_ERR_INVALID_ARG, "NULL argument");
        const void* src = nullptr;
        size_t want = 0;
        const bool blk = plan->partition == AGCN_PARTITION_BLOCK;
        switch (field) {
            case AGCN_FIELD_PERM: src = plan->perm; want = 4 * (size_t)plan->n; break;
            case AGCN_FIELD_BLOCKS: src = plan->desc; want = 16 * (size_t)plan->nblocks; break;
            case AGCN_FIELD_SORTED_COLIDX: src = plan->perm; want = 4 * (size_t)plan->nnz; break;
            case AGCN_FIELD_ROW_SRC_OFF: src = plan->row_src_off; want = 4 * (size_t)plan->n; break;
            case AGCN_FIELD_TASKS: src = plan->tasks; want = 16 * (size_t)plan->ntasks; break;
            case AGCN_FIELD_SORTED_ROWPTR: src = plan->sorted_rowptr; want = 4 * (size_t)(plan->n + 1); break;
            case AGCN_FIELD_HOT_COLS: src = plan->hot_cols; want = 4 * (size_t)plan->n_hot; break;
            default: throw Error{AGCN_ERR_INVALID_ARG, "unknown field"};
        }
        const bool is_task = field == AGCN_FIELD_TASKS;
        AGCN_CHECK(is_task ? !blk : blk, AGCN_ERR_INVALID_ARG, "field not present for this partition");
        AGCN_CHECK(bytes == want, AGCN_ERR_INVALID_ARG,
                   "bytes must equal the field size (" + std::to_string(want) + ")");
        if (field == AGCN_FIELD_SORTED_COLIDX) {  // hot encoding undone on the way
            plan_copy_sorted_colidx(plan, static_cast<int32_t*>(host_dst));
            return;
        }
        if (want) AGCN_CUDA(cudaMemcpy(host_dst, src, want, cudaMemcpyDeviceToHost));
    });
}

agcn_status_t agcn_auto_partition(int64_t n, int64_t nnz, int32_t sms, int32_t* max_block_warps,
                                  int32_t* max_warp_nzs) {
    return guarded([&] {
        AGCN_CHECK(n >= 0 && nnz >= 0 && max_block_warps && max_warp_nzs, AGCN_ERR_INVALID_ARG,
                   "n, nnz must be >= 0 and the outputs non-NULL");
        auto_partition(n, nnz, sms, max_block_warps, max_warp_nzs);
    });
}

agcn_status_t agcn_shard_bounds(const int32_t* rowptr, int64_t n, int32_t nranks, int64_t* bounds_host,
                                agcn_stream_t stream) {
    return guarded([&] {
        AGCN_CHECK(rowptr && bounds_host && n >= 0 && nranks >= 1, AGCN_ERR_INVALID_ARG, "bad argument");
        cudaStream_t s = (cudaStream_t)stream;
        Scratch tmp(s);
        int64_t* d = tmp.alloc<int64_t>(nranks + 1);
        k_shard_bounds<<<(nranks + 1 + 127) / 128, 128, 0, s>>>(rowptr, n, nranks, d);
        post_launch();
        AGCN_CUDA(cudaMemcpyAsync(bounds_host, d, sizeof(int64_t) * (nranks + 1), cudaMemcpyDeviceToHost, s));
        AGCN_CUDA(cudaStreamSynchronize(s));
    });
}

agcn_status_t agcn_propagate_host(const int32_t* rowptr_h, const int32_t* colidx_h, const float* vals_h,
                                  int64_t n, int64_t nnz, const float* X_h, int32_t F, int32_t layers,
                                  float* Y_h, const agcn_opts_t* opts) {
    return guarded([&] {
        AGCN_CHECK(rowptr_h && X_h && Y_h && F > 0 && layers >= 1 && n >= 0 && nnz >= 0,
                   AGCN_ERR_INVALID_ARG, "bad argument");
        AGCN_CHECK(nnz == 0 || (colidx_h && vals_h), AGCN_ERR_INVALID_ARG, "colidx / vals is NULL");
        agcn_opts_t o;
        if (opts) o = *opts; else agcn_default_opts(&o);
        AGCN_CHECK(o.col_nparts == 0, AGCN_ERR_INVALID_ARG, "padded layouts are not supported here");
        const int64_t n_cols = o.n_cols > 0 ? o.n_cols : n;
        AGCN_CHECK(layers == 1 || n_cols == n, AGCN_ERR_INVALID_ARG, "layers > 1 needs a square A");
        cudaStream_t s = (cudaStream_t)o.stream;
        const size_t xb = sizeof(float) * (size_t)n_cols * F, yb = sizeof(float) * (size_t)n * F;
        struct Sync {       // the call is synchronous, also when it fails half-way (destroyed last)
            cudaStream_t s;
            ~Sync() { cudaStreamSynchronize(s); }
        } sync{s};
        struct PlanGuard {  // plan arrays + scratch released (stream-ordered) on every exit path
            agcn_plan_s* p = nullptr;
            ~PlanGuard() {
                if (p) { free_plan_arrays(p); delete p; }
            }
        } pg;
        Scratch tmp(s);
        int32_t* rp = tmp.alloc<int32_t>(n + 1);
        int32_t* ci = tmp.alloc<int32_t>(nnz);
        float* va = tmp.alloc<float>(nnz);
        float* x = tmp.alloc<float>((size_t)n_cols * F);
        float* y = tmp.alloc<float>((size_t)n * F);
        float* y2 = layers > 1 ? tmp.alloc<float>((size_t)n * F) : nullptr;
        // colidx_h / vals_h are indexed by rowptr values: copy the [rowptr[0], rowptr[n]) run
        const int32_t base = rowptr_h[0];
        AGCN_CUDA(cudaMemcpyAsync(rp, rowptr_h, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
        if (nnz) {
            AGCN_CUDA(cudaMemcpyAsync(ci, colidx_h + base, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
            AGCN_CUDA(cudaMemcpyAsync(va, vals_h + base, sizeof(float) * nnz, cudaMemcpyHostToDevice, s));
        }
        AGCN_CUDA(cudaMemcpyAsync(x, X_h, xb, cudaMemcpyHostToDevice, s));
        pg.p = build_plan(rp, ci - base, n, nnz, o);
        agcn_spmm_opts_t so;
        agcn_default_spmm_opts(&so);
        const float* cur = x;
        float* out = y;
        for (int l = 0; l < layers; ++l) {
            spmm_launch(pg.p, va - base, cur, F, out, s, so);
            cur = out;
            out = (out == y) ? y2 : y;
        }
        AGCN_CUDA(cudaMemcpyAsync(Y_h, cur, yb, cudaMemcpyDeviceToHost, s));
        AGCN_CUDA(cudaStreamSynchronize(s));
    });
}

agcn_status_t agcn_transpose(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t n_cols,
                             int64_t nnz, int32_t* rowptr_t, int32_t* colidx_t, int32_t* src,
                             agcn_stream_t stream) {
    return guarded([&] { transpose_csr(rowptr, colidx, n, n_cols, nnz, rowptr_t, colidx_t, src, (cudaStream_t)stream); });
}

agcn_status_t agcn_gather_vals(const float* vals, const int32_t* src, int64_t nnz, float* out,
                               agcn_stream_t stream) {
    return guarded([&] { gather_vals(vals, src, nnz, out, (cudaStream_t)stream); });
}

agcn_status_t agcn_gemm_xw(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y,
                           const float* bias, int32_t relu, agcn_stream_t stream) {
    return guarded([&] { gemm_xw_tf32(X, M, K, Wt, N, Y, bias, relu, (cudaStream_t)stream); });
}

agcn_status_t agcn_gemm_xw_ex(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y,
                              const float* bias, int32_t relu, int32_t precision, agcn_stream_t stream) {
    return guarded([&] {
        AGCN_CHECK(precision == AGCN_GEMM_FP32 || precision == AGCN_GEMM_TF32, AGCN_ERR_INVALID_ARG, "unknown precision");
        if (precision == AGCN_GEMM_TF32)
            gemm_xw_tf32(X, M, K, Wt, N, Y, bias, relu, (cudaStream_t)stream);
        else
            gemm_xw_fp32(X, M, K, Wt, N, Y, bias, relu, (cudaStream_t)stream);
    });
}

agcn_status_t agcn_device_alloc(size_t bytes, void** ptr) {
    return guarded([&] {
        AGCN_CHECK(ptr != nullptr, AGCN_ERR_INVALID_ARG, "ptr is NULL");
        *ptr = nullptr;
        AGCN_CUDA(cudaMalloc(ptr, bytes ? bytes : 16));
    });
}

agcn_status_t agcn_device_free(void* ptr) {
    return guarded([&] {
        if (ptr) AGCN_CUDA(cudaFree(ptr));
    });
}

agcn_status_t agcn_ipc_export(const void* ptr, void* handle64) {
    return guarded([&] {
        AGCN_CHECK(ptr && handle64, AGCN_ERR_INVALID_ARG, "NULL pointer");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
        cudaIpcMemHandle_t h;
        AGCN_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
        memcpy(handle64, &h, sizeof(h));
    });
}

agcn_status_t agcn_ipc_open(const void* handle64, void** ptr) {
    return guarded([&] {
        AGCN_CHECK(handle64 && ptr, AGCN_ERR_INVALID_ARG, "NULL pointer");
        cudaIpcMemHandle_t h;
        memcpy(&h, handle64, sizeof(h));
        AGCN_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

agcn_status_t agcn_ipc_close(void* ptr) {
    return guarded([&] {
        if (ptr) AGCN_CUDA(cudaIpcCloseMemHandle(ptr));
    });
}

agcn_status_t agcn_last_status(void) { return agcn::last_status(); }
const char* agcn_last_error(void) { return agcn::last_message(); }
uint64_t agcn_launch_count(void) { return agcn::g_launches.load(); }
const char* agcn_version(void) { return "agcn 0.1 sm_100a (Accel-GCN arXiv 2308.11825)"; }

}  // extern "C"
