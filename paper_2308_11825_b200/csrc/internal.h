// internal.h -- shared declarations of the agcn CUDA library (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <new>
#include <string>
#include <vector>

#include "../../include/agcn.h"
#include "colmap.cuh"

namespace agcn {

// ------------------------------------------------------------------ error state
void set_error(agcn_status_t code, const std::string& msg);
void clear_error();
agcn_status_t last_status();
const char* last_message();
agcn_status_t cuda_status(cudaError_t e);  // maps OOM -> AGCN_ERR_OOM, else AGCN_ERR_CUDA

struct Error {
    agcn_status_t code;
    std::string msg;
};

#define AGCN_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t e__ = (call);                                                          \
        if (e__ != cudaSuccess)                                                            \
            throw ::agcn::Error{::agcn::cuda_status(e__),                                  \
                                std::string(#call) + ": " + cudaGetErrorString(e__)};      \
    } while (0)

#define AGCN_CHECK(cond, code, msg)                                  \
    do {                                                             \
        if (!(cond)) throw ::agcn::Error{(code), std::string(msg)};  \
    } while (0)

// run f() behind the C ABI: exceptions become a status code + the thread's error message
template <class F>
agcn_status_t guarded(F&& f) {
    try {
        clear_error();
        f();
        return AGCN_OK;
    } catch (const Error& e) {
        set_error(e.code, e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error(AGCN_ERR_OOM, "host allocation failed");
        return AGCN_ERR_OOM;
    } catch (...) {
        set_error(AGCN_ERR_CUDA, "unknown exception");
        return AGCN_ERR_CUDA;
    }
}

// plan construction / release (plan.cu)
agcn_plan_s* build_plan(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz,
                        const agcn_opts_t& o);
void free_plan_arrays(agcn_plan_s* p);

// ------------------------------------------------------------------ launch accounting
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
// check the launch itself (configuration errors); never synchronises
inline void post_launch() {
    count_launch();
    AGCN_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocations (cudaMallocAsync): no device-wide synchronisation.
template <class T>
T* dalloc(size_t count, cudaStream_t s) {
    void* p = nullptr;
    if (count == 0) count = 1;
    AGCN_CUDA(cudaMallocAsync(&p, count * sizeof(T), s));
    return static_cast<T*>(p);
}
inline void dfree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Temporaries of one call: freed stream-ordered when the scope ends (also on errors).
class Scratch {
public:
    explicit Scratch(cudaStream_t s) : s_(s) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        for (void* p : ptrs_) cudaFreeAsync(p, s_);
    }
    template <class T>
    T* alloc(size_t count) {
        T* p = dalloc<T>(count, s_);
        ptrs_.push_back(p);
        return p;
    }

private:
    cudaStream_t s_;
    std::vector<void*> ptrs_;
};

// ------------------------------------------------------------------ scan (scan.cu)
// out[i] = sum_{j<i} in[i] for i in [0, n]; out has n+1 entries (out[n] = total).
// In-place (out == in) is allowed only if in has n+1 entries.  int32 values.
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s);

// ------------------------------------------------------------------ SpMM epilogue
// y_i = agg(i) * (mean ? 1/deg_i : 1) + self_scale * self[i] + bias; relu (agcn_spmm_opts_t)
constexpr int kMaxPeers = 8;
struct Epi {
    const float* self;
    const float* bias;
    float self_scale;
    int32_t mean, relu;
    int32_t F;
    int32_t npeer;                 // fused all-gather: output rows also stored to peer[q] + row * F
    float* peer[kMaxPeers];
    __host__ __device__ bool active() const { return mean || self || bias || relu || npeer; }
};

// the fused all-gather's extra copies of a finished output row slice (16 bytes at `off`)
__device__ __forceinline__ void fanout4(const Epi& e, int64_t off, const float4& v) {
    for (int q = 0; q < e.npeer; ++q) __stcs(reinterpret_cast<float4*>(e.peer[q] + off), v);
}
__device__ __forceinline__ void fanout1(const Epi& e, int64_t off, float v) {
    for (int q = 0; q < e.npeer; ++q) __stcs(e.peer[q] + off, v);
}

__device__ __forceinline__ float4 epi4(float4 y, int32_t deg, int64_t orow, int32_t c, const Epi& e) {
    if (e.mean) {
        const float sc = deg > 0 ? 1.f / (float)deg : 0.f;
        y.x *= sc; y.y *= sc; y.z *= sc; y.w *= sc;
    }
    if (e.self) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(e.self + orow * e.F + c));
        y.x = fmaf(e.self_scale, v.x, y.x); y.y = fmaf(e.self_scale, v.y, y.y);
        y.z = fmaf(e.self_scale, v.z, y.z); y.w = fmaf(e.self_scale, v.w, y.w);
    }
    if (e.bias) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(e.bias + c));
        y.x += v.x; y.y += v.y; y.z += v.z; y.w += v.w;
    }
    if (e.relu) {
        y.x = fmaxf(y.x, 0.f); y.y = fmaxf(y.y, 0.f); y.z = fmaxf(y.z, 0.f); y.w = fmaxf(y.w, 0.f);
    }
    return y;
}

__device__ __forceinline__ float epi1(float y, int32_t deg, int64_t orow, int32_t c, const Epi& e) {
    if (e.mean) y *= deg > 0 ? 1.f / (float)deg : 0.f;
    if (e.self) y = fmaf(e.self_scale, __ldg(e.self + orow * e.F + c), y);
    if (e.bias) y += __ldg(e.bias + c);
    if (e.relu) y = fmaxf(y, 0.f);
    return y;
}

// ------------------------------------------------------------------ plan object
struct PlanFlags {          // device-written, read back once (validation + sizes)
    int32_t bad_rowptr;     // rowptr decreases somewhere
    int32_t bad_colidx;     // colidx out of [0, n_cols)
    int32_t max_deg;
    int32_t rowptr_first;
    int32_t rowptr_last;
    int32_t n_ov_heavy;     // oversized rows of more than kHeavyChunks deg_bound chunks
    int32_t hot_tau;        // hot set from the histogram (k_hot_tau): rows of degree > hot_tau ...
    int32_t hot_first;      // ... and the degree-hot_tau rows of rank >= hot_first (row order)
    int32_t hot_fallback;   // 1: the threshold falls among the oversized rows (use the sorted tail)
    int64_t ov_chunks;      // sum over oversized rows of ceil(deg / deg_bound)
    int64_t ov_chunks_heavy;  // the part of ov_chunks from rows of degree >= kColBlockMinDeg
    int64_t n_hot;          // hot rows selected by k_hot_tau
};

constexpr int32_t kHeavyChunks = 16;     // oversized rows above this many chunks: CTA-wide merge
constexpr int32_t kColBlockMinDeg = 2048;  // (statistics only: chunks of rows at least this long)

}  // namespace agcn

struct agcn_plan_s {
    int device = 0;
    int64_t n = 0, n_cols = 0, nnz = 0;
    int32_t mbw = 12, mwn = 32, deg_bound = 384, partition = 0;
    int64_t x_rows = 0;  // rows of X the SpMM reads (n_cols, or the padded layout)
    int64_t rp_base = 0; // rowptr[0] (vals/colidx are indexed by rowptr values)

    // AGCN_PARTITION_BLOCK
    int64_t nblocks = 0, nb_small = 0, n_zero = 0, n_ov = 0, ov_start = 0, ov_chunks = 0;
    int64_t ov_chunks_heavy = 0;       // chunks of rows of degree >= kColBlockMinDeg
    int64_t n_ov_heavy = 0;            // oversized rows of more than kHeavyChunks chunks (a suffix)
    int64_t max_deg = 0;
    int32_t* perm = nullptr;           // [n]   sorted position -> original row
    int32_t* sorted_rowptr = nullptr;  // [n+1] row pointer of the degree-sorted CSR (P:295 (3))
    int32_t* row_src_off = nullptr;    // [n]   rowptr[perm[k]] - rowptr[0]
    // plan-owned column indices (the plan copies colidx):
    int32_t* cols_copy = nullptr;      // [nnz] colidx in the caller's order (rowptr-relative): the
                                       // SpMM reads it at row_src_off like vals; padded-layout
                                       // relabel applied; BLOCK plans: hot column -> -1 - slot
    int64_t n_hot = 0;                 // hot X rows (the n_hot highest-degree vertices, square A)
    int32_t* hot_cols = nullptr;       // [n_hot] column of hot slot k (slots in column order)
    float* xhot = nullptr;             // SpMM scratch: X rows of the hot slots [n_hot][F]
    size_t xhot_floats = 0;
    agcn::ColMap cmap{};               // optional padded-layout column relabel
    int4* desc = nullptr;              // [nblocks]
    int32_t* ov_chunk_start = nullptr; // [n_ov + 1]
    int32_t* ov_order = nullptr;       // [ov_chunks] execution order of the oversized chunks

    // AGCN_PARTITION_WARP
    int64_t ntasks = 0;
    int4* tasks = nullptr;             // [ntasks] (row, col, len, 0)
    int32_t* rowptr_copy = nullptr;    // [n+1] (rebased to 0)

    // SpMM scratch (oversized-row partial sums, chunk-major [ov_chunks][F])
    float* ov_partial = nullptr;
    size_t ov_partial_floats = 0;
    int32_t* ov_cnt = nullptr;         // [n_ov] finished-chunk counters of the fused level 3 (zero at rest)

    size_t device_bytes = 0;
    bool capturing = false;         // agcn_graph_create: SpMMs being captured (plan complete)
    std::atomic<int> n_graphs{0};   // live agcn_graph_t holding this plan's scratch pointers
    cudaStream_t stream = nullptr;  // stream the plan was built on
    cudaEvent_t ready = nullptr;    // recorded on `stream` when the plan is complete
    cudaEvent_t last_use = nullptr; // recorded after an SpMM issued on a stream != `stream`
};

namespace agcn {
void spmm_launch(agcn_plan_s* p, const float* vals, const float* X, int32_t F, float* Y,
                 cudaStream_t s, const agcn_spmm_opts_t& o);
// spmm_wide.cu: 256-bit-per-lane kernel for F = 8 L <= 256
bool wide_supported(const agcn_plan_s* p, const float* X, const float* Y, int32_t F);
// l2: agcn_l2_hint_t resolved (NONE / KEEP_ALL / HOT_WINDOW / HOT_HINTS); Xh: the hot rows
// (plans with n_hot > 0); win_bytes: the persisting window over Xh (HOT_WINDOW)
void launch_wide(agcn_plan_s* p, const float* vals, const float* X, const float* Xh, int32_t F, float* Y,
                 int l2, size_t win_bytes, bool fuse_ov, int chunk_shape, bool chunk_order, const Epi& epi,
                 cudaStream_t s);
// spmm.cu: set the device's persisting-L2 limit to at least `bytes` (once per device and size);
// returns the window size usable (0 if the device refuses)
size_t ensure_persisting_l2(size_t bytes);
// plan.cu: stable LSD radix sort of (key, val) pairs (8-bit digits); result in ka/va
void radix_sort_pairs(int32_t*& ka, int32_t*& va, int32_t*& kb, int32_t*& vb, int64_t m, int64_t max_key,
                      cudaStream_t s);
// gemm_tc.cu: Y = X W on tcgen05 (kind::tf32); Wt = W^T [N x K] row-major
void gemm_xw_tf32(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y, const float* bias,
                  int32_t relu, cudaStream_t s);
// fp32 accuracy: 3xTF32 split operands on tcgen05 (W^T split fits in shared memory), else CUDA-core FFMA
void gemm_xw_fp32(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y, const float* bias,
                  int32_t relu, cudaStream_t s);
// transpose.cu
void transpose_csr(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t n_cols, int64_t nnz,
                   int32_t* rowptr_t, int32_t* colidx_t, int32_t* src, cudaStream_t s);
void gather_vals(const float* vals, const int32_t* src, int64_t nnz, float* out, cudaStream_t s);
int num_sms();
}  // namespace agcn
