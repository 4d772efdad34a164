// plan.cu -- agcn_plan: the preprocessing of Accel-GCN section III-C on the device.
//
//  (1) degree of every row from the row pointer                       P:295 step (1)
//  (2) stable counting sort of the rows by degree, ascending           P:295 step (2)
//      - buckets 0..deg_bound exact, one bucket for degree > deg_bound;
//        per-tile histograms -> one exclusive scan (bucket-major) -> stable scatter
//      - the (few) oversized rows are then stably LSD-radix sorted by degree
//  (3) row-pointer / column-index update in the new order              P:295 step (3)
//  (4) Algorithm 1 patterns (closed form per degree)
//  (5) Algorithm 2 block descriptors, emitted in parallel in closed form per degree
//      bucket (equal to the sequential cursor walk), int4 {deg, loc, row, info}
//                                                                      P:335-382
// and, for the ablation arm, the warp-level partition of Fig. 3(b)    P:417.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"
#include "scan_lb.cuh"

namespace agcn {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSubTile = 256;                 // rows per warp per tile
constexpr int kTile = kWarps * kSubTile;      // rows per CTA tile
constexpr int kMaxDegBound = 2048;


__device__ __forceinline__ int32_t row_key(const int32_t* rowptr, int64_t i, int32_t db) {
    int32_t d = rowptr[i + 1] - rowptr[i];
    return d <= 0 ? 0 : (d <= db ? d : db + 1);
}

// ---------------------------------------------------------------- (1)+(2) histogram
// rp_copy (optional): the plan's scratch copy of rowptr, written on the way (every later plan
// kernel reads the copy, so nothing reads the caller's rowptr after agcn_plan returns)
__global__ void __launch_bounds__(kThreads) k_deg_hist(const int32_t* __restrict__ rowptr, int64_t n,
                                                      int32_t db, int32_t nbins, int64_t ntiles,
                                                      int32_t* __restrict__ table,
                                                      PlanFlags* __restrict__ flags,
                                                      int32_t* __restrict__ rp_copy) {
    extern __shared__ int32_t hist[];
    for (int b = threadIdx.x; b < nbins; b += kThreads) hist[b] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * kTile, hi = min(n, lo + kTile);
    int32_t maxd = 0, bad = 0;
    long long ovc = 0, ovh = 0;
    int32_t nhv = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
        const int32_t r0 = rowptr[i];
        int32_t d = rowptr[i + 1] - r0;
        if (rp_copy) rp_copy[i] = r0;
        if (d < 0) bad = 1;
        int32_t key = d <= 0 ? 0 : (d <= db ? d : db + 1);
        // power-law degrees: most lanes of a warp share a few keys (C5: 54 % degree 0) ->
        // one shared-memory atomic per distinct key per warp
        const unsigned act = __activemask();
        const unsigned same = __match_any_sync(act, key);
        if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&hist[key], __popc(same));
        maxd = max(maxd, d);
        if (d > db) ovc += (d + db - 1) / db;
        if (d > db && d >= kColBlockMinDeg) ovh += (d + db - 1) / db;
        if ((int64_t)d > (int64_t)kHeavyChunks * db) ++nhv;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        maxd = max(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        ovc += __shfl_xor_sync(0xffffffffu, ovc, o);
        ovh += __shfl_xor_sync(0xffffffffu, ovh, o);
        nhv += __shfl_xor_sync(0xffffffffu, nhv, o);
    }
    // per-CTA totals first: one set of global atomics per CTA, not per warp (C5: 4096 CTAs x 8
    // warps on the same few addresses serialised the kernel)
    __shared__ long long s_ov[2][kWarps];
    __shared__ int32_t s_i[3][kWarps];
    const int wi = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_ov[0][wi] = ovc;
        s_ov[1][wi] = ovh;
        s_i[0][wi] = maxd;
        s_i[1][wi] = bad;
        s_i[2][wi] = nhv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kWarps; ++k) {
            ovc += s_ov[0][k];
            ovh += s_ov[1][k];
            maxd = max(maxd, s_i[0][k]);
            bad |= s_i[1][k];
            nhv += s_i[2][k];
        }
        if (maxd) atomicMax(&flags->max_deg, maxd);
        if (bad) flags->bad_rowptr = 1;
        if (ovc) atomicAdd((unsigned long long*)&flags->ov_chunks, (unsigned long long)ovc);
        if (ovh) atomicAdd((unsigned long long*)&flags->ov_chunks_heavy, (unsigned long long)ovh);
        if (nhv) atomicAdd(&flags->n_ov_heavy, nhv);
        if (blockIdx.x == 0) {
            flags->rowptr_first = rowptr[0];
            flags->rowptr_last = rowptr[n];
            if (rp_copy) rp_copy[n] = rowptr[n];
        }
    }
    for (int b = threadIdx.x; b < nbins; b += kThreads) table[(int64_t)b * ntiles + blockIdx.x] = hist[b];
}

// Bucket totals from the exclusive-scanned (bucket-major) tile table.
__global__ void k_bin_totals(const int32_t* __restrict__ table, int64_t ntiles, int32_t nbins, int64_t n,
                             int32_t* __restrict__ bin_cnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nbins) {
        const int64_t hi = b + 1 < nbins ? table[(int64_t)(b + 1) * ntiles] : n;
        bin_cnt[b] = (int32_t)(hi - table[(int64_t)b * ntiles]);
    }
}

// ---------------------------------------------------------------- stable bucket scatter
// One CTA per tile of kTile items; warp w owns items [tile*kTile + w*kSubTile, +kSubTile).
// table_off (bucket-major, exclusive-scanned) gives the first output slot of (bucket, tile).
// Within a tile, ranks follow item order: warp sub-tiles in order, 32-item chunks in order,
// lanes in order (__match_any_sync groups equal keys) -> the scatter is stable.
struct MainSrc {
    const int32_t* rowptr;
    int32_t db;
    int32_t* perm;
    __device__ __forceinline__ int32_t key(int64_t i) const { return row_key(rowptr, i, db); }
    __device__ __forceinline__ void emit(int64_t pos, int64_t i) const { perm[pos] = (int32_t)i; }
};
struct RadixSrc {
    const int32_t* keys_in;
    const int32_t* vals_in;
    int32_t* keys_out;
    int32_t* vals_out;
    int32_t shift;
    __device__ __forceinline__ int32_t key(int64_t i) const { return (keys_in[i] >> shift) & 255; }
    __device__ __forceinline__ void emit(int64_t pos, int64_t i) const {
        keys_out[pos] = keys_in[i];
        vals_out[pos] = vals_in[i];
    }
};

template <class Src>
__global__ void __launch_bounds__(kThreads) k_bucket_hist(Src src, int64_t m, int32_t nbins,
                                                         int64_t ntiles, int32_t* __restrict__ table) {
    extern __shared__ int32_t hist[];
    for (int b = threadIdx.x; b < nbins; b += kThreads) hist[b] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * kTile, hi = min(m, lo + kTile);
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) atomicAdd(&hist[src.key(i)], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += kThreads)
        table[(int64_t)b * ntiles + blockIdx.x] = hist[b];
}

template <class Src>
__global__ void __launch_bounds__(kThreads) k_bucket_scatter(Src src, int64_t m, int32_t nbins,
                                                            int64_t ntiles,
                                                            const int32_t* __restrict__ table_off) {
    extern __shared__ int32_t h[];  // [kWarps][nbins]
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < kWarps * nbins; b += kThreads) h[b] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * kTile + (int64_t)w * kSubTile;
    const int64_t hi = min(m, lo + kSubTile);
    int32_t* hw = h + w * nbins;
    for (int64_t i = lo + lane; i < hi; i += 32) atomicAdd(&hw[src.key(i)], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += kThreads) {
        int32_t run = table_off[(int64_t)b * ntiles + blockIdx.x];
        for (int ww = 0; ww < kWarps; ++ww) {
            int32_t c = h[ww * nbins + b];
            h[ww * nbins + b] = run;
            run += c;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t c0 = lo; c0 < hi; c0 += 32) {
        const int64_t i = c0 + lane;
        const bool valid = i < hi;
        const int32_t k = valid ? src.key(i) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, k);
        int32_t base = 0;
        if (valid) {
            base = hw[k];
            src.emit((int64_t)base + __popc(peers & lt), i);
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) hw[k] = base + __popc(peers);
        __syncwarp();
    }
}

__global__ void k_ov_init(const int32_t* __restrict__ perm_ov, const int32_t* __restrict__ rowptr,
                          int64_t m, int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) {
        int32_t r = perm_ov[k];
        keys[k] = rowptr[r + 1] - rowptr[r];
        vals[k] = r;
    }
}

// ---------------------------------------------------------------- (3) sorted CSR
// Element k of the sorted-rowptr scan: the degree of sorted row k; on the way, where that row
// starts in the caller's arrays (row_src_off).  The scan (scan_lb.cuh) turns the sorted degrees
// into sorted_rowptr in the same pass.
struct SortedRowsSrc {
    const int32_t* perm;
    const int32_t* rowptr;
    int32_t* rso;
    __device__ __forceinline__ int32_t get(int64_t k) const {
        const int32_t r = __ldg(perm + k);
        const int32_t a = __ldg(rowptr + r);
        rso[k] = a - __ldg(rowptr);
        return __ldg(rowptr + r + 1) - a;
    }
};

// Bucket tables for degrees 1..db (index db+1 = end sentinel), in shared memory.
struct BinTables {
    const int32_t* nnz_start;  // first sorted nnz of bucket d
    const int32_t* row_start;  // first sorted row of bucket d
    const int32_t* blk_start;  // first descriptor of bucket d
    const int32_t* cnt;        // rows of degree d
    const int32_t* br;         // Alg. 1 block_rows of d
    const int32_t* wn;         // Alg. 1 warp_nzs of d
};

// last d in [1, db] with a[d] <= v  (a non-decreasing on 1..db+1)
__device__ __forceinline__ int32_t bin_search(const int32_t* a, int32_t db, int32_t v) {
    int32_t lo = 1, hi = db + 1;  // upper_bound over [1, db+1)
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo - 1;
}

// The plan's copy of colidx (the caller may free its arrays after agcn_plan),
// in the caller's order -- the SpMM reads a sorted row's column indices and vals at the same
// offsets (row_src_off, P:295 step (3)) -- made in one flat, coalesced pass: 4 entries per
// thread in flight.  On the way: the colidx range check (flags != NULL), the padded-layout
// relabel (ColMap, multi-GPU) or the hot-column encoding c -> -1 - slot, slot = rank of c among
// the hot columns, from one 8-byte entry {bitmap word, exclusive popcount prefix} per 32
// columns (n_cols / 4 bytes, L2-resident).  Out-of-range columns are copied unchanged (the plan
// is rejected by the flags before use; with validation off the caller guarantees the range).
__device__ __forceinline__ int32_t encode_col(int32_t c, int64_t n_cols, const ColMap& cm,
                                              const uint2* __restrict__ hot) {
    if (cm.nparts > 0) return map_col(c, cm);
    if (hot && c >= 0 && (int64_t)c < n_cols) {
        const uint2 w = __ldg(hot + (c >> 5));
        const uint32_t bit = 1u << (c & 31);
        if (w.x & bit) return -1 - (int32_t)(w.y + __popc(w.x & (bit - 1)));
    }
    return c;
}

// cols: the caller's colidx array when rp != NULL (the run [rp[0], rp[n]) is copied, read on the
// device; an inconsistent rowptr -- rp[n] - rp[0] != nnz, reported by the plan's flags -- copies
// nothing), else an array of nnz entries re-encoded in place (out == cols).
__global__ void k_copy_cols_enc(const int32_t* cols, const int32_t* __restrict__ rp, int64_t n, int64_t nnz,
                                int64_t n_cols, ColMap cm, const uint2* __restrict__ hot, int32_t* out,
                                PlanFlags* __restrict__ flags) {
    if (rp) {
        const int32_t base = __ldg(rp);
        if ((int64_t)__ldg(rp + n) - base != nnz) return;
        cols += base;
    }
    int32_t bad = 0;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < nnz; q0 += 4 * T) {
        int32_t c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = q0 + k * T < nnz ? __ldcs(cols + q0 + k * T) : 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (q0 + k * T < nnz) {
                bad |= (c[k] < 0) | ((int64_t)c[k] >= n_cols);
                __stcs(out + q0 + k * T, encode_col(c[k], n_cols, cm, hot));
            }
        }
    }
    if (flags && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flags->bad_colidx = 1;
}

// hot vertices: the H highest-degree ones (sorted positions n - H .. n - 1) -> column bitmap
// (hot[w].x), then per-word popcounts (hot[w].y) turned into exclusive prefixes by a scan
__global__ void k_hot_bits(const int32_t* __restrict__ perm, int64_t n, int64_t H, uint2* __restrict__ hot) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < H) {
        const int32_t c = perm[n - 1 - k];
        atomicOr(&hot[c >> 5].x, 1u << (c & 31));
    }
}
__global__ void k_popc_words(const uint2* __restrict__ hot, int64_t nw, int32_t* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nw) cnt[i] = __popc(hot[i].x);
}
// hot[w].y = prefix[w]; hot_cols[slot] = column of hot slot `slot` (slots in column order)
__global__ void k_hot_list(uint2* __restrict__ hot, const int32_t* __restrict__ pre, int64_t nw,
                           int32_t* __restrict__ hot_cols) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nw) return;
    uint32_t w = hot[i].x;
    int32_t k = pre[i];
    hot[i].y = (uint32_t)k;
    while (w) {
        const int b = __ffs(w) - 1;
        hot_cols[k++] = (int32_t)(i * 32 + b);
        w &= w - 1;
    }
}

// The same hot set from the degree histogram alone, so the colidx copy can run before the degree
// order exists (while the host reads the bucket counts back): the H largest (degree, row) keys
// of the stable ascending order are every row of degree > tau and the degree-tau rows of rank
// >= first among them in row order.  One warp: lane l walks its chunk of degrees from the top
// with the count of all rows above it; the highest lane that reaches H holds tau.  When more
// than H rows exceed deg_bound (the histogram does not resolve their degrees) the plan takes
// the tail of the sorted order instead (hot_fallback).
__global__ void k_hot_tau(const int32_t* __restrict__ bin_cnt, int32_t db, int64_t n, int64_t Hreq,
                          PlanFlags* __restrict__ f) {
    const int lane = threadIdx.x & 31;
    const int64_t live = n - bin_cnt[0];
    const int64_t H = Hreq < live ? Hreq : live;
    const int64_t over = bin_cnt[db + 1];
    const int32_t chunk = (db + 31) / 32;
    const int32_t lo = 1 + lane * chunk, hi = min(db + 1, lo + chunk);   // degrees [lo, hi)
    int64_t mine = 0;
    for (int32_t d = lo; d < hi; ++d) mine += bin_cnt[d];
    int64_t above = mine;                                   // rows in chunks >= this lane's
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_down_sync(0xffffffffu, above, o);
        if (lane + o < 32) above += t;
    }
    above = above - mine + over;                            // rows of degree >= hi
    int32_t tau = 0, first = 0;
    bool hit = false;
    if (H > 0 && over <= H) {
        for (int32_t d = hi - 1; d >= lo; --d) {
            if (above + bin_cnt[d] >= H) {
                tau = d;
                first = (int32_t)(bin_cnt[d] - (H - above));
                hit = true;
                break;
            }
            above += bin_cnt[d];
        }
    }
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) {
        f->hot_tau = 0x7fffffff;
        f->hot_first = 0;
        f->hot_fallback = H > 0 && over > H;
        f->n_hot = 0;
    }
    __syncwarp();
    if (b && lane == 31 - __clz(b)) {
        f->hot_tau = tau;
        f->hot_first = first;
        f->n_hot = H;
    }
}
// Pass A, one warp per 32 rows = one bitmap word: ballots of degree > tau and degree == tau, the
// latter's popcount per word (scanned into ranks).  rp: the plan's rowptr copy.
__global__ void k_hot_deg_a(const int32_t* __restrict__ rp, int64_t n, const PlanFlags* __restrict__ f,
                            uint2* __restrict__ hot, uint32_t* __restrict__ eqw, int32_t* __restrict__ eqc) {
    const int32_t tau = f->hot_tau;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t d = i < n ? rp[i + 1] - rp[i] : -1;
    const uint32_t gt = __ballot_sync(0xffffffffu, d > tau), eq = __ballot_sync(0xffffffffu, d == tau);
    if ((threadIdx.x & 31) == 0 && i < n) {
        hot[i >> 5] = make_uint2(gt, 0u);
        eqw[i >> 5] = eq;
        eqc[i >> 5] = __popc(eq);
    }
}
// Pass B: the degree-tau rows of rank >= first join; cnt[w] = popcount of the final word
__global__ void k_hot_deg_b(uint2* __restrict__ hot, const uint32_t* __restrict__ eqw,
                            const int32_t* __restrict__ eqpre, int64_t nw, const PlanFlags* __restrict__ f,
                            int32_t* __restrict__ cnt) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int32_t first = f->hot_first;
    uint32_t e = eqw[w], bits = hot[w].x;
    int32_t r = eqpre[w];
    while (e) {
        const uint32_t b = e & (0u - e);
        if (r >= first) bits |= b;
        ++r;
        e ^= b;
    }
    hot[w].x = bits;
    cnt[w] = __popc(bits);
}

// Execution order of the oversized-row chunks (kernel-internal; the descriptors keep Alg. 2's
// order): chunk j of a row of nc chunks covers the j-th run of the row's columns, which lie
// around fraction (j + 0.5) / nc of the column range when the row's columns are sorted and
// spread over it; executing the chunks bucketed by that fraction lets concurrently running
// warps gather from the same part of X, so X rows are reused across hub rows in L2 (P:491,
// "improving cache hit rate").  key = bucket in [0, kOvBuckets), stable sort by key.
constexpr int kOvBuckets = 64;
__global__ void k_ov_keys(const int4* __restrict__ desc, int64_t nb_small, int64_t nch, int32_t db, int32_t nbk,
                          const int32_t* __restrict__ srp, int32_t* __restrict__ key, int32_t* __restrict__ idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nch) return;
    const int4 m = desc[nb_small + i];
    const int32_t j = (m.y - srp[m.z]) / db, nc = (m.x + db - 1) / db;
    key[i] = (int32_t)min((int64_t)nbk - 1, ((2 * (int64_t)j + 1) * nbk) / (2 * (int64_t)nc));
    idx[i] = (int32_t)i;
}

// Introspection (agcn_plan_copy(AGCN_FIELD_SORTED_COLIDX)): the colidx of the degree-sorted
// CSR, gathered on demand from the plan's copy (one warp per sorted row), hot encoding undone.
__global__ void k_gather_sorted_cols(int64_t n, const int32_t* __restrict__ sorted_rowptr,
                                     const int32_t* __restrict__ rso, const int32_t* __restrict__ cols,
                                     const int32_t* __restrict__ hot_cols, int32_t* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (k >= n) return;
    const int32_t dst = sorted_rowptr[k], d = sorted_rowptr[k + 1] - dst, src = rso[k];
    for (int32_t j = threadIdx.x & 31; j < d; j += 32) {
        const int32_t c = cols[src + j];
        out[dst + j] = c >= 0 ? c : hot_cols[-1 - c];
    }
}

// ---------------------------------------------------------------- (5) Algorithm 2 emission
// Descriptor b of the degree<=db part: bucket d = last d with blk_start[d] <= b; block i of
// bucket d covers rows row_start[d] + i*br .. and nnz nnz_start[d] + i*br*d ..; the residual
// block carries rows = cnt[d] - i*br (< br).  info = warp_nzs << 16 | rows.
__global__ void __launch_bounds__(kThreads) k_emit_small(int64_t nb_small, int32_t db,
                                                        const int32_t* __restrict__ g_tab,
                                                        int4* __restrict__ desc) {
    extern __shared__ int32_t sm[];
    const int32_t W = db + 2;
    for (int t = threadIdx.x; t < 6 * W; t += kThreads) sm[t] = g_tab[t];
    __syncthreads();
    const int32_t* nnz_start = sm;
    const int32_t* row_start = sm + W;
    const int32_t* blk_start = sm + 2 * W;
    const int32_t* cnt = sm + 3 * W;
    const int32_t* br = sm + 4 * W;
    const int32_t* wn = sm + 5 * W;
    for (int64_t b = (int64_t)blockIdx.x * kThreads + threadIdx.x; b < nb_small;
         b += (int64_t)gridDim.x * kThreads) {
        int32_t d = bin_search(blk_start, db, (int32_t)b);
        int32_t i = (int32_t)b - blk_start[d];
        int32_t rows = min(br[d], cnt[d] - i * br[d]);
        desc[b] = make_int4(d, nnz_start[d] + i * br[d] * d, row_start[d] + i * br[d],
                            (int32_t)(((uint32_t)wn[d] << 16) | (uint32_t)rows));
    }
}

__global__ void k_ov_chunk_count(const int32_t* __restrict__ sorted_rowptr, int64_t ov_start,
                                 int64_t n_ov, int32_t db, int32_t* __restrict__ out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n_ov) {
        int32_t d = sorted_rowptr[ov_start + k + 1] - sorted_rowptr[ov_start + k];
        out[k] = (d + db - 1) / db;
    }
}

// Oversized row k (sorted position ov_start + k): chunk j = {deg, loc + j*db, row, min(db, deg - j*db)}
__global__ void k_emit_ov(const int32_t* __restrict__ sorted_rowptr, int64_t ov_start, int64_t n_ov,
                          int32_t db, int64_t nb_small, const int32_t* __restrict__ chunk_start,
                          int4* __restrict__ desc) {
    const int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (k >= n_ov) return;
    const int32_t row = (int32_t)(ov_start + k);
    const int32_t loc = sorted_rowptr[row], d = sorted_rowptr[row + 1] - loc;
    const int32_t c0 = chunk_start[k], nc = chunk_start[k + 1] - c0;
    for (int32_t j = threadIdx.x & 31; j < nc; j += 32)
        desc[nb_small + c0 + j] = make_int4(d, loc + j * db, row, min(db, d - j * db));
}

// ---------------------------------------------------------------- warp-level partition
__global__ void k_rowptr_check(const int32_t* __restrict__ rowptr, int64_t n, int32_t mwn,
                               int32_t* __restrict__ rp_copy, int32_t* __restrict__ ntask,
                               PlanFlags* __restrict__ flags) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        int32_t d = rowptr[i + 1] - rowptr[i];
        if (d < 0) flags->bad_rowptr = 1;
        rp_copy[i] = rowptr[i] - rowptr[0];
        ntask[i] = d > 0 ? (d + mwn - 1) / mwn : 0;
        atomicMax(&flags->max_deg, max(d, 0));
    }
    if (i == 0) {
        flags->rowptr_first = rowptr[0];
        flags->rowptr_last = rowptr[n];
        rp_copy[n] = rowptr[n] - rowptr[0];
    }
}

__global__ void k_emit_tasks(const int32_t* __restrict__ rp, int64_t n, int32_t mwn,
                             const int32_t* __restrict__ tstart, int4* __restrict__ tasks) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t d = rp[i + 1] - rp[i];
    int32_t t = tstart[i];
    for (int32_t c = 0; c < d; c += mwn) tasks[t++] = make_int4((int32_t)i, c, min(mwn, d - c), 0);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// Library-side Algorithm 1 in closed form: smallest factor f of mbw with f*mwn >= d,
// block_rows = mbw / f, warp_nzs = ceil(d / f).
void host_patterns(int32_t mbw, int32_t mwn, std::vector<int32_t>& br, std::vector<int32_t>& wn) {
    const int32_t db = mbw * mwn;
    br.assign(db + 2, 0);
    wn.assign(db + 2, 0);
    for (int32_t d = 1; d <= db; ++d) {
        int32_t f = 1;
        while (!(mbw % f == 0 && (int64_t)f * mwn >= d)) ++f;
        br[d] = mbw / f;
        wn[d] = (d + f - 1) / f;
    }
}

}  // namespace

ColMap make_colmap(const agcn_opts_t& o, int64_t n_cols) {
    ColMap cm{};
    cm.n_cols = n_cols;
    cm.nparts = o.col_nparts;
    cm.slot_rows = (int32_t)o.col_slot_rows;
    if (o.col_nparts > 0) {
        AGCN_CHECK(o.col_nparts <= kMaxColParts && o.col_bounds != nullptr,
                   AGCN_ERR_INVALID_ARG, "col_nparts > 64 or col_bounds == NULL");
        AGCN_CHECK(o.col_slot_rows > 0 && (int64_t)o.col_nparts * o.col_slot_rows < (1ll << 31),
                   AGCN_ERR_INVALID_ARG, "bad col_slot_rows");
        AGCN_CHECK(o.col_bounds[0] == 0 && o.col_bounds[o.col_nparts] == n_cols, AGCN_ERR_INVALID_ARG,
                   "col_bounds must span [0, n_cols]");
        for (int p = 0; p <= o.col_nparts; ++p) cm.bounds[p] = o.col_bounds[p];
        for (int p = 0; p < o.col_nparts; ++p)
            AGCN_CHECK(o.col_bounds[p + 1] >= o.col_bounds[p] &&
                           o.col_bounds[p + 1] - o.col_bounds[p] <= o.col_slot_rows,
                       AGCN_ERR_INVALID_ARG, "col_bounds not monotone or slot too small");
    }
    return cm;
}

namespace {

// Pinned host staging for the plan's readbacks (a pageable destination makes the driver bounce
// the copy through its own pinned buffer); one per host thread, grown on demand.
void* pinned_staging(size_t bytes) {
    thread_local void* buf = nullptr;
    thread_local size_t cap = 0;
    if (bytes > cap) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        if (cudaMallocHost(&buf, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        cap = bytes;
    }
    return buf;
}

void read_flags(PlanFlags* d_flags, PlanFlags* h, cudaStream_t s) {
    AGCN_CUDA(cudaMemcpyAsync(h, d_flags, sizeof(PlanFlags), cudaMemcpyDeviceToHost, s));
    AGCN_CUDA(cudaStreamSynchronize(s));
}

void check_csr_flags(const PlanFlags& f, int64_t nnz) {
    AGCN_CHECK(!f.bad_rowptr, AGCN_ERR_BAD_CSR, "rowptr is not non-decreasing");
    AGCN_CHECK((int64_t)f.rowptr_last - f.rowptr_first == nnz, AGCN_ERR_BAD_CSR,
               "rowptr[n] - rowptr[0] != nnz");
}

// The plan's copy of colidx (k_copy_cols_enc, flat, 4 entries per thread in flight): rp is a
// DEVICE rowptr (the caller's or the plan's copy; the run [rp[0], rp[n]) is copied) or NULL to
// re-encode p->cols_copy in place.  hot: the hot-column table or NULL; d_flags != NULL:
// validate the column range on the way.
void launch_copy_cols(agcn_plan_s* p, const int32_t* cols, const int32_t* rp, const uint2* hot,
                      PlanFlags* d_flags, cudaStream_t s) {
    if (p->nnz == 0) return;
    const unsigned g = (unsigned)std::min<int64_t>(blocks_for(p->nnz, 256 * 4), (int64_t)num_sms() * 8);
    k_copy_cols_enc<<<g, 256, 0, s>>>(cols, rp, p->n, p->nnz, p->n_cols, p->cmap, hot, p->cols_copy, d_flags);
    post_launch();
}

// Hot rows requested (agcn_opts_t.hot_rows) before the degrees are known: square A without a
// padded layout only; -1: 524288 for graphs of >= 2^19 rows (C5 sweep: profiles/r02af).
int64_t hot_rows_req(const agcn_plan_s* p, int64_t req) {
    if (p->n_cols != p->n || p->cmap.nparts > 0 || req == 0) return 0;
    const int64_t H = req > 0 ? req : (p->n >= (1ll << 19) ? 524288 : 0);
    return std::min(H, p->n);
}

// Hot rows of a plan (agcn_opts_t.hot_rows): square A without a padded layout only.
// ... capped at the rows of degree >= 1 (n_zero known)
int64_t hot_rows_for(const agcn_plan_s* p, int64_t req) {
    return std::max<int64_t>(0, std::min(hot_rows_req(p, req), p->n - p->n_zero));
}

// BLOCK plan, after the descriptors: the execution order of the oversized chunks (k_ov_keys).
void build_ov_order(agcn_plan_s* p, int32_t buckets, cudaStream_t s) {
    const int64_t m = p->ov_chunks;
    const int32_t nbk = buckets > 0 ? buckets : kOvBuckets;
    if (m <= 1) return;
    Scratch tmp(s);
    int32_t* ka = tmp.alloc<int32_t>(m);
    int32_t* va = tmp.alloc<int32_t>(m);
    int32_t* kb = tmp.alloc<int32_t>(m);
    int32_t* vb = tmp.alloc<int32_t>(m);
    k_ov_keys<<<blocks_for(m, 256), 256, 0, s>>>(p->desc, p->nb_small, m, p->deg_bound, nbk, p->sorted_rowptr,
                                                  ka, va);
    post_launch();
    radix_sort_pairs(ka, va, kb, vb, m, nbk - 1, s);
    p->ov_order = dalloc<int32_t>(m, s);
    p->device_bytes += sizeof(int32_t) * (size_t)m;
    AGCN_CUDA(cudaMemcpyAsync(p->ov_order, va, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, s));
}

// BLOCK plan, after the degree order, when the hot set could not be taken from the histogram
// (k_hot_tau: more than H oversized rows; or the one-CTA plan): the hot_rows highest-degree
// vertices = the tail of the degree order -> bitmap + prefixes -> hot_cols, then the plan's
// colidx copy (already made) re-encoded in place.
void encode_hot_from_tail(agcn_plan_s* p, int64_t H, cudaStream_t s) {
    p->n_hot = H;
    if (H <= 0 || p->nnz == 0) return;
    Scratch tmp(s);
    const int64_t nw = (p->n_cols + 31) / 32;
    uint2* hot = tmp.alloc<uint2>(nw);
    int32_t* pre = tmp.alloc<int32_t>(nw + 1);
    if (!p->hot_cols) {
        p->hot_cols = dalloc<int32_t>(H, s);
        p->device_bytes += sizeof(int32_t) * (size_t)H;
    }
    AGCN_CUDA(cudaMemsetAsync(hot, 0, sizeof(uint2) * nw, s));
    k_hot_bits<<<blocks_for(H, 256), 256, 0, s>>>(p->perm, p->n, H, hot);
    post_launch();
    k_popc_words<<<blocks_for(nw, 256), 256, 0, s>>>(hot, nw, pre);
    post_launch();
    exclusive_scan_i32(pre, pre, nw, s);
    k_hot_list<<<blocks_for(nw, 256), 256, 0, s>>>(hot, pre, nw, p->hot_cols);
    post_launch();
    launch_copy_cols(p, p->cols_copy, nullptr, hot, nullptr, s);
}

}  // namespace

// Stable LSD radix sort of (key, val) int32 pairs by key (0 <= key <= max_key), 8-bit digits,
// through the stable bucket scatter above.  ka/va in, kb/vb scratch; on return ka/va point at
// the sorted pairs (either buffer pair).
void radix_sort_pairs(int32_t*& ka, int32_t*& va, int32_t*& kb, int32_t*& vb, int64_t m, int64_t max_key,
                      cudaStream_t s) {
    if (m <= 1) return;
    int passes = 0;
    for (int64_t v = max_key; v > 0; v >>= 8) ++passes;
    const int64_t mt = (m + kTile - 1) / kTile;
    AGCN_CHECK(256 * mt < (1ll << 31), AGCN_ERR_OVERFLOW, "radix sort too large");
    Scratch tmp(s);
    int32_t* rt = tmp.alloc<int32_t>(256 * mt + 1);
    for (int pass = 0; pass < passes; ++pass) {
        RadixSrc src{ka, va, kb, vb, 8 * pass};
        k_bucket_hist<RadixSrc><<<(unsigned)mt, kThreads, 256 * sizeof(int32_t), s>>>(src, m, 256, mt, rt);
        post_launch();
        exclusive_scan_i32(rt, rt, 256 * mt, s);
        k_bucket_scatter<RadixSrc><<<(unsigned)mt, kThreads, kWarps * 256 * sizeof(int32_t), s>>>(src, m, 256, mt, rt);
        post_launch();
        std::swap(ka, kb);
        std::swap(va, vb);
    }
}

namespace {

// ---------------------------------------------------------------- small graphs: one CTA
// For n <= kSmallRows the whole block plan (steps (1)-(5) above, the same algorithm and the
// same stable order) runs in ONE 1024-thread CTA with one host synchronisation at the end:
// C1 / C2-sized graphs are bound by launch and synchronisation latency (~20 launches +
// allocations + a mid-course readback in the general path), not by work.  Warp w owns rows
// [w R, (w+1) R); the stable counting sort is per-warp histograms -> (bin, warp) offsets ->
// match_any ranks, exactly the tile scheme of k_bucket_scatter with one tile.  Oversized rows
// (at most kSmallOv) are ranked by (degree, row) directly.  If there are more, the kernel
// reports it before writing anything and the general path runs instead.
constexpr int64_t kSmallRows = 32768;
constexpr int64_t kSmallNnz = 1 << 20;
constexpr int32_t kSmallDb = 512;
constexpr int32_t kSmallOv = 1024;
constexpr int kSmallThreads = 1024;

struct SmallOut {
    int32_t fallback, bad_rowptr, bad_colidx, max_deg;
    int32_t rowptr_first, rowptr_last, n_ov_heavy, pad;
    int64_t nb_small, n_zero, n_ov, ov_chunks, ov_chunks_heavy;
};

// exclusive scan of v over the block (1024 threads); returns the prefix, *total the sum
__device__ __forceinline__ int64_t block_exscan(int64_t v, int64_t* wsum, int64_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        wsum[32 + lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = (w ? wsum[32 + w - 1] : 0) + x - v;
    *total = wsum[32 + 31];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(kSmallThreads, 1)
k_plan_small(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx_g, int64_t n, int64_t nnz,
             int64_t n_cols, int32_t db, int32_t mbw, int32_t mwn, int32_t validate, int32_t* __restrict__ perm,
             int32_t* __restrict__ srp, int32_t* __restrict__ rso, int4* __restrict__ desc,
             int32_t* __restrict__ ov_chunk_start, SmallOut* __restrict__ out) {
    extern __shared__ int32_t sm[];
    const int32_t nbins = db + 2;
    int32_t* wh = sm;                                    // [32][nbins]: counts, then offsets
    int32_t* tot = wh + 32 * nbins;                      // [nbins]
    int32_t* blk = tot + nbins;                          // [db + 2] first descriptor of degree d
    int32_t* ovd = blk + db + 2;                         // [kSmallOv]
    int32_t* ovr = ovd + kSmallOv;                       // [kSmallOv]
    int32_t* rs = ovr + kSmallOv;                        // [nbins] first sorted row of bucket b
    int64_t* wsum = reinterpret_cast<int64_t*>(sm + ((33 * nbins + db + 2 + 2 * kSmallOv + nbins + 1) & ~1));  // [64]
    int16_t* keys = reinterpret_cast<int16_t*>(wsum + 64);  // [n] bucket of every row
    __shared__ int32_t s_max, s_bad, s_badc, s_nhv;
    __shared__ unsigned long long s_ovc, s_ovh;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < 32 * nbins; i += kSmallThreads) wh[i] = 0;
    if (tid == 0) { s_max = 0; s_bad = 0; s_badc = 0; s_nhv = 0; s_ovc = 0; s_ovh = 0; }
    __syncthreads();
    const int32_t base = rowptr[0];
    const int64_t R = (n + 31) / 32, lo = w * R, hi = min(n, lo + R);
    int32_t* hw = wh + w * nbins;
    // (1) degrees -> bucket keys in shared memory (independent coalesced loads) + flags
    int32_t maxd = 0, bad = 0, nhv = 0;
    long long ovc = 0, ovh = 0;
#pragma unroll 4
    for (int64_t i = tid; i < n; i += kSmallThreads) {
        const int32_t d = rowptr[i + 1] - rowptr[i];
        keys[i] = (int16_t)(d <= 0 ? 0 : (d <= db ? d : db + 1));
        bad |= d < 0;
        maxd = max(maxd, d);
        if (d > db) ovc += (d + db - 1) / db;
        if (d > db && d >= kColBlockMinDeg) ovh += (d + db - 1) / db;
        if ((int64_t)d > (int64_t)kHeavyChunks * db) ++nhv;
    }
    __syncthreads();
    // (2a) per-warp bucket counts over the warp's row range
    for (int64_t c0 = lo; c0 < hi; c0 += 32) {
        const int64_t i = c0 + lane;
        const bool valid = i < hi;
        const int32_t key = valid ? keys[i] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        if (valid && lane == __ffs(peers) - 1) hw[key] += __popc(peers);
        __syncwarp();
    }
    int32_t badc = 0;
    if (validate) {
        const int32_t* colidx = colidx_g + base;
#pragma unroll 8
        for (int64_t q = tid; q < nnz; q += kSmallThreads) {
            const int32_t j = colidx[q];
            badc |= (j < 0) | ((int64_t)j >= n_cols);
        }
    }
    if (maxd) atomicMax(&s_max, maxd);
    if (bad) s_bad = 1;
    if (badc) s_badc = 1;
    if (nhv) atomicAdd(&s_nhv, nhv);
    if (ovc) atomicAdd(&s_ovc, (unsigned long long)ovc);
    if (ovh) atomicAdd(&s_ovh, (unsigned long long)ovh);
    __syncthreads();
    // an invalid rowptr (decreasing, or rowptr[n] - rowptr[0] != nnz) would size the descriptor
    // array wrongly (it has room for n + nnz / db + kSmallOv + 1 entries): report before any
    // global write (the host turns the flags into AGCN_ERR_BAD_CSR)
    if (s_bad || (int64_t)rowptr[n] - base != nnz) {
        if (tid == 0) {
            out->fallback = 0;
            out->bad_rowptr = s_bad;
            out->rowptr_first = base;
            out->rowptr_last = rowptr[n];
        }
        return;
    }
    // (2b) bucket totals, bucket starts, (bin, warp) offsets in item order
    for (int b = tid; b < nbins; b += kSmallThreads) {
        int32_t t = 0;
        for (int ww = 0; ww < 32; ++ww) t += wh[ww * nbins + b];
        tot[b] = t;
    }
    __syncthreads();
    {
        // nbins <= 514 < 1024: one bin per thread
        const int64_t v = tid < nbins ? tot[tid] : 0;
        int64_t all;
        const int64_t start = block_exscan(v, wsum, &all);
        if (tid < nbins) {
            rs[tid] = (int32_t)start;
            int32_t run = (int32_t)start;
            for (int ww = 0; ww < 32; ++ww) {
                const int32_t c = wh[ww * nbins + tid];
                wh[ww * nbins + tid] = run;
                run += c;
            }
        }
    }
    const int64_t n_ov = tot[db + 1], n_zero = tot[0], ov_start = n - n_ov;
    if (n_ov > kSmallOv) {
        if (tid == 0) out->fallback = 1;
        return;
    }
    __syncthreads();
    // (2c) stable scatter
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t c0 = lo; c0 < hi; c0 += 32) {
        const int64_t i = c0 + lane;
        const bool valid = i < hi;
        const int32_t key = valid ? keys[i] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        int32_t b0 = 0;
        if (valid) {
            b0 = hw[key];
            perm[b0 + __popc(peers & lt)] = (int32_t)i;
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) hw[key] = b0 + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // (2d) oversized rows (kept in row order by the scatter): rank by (degree, row)
    if (tid < n_ov) {
        const int32_t r = perm[ov_start + tid];
        ovr[tid] = r;
        ovd[tid] = rowptr[r + 1] - rowptr[r];
    }
    __syncthreads();
    if (tid < n_ov) {
        const int32_t d = ovd[tid];
        int32_t rank = 0;
        for (int j = 0; j < (int)n_ov; ++j) rank += (ovd[j] < d) | ((ovd[j] == d) & (j < tid));
        perm[ov_start + rank] = ovr[tid];
    }
    __syncthreads();
    // (3) sorted degrees and row offsets (independent strided iterations), then the exclusive
    // scan -> sorted_rowptr (contiguous segment per thread)
#pragma unroll 4
    for (int64_t r = tid; r < n; r += kSmallThreads) {
        const int32_t i = perm[r];
        const int32_t a = rowptr[i];
        srp[r] = rowptr[i + 1] - a;
        rso[r] = a - base;
    }
    __syncthreads();
    const int64_t per = (n + kSmallThreads - 1) / kSmallThreads;
    const int64_t a0 = min(n, tid * per), a1 = min(n, a0 + per);
    int64_t sum = 0;
    for (int64_t r = a0; r < a1; ++r) sum += srp[r];
    {
        int64_t all;
        int64_t run = block_exscan(sum, wsum, &all);
        for (int64_t r = a0; r < a1; ++r) {
            const int32_t d = srp[r];
            srp[r] = (int32_t)run;
            run += d;
        }
        if (tid == 0) srp[n] = (int32_t)all;
    }
    __syncthreads();
    // (4) Alg. 1 per degree and the descriptor count of each bucket, scanned
    {
        const int32_t d = tid + 1;
        int64_t nb = 0;
        if (d <= db) {
            int32_t f = 1;
            while (!(mbw % f == 0 && (int64_t)f * mwn >= d)) ++f;
            const int32_t br = mbw / f;
            nb = (tot[d] + br - 1) / br;
        }
        int64_t all;
        const int64_t st = block_exscan(nb, wsum, &all);
        if (d <= db) blk[d] = (int32_t)st;
        if (tid == 0) blk[db + 1] = (int32_t)all;
    }
    __syncthreads();
    const int32_t nb_small = blk[db + 1];
    // (5) descriptors of the degree <= db part: descriptor b is block i of bucket d
    for (int32_t b = tid; b < nb_small; b += kSmallThreads) {
        int32_t lo_d = 1, hi_d = db + 1;  // last d in [1, db] with blk[d] <= b
        while (lo_d < hi_d) {
            const int32_t mid = (lo_d + hi_d) >> 1;
            if (blk[mid] <= b) lo_d = mid + 1; else hi_d = mid;
        }
        const int32_t d = lo_d - 1;
        int32_t f = 1;
        while (!(mbw % f == 0 && (int64_t)f * mwn >= d)) ++f;
        const int32_t br = mbw / f, wn = (d + f - 1) / f;
        const int32_t i = b - blk[d];
        const int32_t row = rs[d] + i * br;
        const int32_t rows = min(br, tot[d] - i * br);
        desc[b] = make_int4(d, srp[row], row, (int32_t)(((uint32_t)wn << 16) | (uint32_t)rows));
    }
    // oversized chunks: row k of the suffix -> ceil(d / db) chunks
    {
        int64_t nc = 0, loc = 0, d = 0;
        const int64_t row = ov_start + tid;
        if (tid < n_ov) {
            loc = srp[row];
            d = srp[row + 1] - loc;
            nc = (d + db - 1) / db;
        }
        int64_t all;
        const int64_t c0 = block_exscan(nc, wsum, &all);
        if (tid < n_ov) {
            ov_chunk_start[tid] = (int32_t)c0;
            for (int64_t j = 0; j < nc; ++j)
                desc[nb_small + c0 + j] = make_int4((int32_t)d, (int32_t)(loc + j * db), (int32_t)row,
                                                    (int32_t)(d - j * db < db ? d - j * db : db));
        }
        if (tid == 0) {
            ov_chunk_start[n_ov] = (int32_t)all;
            out->fallback = 0;
            out->bad_rowptr = s_bad;
            out->bad_colidx = s_badc;
            out->max_deg = s_max;
            out->rowptr_first = base;
            out->rowptr_last = rowptr[n];
            out->n_ov_heavy = s_nhv;
            out->nb_small = nb_small;
            out->n_zero = n_zero;
            out->n_ov = n_ov;
            out->ov_chunks = (int64_t)s_ovc;
            out->ov_chunks_heavy = (int64_t)s_ovh;
        }
    }
}

// Returns false (nothing allocated) when the graph is outside the one-CTA limits or has more
// than kSmallOv oversized rows; errors (bad CSR) are thrown as in the general path.
bool build_block_plan_small(agcn_plan_s* p, const int32_t* rowptr, const int32_t* colidx,
                            const agcn_opts_t& o, cudaStream_t s) {
    if (!o.small_plan) return false;
    const int64_t n = p->n, nnz = p->nnz;
    const int32_t db = p->deg_bound;
    if (n <= 0 || n > kSmallRows || nnz > kSmallNnz || db > kSmallDb) return false;
    const int32_t nbins = db + 2;
    const size_t smem = sizeof(int32_t) * (size_t)(33 * nbins + db + 2 + 2 * kSmallOv + nbins + 2) +
                        sizeof(int64_t) * 64 + sizeof(int16_t) * (size_t)n + 16;
    const int64_t desc_cap = n + nnz / db + kSmallOv + 1;
    const int64_t ovc_cap = std::min<int64_t>(n, kSmallOv) + 1;
    Scratch tmp(s);
    SmallOut* d_out = tmp.alloc<SmallOut>(1);
    AGCN_CUDA(cudaMemsetAsync(d_out, 0, sizeof(SmallOut), s));
    p->perm = dalloc<int32_t>(n, s);
    p->sorted_rowptr = dalloc<int32_t>(n + 1, s);
    p->row_src_off = dalloc<int32_t>(n, s);
    p->desc = dalloc<int4>(desc_cap, s);
    p->ov_chunk_start = dalloc<int32_t>(ovc_cap, s);
    static bool attr[64] = {};  // the shared-memory opt-in is per device
    if (p->device < 0 || p->device >= 64 || !attr[p->device]) {
        AGCN_CUDA(cudaFuncSetAttribute(k_plan_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(int32_t) * (35 * (kSmallDb + 2) + 2 * kSmallOv + 2) +
                                             sizeof(int64_t) * 64 + sizeof(int16_t) * kSmallRows + 16)));
        if (p->device >= 0 && p->device < 64) attr[p->device] = true;
    }
    k_plan_small<<<1, kSmallThreads, smem, s>>>(rowptr, colidx, n, nnz, p->n_cols, db, p->mbw, p->mwn,
                                                o.validate, p->perm, p->sorted_rowptr, p->row_src_off,
                                                p->desc, p->ov_chunk_start, d_out);
    post_launch();
    // the plan's colidx copy, before the readback: nothing reads the caller's arrays after return
    p->cols_copy = dalloc<int32_t>(nnz, s);
    launch_copy_cols(p, colidx, rowptr, nullptr, nullptr, s);
    SmallOut h{};
    auto* pin = static_cast<SmallOut*>(pinned_staging(sizeof(SmallOut)));
    AGCN_CUDA(cudaMemcpyAsync(pin ? pin : &h, d_out, sizeof(SmallOut), cudaMemcpyDeviceToHost, s));
    AGCN_CUDA(cudaStreamSynchronize(s));
    if (pin) h = *pin;
    if (h.fallback) {
        for (void* q : {(void*)p->perm, (void*)p->sorted_rowptr, (void*)p->row_src_off, (void*)p->desc,
                        (void*)p->ov_chunk_start, (void*)p->cols_copy})
            cudaFreeAsync(q, s);
        p->perm = p->sorted_rowptr = p->row_src_off = p->ov_chunk_start = p->cols_copy = nullptr;
        p->desc = nullptr;
        return false;
    }
    PlanFlags f{};
    f.bad_rowptr = h.bad_rowptr;
    f.rowptr_first = h.rowptr_first;
    f.rowptr_last = h.rowptr_last;
    check_csr_flags(f, nnz);
    AGCN_CHECK(!h.bad_colidx, AGCN_ERR_BAD_CSR, "colidx out of [0, n_cols)");
    p->rp_base = h.rowptr_first;
    p->n_zero = h.n_zero;
    p->n_ov = h.n_ov;
    p->ov_start = n - h.n_ov;
    p->ov_chunks = h.ov_chunks;
    p->ov_chunks_heavy = h.ov_chunks_heavy;
    p->n_ov_heavy = h.n_ov_heavy;
    p->max_deg = h.max_deg;
    p->nb_small = h.nb_small;
    p->nblocks = h.nb_small + h.ov_chunks;
    p->device_bytes = sizeof(int32_t) * (size_t)(3 * n + 1 + ovc_cap + nnz) + sizeof(int4) * (size_t)desc_cap;
    encode_hot_from_tail(p, hot_rows_for(p, o.hot_rows), s);
    build_ov_order(p, o.chunk_buckets, s);
    return true;
}

// ---------------------------------------------------------------- block-partition plan
// Host synchronisation: the plan waits for two events on its stream and never for the stream
// itself.  Stream order:
//   [deg_hist (+ the plan's rowptr copy), bucket-table scan, bucket totals, hot threshold]
//   -> D2H of the flags + bucket counts, event E1
//   [hot set from the histogram, the colidx copy with the hot encoding + colidx validation]
//   -> D2H of the colidx flag, event E2
//   [scatter, oversized radix sort, sorted rows, Alg. 1/2 descriptors, chunk order]
// The host waits for E1 (sizes, rowptr validity) while the GPU runs the copy, enqueues the
// rest behind it, then waits for E2 (colidx validity) and returns while the GPU finishes the
// sort: no GPU idle time at either wait, and the caller's next launches queue behind the plan.
// After E2 nothing reads the caller's rowptr / colidx (the later kernels read the plan's
// rowptr copy), so the caller may free or change them once agcn_plan has returned.
namespace {

// Small device -> host read-backs without a copy engine: a one-CTA kernel stores the words
// straight into mapped pinned host memory (PCIe posted writes).  A cudaMemcpyAsync would queue
// on the D2H copy engine -- behind the previous job's gigabyte copy-out in the pipelined
// executor.  Visible to the host once an event recorded after the kernel has completed.
__global__ void k_readback(const uint32_t* __restrict__ src, uint32_t* dst, int32_t nwords) {
    for (int32_t i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
}
void readback(void* host_mapped, const void* dev, size_t bytes, cudaStream_t s) {
    k_readback<<<1, 256, 0, s>>>(static_cast<const uint32_t*>(dev), static_cast<uint32_t*>(host_mapped),
                                 (int32_t)(bytes / 4));
    post_launch();
}

// mapped pinned host staging (cudaHostAllocMapped: device-writable through the same pointer);
// only written by read-back kernels the host has waited for before the next plan reuses it
struct PinnedSlot {
    void* buf = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (buf) cudaFreeHost(buf);
            buf = nullptr;
            cap = 0;
            AGCN_CUDA(cudaHostAlloc(&buf, bytes, cudaHostAllocMapped));
            cap = bytes;
        }
        return buf;
    }
};
// per host thread and device: 0 the readbacks, 1 the colidx flag; E1, E2
struct PlanSync {
    PinnedSlot pin[2];
    cudaEvent_t e1 = nullptr, e2 = nullptr;
};
PlanSync& plan_sync(int dev) {
    thread_local PlanSync ps[64];
    PlanSync& r = ps[dev >= 0 && dev < 64 ? dev : 0];
    if (!r.e1) {
        AGCN_CUDA(cudaEventCreateWithFlags(&r.e1, cudaEventDisableTiming));
        AGCN_CUDA(cudaEventCreateWithFlags(&r.e2, cudaEventDisableTiming));
    }
    return r;
}

}  // namespace

void build_block_plan(agcn_plan_s* p, const int32_t* rowptr, const int32_t* colidx,
                      const agcn_opts_t& o, cudaStream_t s) {
    const int64_t n = p->n, nnz = p->nnz;
    const int32_t db = p->deg_bound, nbins = db + 2;
    const int64_t ntiles = std::max<int64_t>(1, (n + kTile - 1) / kTile);
    PlanSync& ps = plan_sync(p->device);

    Scratch tmp(s);
    PlanFlags* d_flags = tmp.alloc<PlanFlags>(1);
    int32_t* bin_cnt = tmp.alloc<int32_t>(nbins);
    int32_t* table = tmp.alloc<int32_t>((size_t)nbins * ntiles + 1);
    int32_t* rp = tmp.alloc<int32_t>(n + 1);  // the plan's rowptr copy (written by k_deg_hist)
    AGCN_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(PlanFlags), s));

    // (1)+(2a) per-tile bucket histograms, bucket totals, max degree, rowptr validation
    k_deg_hist<<<(unsigned)ntiles, kThreads, nbins * sizeof(int32_t), s>>>(rowptr, n, db, nbins, ntiles,
                                                                         table, d_flags, rp);
    post_launch();
    exclusive_scan_i32(table, table, (int64_t)nbins * ntiles, s);
    k_bin_totals<<<(nbins + 255) / 256, 256, 0, s>>>(table, ntiles, nbins, n, bin_cnt);
    post_launch();
    const int64_t Hreq = hot_rows_req(p, o.hot_rows);
    if (Hreq > 0) {  // hot set from the histogram (reading Q35 = the tail of the stable degree order)
        k_hot_tau<<<1, 32, 0, s>>>(bin_cnt, db, n, Hreq, d_flags);
        post_launch();
    }
    auto* pin0 = static_cast<unsigned char*>(ps.pin[0].get(sizeof(PlanFlags) + sizeof(int32_t) * nbins));
    readback(pin0, d_flags, sizeof(PlanFlags), s);
    readback(pin0 + sizeof(PlanFlags), bin_cnt, sizeof(int32_t) * nbins, s);
    AGCN_CUDA(cudaEventRecord(ps.e1, s));

    // the plan's colidx copy (caller's order) with the hot encoding and the range check
    p->cols_copy = dalloc<int32_t>(nnz, s);
    p->device_bytes = sizeof(int32_t) * (size_t)nnz;
    uint2* hot = nullptr;
    if (Hreq > 0 && nnz > 0) {
        const int64_t nw = (n + 31) / 32;
        hot = tmp.alloc<uint2>(nw);
        uint32_t* eqw = tmp.alloc<uint32_t>(nw);
        int32_t* eqc = tmp.alloc<int32_t>(nw + 1);
        int32_t* cnt = tmp.alloc<int32_t>(nw + 1);
        p->hot_cols = dalloc<int32_t>(Hreq, s);
        p->device_bytes += sizeof(int32_t) * (size_t)Hreq;
        k_hot_deg_a<<<blocks_for(n, 256), 256, 0, s>>>(rp, n, d_flags, hot, eqw, eqc);
        post_launch();
        exclusive_scan_i32(eqc, eqc, nw, s);
        k_hot_deg_b<<<blocks_for(nw, 256), 256, 0, s>>>(hot, eqw, eqc, nw, d_flags, cnt);
        post_launch();
        exclusive_scan_i32(cnt, cnt, nw, s);
        k_hot_list<<<blocks_for(nw, 256), 256, 0, s>>>(hot, cnt, nw, p->hot_cols);
        post_launch();
    }
    launch_copy_cols(p, colidx, rp, hot, o.validate ? d_flags : nullptr, s);
    auto* pin1 = static_cast<int32_t*>(ps.pin[1].get(sizeof(int32_t)));
    readback(pin1, &d_flags->bad_colidx, sizeof(int32_t), s);
    AGCN_CUDA(cudaEventRecord(ps.e2, s));

    // the bucket counts and flags (the GPU runs the copy meanwhile)
    AGCN_CUDA(cudaEventSynchronize(ps.e1));
    PlanFlags hf{};
    std::vector<int32_t> h_cnt(nbins);
    memcpy(&hf, pin0, sizeof(PlanFlags));
    memcpy(h_cnt.data(), pin0 + sizeof(PlanFlags), sizeof(int32_t) * nbins);
    check_csr_flags(hf, nnz);
    p->rp_base = hf.rowptr_first;

    // host-side bucket bookkeeping (tiny: deg_bound + 2 entries)
    std::vector<int32_t> br, wn;
    host_patterns(p->mbw, p->mwn, br, wn);
    const int32_t W = db + 2;
    // (pageable on purpose: a small pageable H2D is staged through the command stream at once,
    // while a pinned one waits for the copy engine -- behind a job's gigabyte copy-in in the
    // pipelined executor, which measured 488 -> 435 GFLOP/s e2e)
    std::vector<int32_t> tabv(6 * W, 0);
    int32_t* tab = tabv.data();
    int32_t* nnz_start = tab;
    int32_t* row_start = tab + W;
    int32_t* blk_start = tab + 2 * W;
    int32_t* cntv = tab + 3 * W;
    int32_t* brv = tab + 4 * W;
    int32_t* wnv = tab + 5 * W;
    int64_t row = h_cnt[0], loc = 0, blk = 0;
    for (int32_t d = 1; d <= db + 1; ++d) {
        nnz_start[d] = (int32_t)loc;
        row_start[d] = (int32_t)row;
        blk_start[d] = (int32_t)blk;
        if (d <= db) {
            cntv[d] = h_cnt[d];
            brv[d] = br[d];
            wnv[d] = wn[d];
            row += h_cnt[d];
            loc += (int64_t)h_cnt[d] * d;
            blk += (h_cnt[d] + br[d] - 1) / br[d];
        }
    }
    p->n_zero = h_cnt[0];
    p->n_ov = h_cnt[db + 1];
    p->ov_start = n - p->n_ov;
    p->ov_chunks = hf.ov_chunks;
    p->ov_chunks_heavy = hf.ov_chunks_heavy;
    p->n_ov_heavy = hf.n_ov_heavy;
    p->max_deg = hf.max_deg;
    p->nb_small = blk;
    p->nblocks = blk + hf.ov_chunks;
    p->n_hot = hot ? hf.n_hot : 0;
    AGCN_CHECK(p->nblocks < (1ll << 31), AGCN_ERR_OVERFLOW, "too many descriptors");

    // plan-owned arrays
    p->perm = dalloc<int32_t>(n, s);
    p->sorted_rowptr = dalloc<int32_t>(n + 1, s);
    p->row_src_off = dalloc<int32_t>(n, s);
    p->desc = dalloc<int4>(p->nblocks, s);
    p->ov_chunk_start = dalloc<int32_t>(p->n_ov + 1, s);
    p->device_bytes += sizeof(int32_t) * (size_t)(3 * n + 1 + p->n_ov + 1) + sizeof(int4) * (size_t)p->nblocks;

    // (2b) stable scatter into bucket order
    const size_t scat_smem = (size_t)kWarps * nbins * sizeof(int32_t);
    if (scat_smem > 48 * 1024)
        AGCN_CUDA(cudaFuncSetAttribute(k_bucket_scatter<MainSrc>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scat_smem));
    k_bucket_scatter<MainSrc><<<(unsigned)ntiles, kThreads, scat_smem, s>>>(MainSrc{rp, db, p->perm}, n, nbins, ntiles, table);
    post_launch();

    // (2c) oversized rows (degree > deg_bound) keep row order within the bucket; stable LSD
    // radix sort of that bucket by degree (8-bit digits) completes the ascending stable order.
    const int64_t m = p->n_ov;
    if (m > 1) {
        int32_t* ka = tmp.alloc<int32_t>(m);
        int32_t* va = tmp.alloc<int32_t>(m);
        int32_t* kb = tmp.alloc<int32_t>(m);
        int32_t* vb = tmp.alloc<int32_t>(m);
        k_ov_init<<<blocks_for(m, 256), 256, 0, s>>>(p->perm + p->ov_start, rp, m, ka, va);
        post_launch();
        radix_sort_pairs(ka, va, kb, vb, m, p->max_deg, s);
        AGCN_CUDA(cudaMemcpyAsync(p->perm + p->ov_start, va, sizeof(int32_t) * m,
                                  cudaMemcpyDeviceToDevice, s));
    }

    // (3) "updating the row pointer array to reflect the new row order", O(n):
    // sorted degrees -> sorted_rowptr (scan) and row_src_off (where each sorted row starts in
    // the caller's colidx / vals), one look-back scan pass.
    if (n > 0) {
        const int64_t nt = (n + kLbTile - 1) / kLbTile;
        launch_scan_lb(SortedRowsSrc{p->perm, rp, p->row_src_off}, p->sorted_rowptr, n,
                       nt > 1 ? tmp.alloc<unsigned long long>(nt + 1) : nullptr, s);
    } else {
        AGCN_CUDA(cudaMemsetAsync(p->sorted_rowptr, 0, sizeof(int32_t), s));
    }

    // (4)+(5) Algorithm 1/2 descriptors
    int32_t* d_tab = tmp.alloc<int32_t>(6 * W);
    AGCN_CUDA(cudaMemcpyAsync(d_tab, tab, sizeof(int32_t) * 6 * W, cudaMemcpyHostToDevice, s));
    if (p->nb_small > 0) {
        unsigned g = (unsigned)std::min<int64_t>(blocks_for(p->nb_small, kThreads), 148 * 8);
        size_t smem = 6 * W * sizeof(int32_t);
        if (smem > 48 * 1024)
            AGCN_CUDA(cudaFuncSetAttribute(k_emit_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        k_emit_small<<<g, kThreads, smem, s>>>(p->nb_small, db, d_tab, p->desc);
        post_launch();
    }
    if (m > 0) {
        k_ov_chunk_count<<<blocks_for(m, 256), 256, 0, s>>>(p->sorted_rowptr, p->ov_start, m, db,
                                                            p->ov_chunk_start);
        post_launch();
        exclusive_scan_i32(p->ov_chunk_start, p->ov_chunk_start, m, s);
        k_emit_ov<<<blocks_for(m, kWarps), kThreads, 0, s>>>(p->sorted_rowptr, p->ov_start, m, db,
                                                              p->nb_small, p->ov_chunk_start, p->desc);
        post_launch();
    } else {
        AGCN_CUDA(cudaMemsetAsync(p->ov_chunk_start, 0, sizeof(int32_t), s));
    }
    // the hot set among the oversized rows: from the sorted tail, encoded in place
    if (hot && hf.hot_fallback) encode_hot_from_tail(p, hot_rows_for(p, o.hot_rows), s);
    build_ov_order(p, o.chunk_buckets, s);

    // the colidx range (the copy has run by now or soon; the sort above stays queued)
    AGCN_CUDA(cudaEventSynchronize(ps.e2));
    if (o.validate && nnz > 0) AGCN_CHECK(!*pin1, AGCN_ERR_BAD_CSR, "colidx out of [0, n_cols)");
}

// ---------------------------------------------------------------- warp-partition plan
void build_warp_plan(agcn_plan_s* p, const int32_t* rowptr, const int32_t* colidx,
                     const agcn_opts_t& o, cudaStream_t s) {
    const int64_t n = p->n, nnz = p->nnz;
    Scratch tmp(s);
    PlanFlags* d_flags = tmp.alloc<PlanFlags>(1);
    AGCN_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(PlanFlags), s));
    p->rowptr_copy = dalloc<int32_t>(n + 1, s);
    int32_t* tstart = tmp.alloc<int32_t>(n + 1);
    k_rowptr_check<<<blocks_for(n + 1, 256), 256, 0, s>>>(rowptr, n, p->mwn, p->rowptr_copy, tstart,
                                                          d_flags);
    post_launch();
    // the plan's colidx copy (original order, padded-layout relabel) with the range check, before
    // the readback: nothing reads the caller's arrays after return
    p->cols_copy = dalloc<int32_t>(nnz, s);
    launch_copy_cols(p, colidx, rowptr, nullptr, o.validate ? d_flags : nullptr, s);
    exclusive_scan_i32(tstart, tstart, n, s);
    int32_t ntasks = 0;
    AGCN_CUDA(cudaMemcpyAsync(&ntasks, tstart + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PlanFlags hf{};
    read_flags(d_flags, &hf, s);
    check_csr_flags(hf, nnz);
    AGCN_CHECK(!hf.bad_colidx, AGCN_ERR_BAD_CSR, "colidx out of [0, n_cols)");
    p->ntasks = ntasks;
    p->max_deg = hf.max_deg;
    p->rp_base = hf.rowptr_first;
    p->tasks = dalloc<int4>(ntasks, s);
    p->device_bytes = sizeof(int32_t) * (size_t)(n + 1 + nnz) + sizeof(int4) * (size_t)ntasks;
    if (n > 0) {
        k_emit_tasks<<<blocks_for(n, 256), 256, 0, s>>>(p->rowptr_copy, n, p->mwn, tstart, p->tasks);
        post_launch();
    }
}

}  // namespace

void free_plan_arrays(agcn_plan_s* p) {
    void* ptrs[] = {p->perm,  p->sorted_rowptr, p->row_src_off, p->desc,       p->ov_chunk_start,
                    p->tasks, p->rowptr_copy,   p->cols_copy,   p->ov_partial, p->ov_cnt,
                    p->xhot, p->hot_cols, p->ov_order};
    // Stream-ordered release on the plan's stream, after the last SpMM that used the plan on
    // another stream (p->last_use); no host synchronisation.
    if (p->last_use) cudaStreamWaitEvent(p->stream, p->last_use, 0);
    for (void* q : ptrs)
        if (q) cudaFreeAsync(q, p->stream);
    if (p->ready) cudaEventDestroy(p->ready);
    if (p->last_use) cudaEventDestroy(p->last_use);
}

// Degree-sorted colidx for introspection (parity tests): the plan's copy, hot encoding undone.
void plan_copy_sorted_colidx(agcn_plan_s* p, int32_t* host_dst) {
    if (p->nnz == 0) return;
    cudaStream_t s = p->stream;
    Scratch tmp(s);
    int32_t* d = tmp.alloc<int32_t>(p->nnz);
    if (p->n > 0) {
        k_gather_sorted_cols<<<blocks_for(p->n, kWarps), kThreads, 0, s>>>(p->n, p->sorted_rowptr, p->row_src_off,
                                                                        p->cols_copy, p->hot_cols, d);
        post_launch();
    }
    AGCN_CUDA(cudaMemcpyAsync(host_dst, d, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToHost, s));
    AGCN_CUDA(cudaStreamSynchronize(s));
}

// Keep freed stream-ordered memory cached in the device pool (plans are rebuilt often).
static void keep_pool_cached(int dev) {
    static bool done[64] = {};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

// Alg. 1 parameters chosen from the graph's size when the caller passes (0, 0).  The paper
// fixes max_block_warps = 12 only for its storage example and never states
// max_warp_nzs (Q18); the rule below is the B200 measurement of
// profiles/r01at_auto_partition.md, in terms of share = nnz per resident warp of the default
// SpMM kernel (SMs x 24):
//   * share < 8 (tiny graphs, launch-bound):          (12, 32) -- the paper's values
//   * share < 960 (small graphs):  deg_bound = largest of 64/128/256 <= max(64, share / 2.5) --
//     oversized-row chunks short against a warp's share, so the chunk tail (processed last,
//     degree order ascending) does not set the critical path: (4,16) / (8,16) / (8,32)
//   * otherwise, mean degree < 64:                    (32, 16) -- many short rows: 32-row
//     descriptors amortise the per-descriptor metadata chain (C5 3.27 vs 3.42 ms at (12, 32))
//   * otherwise:                                       (8, 32)   -- deg_bound 256: with the X
//     loads skipping L1 and the chunks in their own 32-warp/SM kernel, more of a dense-hub
//     graph's rows go to the faster chunk kernel (C4 3.23 vs 3.31 ms at (12, 32); 192-256 all
//     within 0.5 %, profiles/r02bk_c4_partition.txt)
// (Round 1 kept dense-hub graphs, mean degree >= 256, at (24, 32) to keep their rows whole;
// with the oversized chunks executed in column-position order (round 2) (12, 32) was faster on
// C4: 3.64 vs 3.78 ms, profiles/r02x_chunk_order.txt, r02ad_partition_sweep.txt.)
void auto_partition(int64_t n, int64_t nnz, int32_t sms, int32_t* mbw, int32_t* mwn) {
    if (sms <= 0) {
        int dev = 0;
        sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const double share = (double)nnz / ((double)sms * 24.0);
    *mbw = 12;
    *mwn = 32;
    if (share < 8) return;
    if (share < 960) {
        const double t = share / 2.5;
        if (t >= 256) { *mbw = 8; *mwn = 32; }
        else if (t >= 128) { *mbw = 8; *mwn = 16; }
        else { *mbw = 4; *mwn = 16; }
        return;
    }
    if (n > 0 && nnz < 64 * n) {
        *mbw = 32;
        *mwn = 16;
    } else {
        *mbw = 8;
        *mwn = 32;
    }
}

agcn_plan_s* build_plan(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz,
                        const agcn_opts_t& oin) {
    agcn_opts_t o = oin;
    if (o.max_block_warps == 0 && o.max_warp_nzs == 0) auto_partition(n, nnz, 0, &o.max_block_warps, &o.max_warp_nzs);
    AGCN_CHECK(n >= 0 && nnz >= 0, AGCN_ERR_INVALID_ARG, "n and nnz must be >= 0");
    AGCN_CHECK(nnz < (1ll << 31) && n < (1ll << 31) - 1, AGCN_ERR_INVALID_ARG, "n, nnz must be < 2^31");
    AGCN_CHECK(rowptr != nullptr, AGCN_ERR_INVALID_ARG, "rowptr is NULL");
    AGCN_CHECK(colidx != nullptr || nnz == 0, AGCN_ERR_INVALID_ARG, "colidx is NULL");
    AGCN_CHECK(o.max_block_warps >= 1 && o.max_warp_nzs >= 1, AGCN_ERR_INVALID_ARG,
               "max_block_warps and max_warp_nzs must be >= 1");
    AGCN_CHECK(o.max_block_warps < 65536 && o.max_warp_nzs < 65536, AGCN_ERR_OVERFLOW,
               "block_rows / warp_nzs must fit the 16-bit info halves");
    AGCN_CHECK((int64_t)o.max_block_warps * o.max_warp_nzs <= kMaxDegBound, AGCN_ERR_UNSUPPORTED,
               "deg_bound = max_block_warps * max_warp_nzs must be <= 2048 in this build");
    AGCN_CHECK(o.partition == AGCN_PARTITION_BLOCK || o.partition == AGCN_PARTITION_WARP,
               AGCN_ERR_INVALID_ARG, "unknown partition");
    const int64_t n_cols = o.n_cols > 0 ? o.n_cols : n;
    AGCN_CHECK(n_cols < (1ll << 31), AGCN_ERR_INVALID_ARG, "n_cols must be < 2^31");
    cudaStream_t s = (cudaStream_t)o.stream;

    agcn_plan_s* p = new agcn_plan_s();
    try {
        p->cmap = make_colmap(o, n_cols);
        AGCN_CUDA(cudaGetDevice(&p->device));
        keep_pool_cached(p->device);
        p->n = n;
        p->n_cols = n_cols;
        p->nnz = nnz;
        p->mbw = o.max_block_warps;
        p->mwn = o.max_warp_nzs;
        p->deg_bound = o.max_block_warps * o.max_warp_nzs;
        p->partition = o.partition;
        p->x_rows = o.col_nparts > 0 ? (int64_t)o.col_nparts * o.col_slot_rows : n_cols;
        p->stream = s;
        if (o.partition == AGCN_PARTITION_BLOCK)
        {
            if (!build_block_plan_small(p, rowptr, colidx, o, s)) build_block_plan(p, rowptr, colidx, o, s);
        }
        else
            build_warp_plan(p, rowptr, colidx, o, s);
        AGCN_CUDA(cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming));
        AGCN_CUDA(cudaEventRecord(p->ready, s));
    } catch (...) {
        cudaStreamSynchronize(s);
        free_plan_arrays(p);
        delete p;
        throw;
    }
    return p;
}

}  // namespace agcn
