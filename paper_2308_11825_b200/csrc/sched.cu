// sched.cu -- column-blocked execution schedule for the oversized rows (degree > deg_bound).
//
// Not part of the paper's metadata (the plan's descriptors stay exactly Algorithm 2's,
// P:335-382): a B200 execution detail of agcn_spmm for X larger than the L2 share it can
// keep.  Algorithm 2 splits a row with
// degree > deg_bound into chunks of deg_bound nonzeros whose partial rows are merged at
// level 3 (global atomics in the paper; a fixed-order reduction here).  For the
// heavy rows (degree >= kMinDeg) this schedule further cuts every chunk into PIECES where the
// column block changes (block = column >> shift: 2^shift rows of X ~ an L2-sized slice) and
// lists the pieces block-major, so that all warps gather from one L2-resident slice of X at
// a time.  Each piece writes one partial row to its own slot (slots are chunk-major, so the
// slots of a row are contiguous and ordered), and k_ov_reduce sums a row's slots in slot
// order: results are deterministic and independent of the execution order.
//
// A chunk whose columns are not non-decreasing (from the entry before it), or of a lighter
// row, stays one piece (the paper's chunk).  At most kMaxPieces pieces per chunk: later block
// changes stay inside the last piece (still correct, only less local).  Built on the SpMM
// stream on first use for a given block width (it depends on F), one warp per chunk, without
// host synchronisation: the piece count stays on the device and the SpMM grid is sized by
// an upper bound known from the plan.
#include <algorithm>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Chunk {
    int32_t base;  // first entry in the caller's colidx / vals (rowptr-relative)
    int32_t len;   // entries (<= deg_bound)
    bool heavy;    // the row's degree >= kColBlockMinDeg
};

__device__ __forceinline__ Chunk ov_chunk(const int4* __restrict__ desc, const int32_t* __restrict__ srp,
                                          const int32_t* __restrict__ rso, int64_t j) {
    const int4 m = desc[j];  // {deg, loc, row, len} (Algorithm 2, oversized branch)
    return {rso[m.z] + (m.y - srp[m.z]), m.w, m.x >= kColBlockMinDeg};
}

// Walk a chunk in 32-entry batches; fn(e, blk, boundary) per batch (lane-parallel).  A piece
// starts at entry 0 and where the column block changes.  Returns whether the chunk's
// columns are non-decreasing, starting from the entry before it (if any, `prev`).
template <class Fn>
__device__ __forceinline__ bool walk_chunk(const int32_t* __restrict__ cols, Chunk c, int32_t prev, int shift,
                                           Fn&& fn) {
    const int lane = threadIdx.x & 31;
    int32_t carry_col = prev, carry_blk = -1;
    bool sorted = true;
    for (int32_t e0 = 0; e0 < c.len; e0 += 32) {
        const int32_t e = e0 + lane;
        const bool valid = e < c.len;
        const int32_t col = valid ? __ldg(cols + c.base + e) : INT32_MAX;
        const int32_t blk = col >> shift;
        int32_t pcol = __shfl_up_sync(0xffffffffu, col, 1);
        int32_t pblk = __shfl_up_sync(0xffffffffu, blk, 1);
        if (lane == 0) {
            pcol = carry_col;
            pblk = carry_blk;
        }
        if (valid && col < pcol) sorted = false;
        fn(e, blk, valid && (e == 0 || blk != pblk));
        carry_col = __shfl_sync(0xffffffffu, col, 31);
        carry_blk = __shfl_sync(0xffffffffu, blk, 31);
    }
    return __all_sync(0xffffffffu, sorted);
}

__device__ __forceinline__ int32_t prev_entry(const int32_t* __restrict__ cols, const int4* __restrict__ desc,
                                              const int32_t* __restrict__ srp, int64_t j, Chunk c) {
    const int4 m = desc[j];
    return m.y > srp[m.z] ? __ldg(cols + c.base - 1) : INT32_MIN;  // not the row's first chunk
}

// Pass A: pieces per chunk (<= kMaxPieces; 1 for a chunk that stays whole) and pieces per
// column block (bucket nb: whole chunks).  kind[j] = 1 when the chunk is cut at blocks.
__global__ void __launch_bounds__(kThreads) k_seg_count(const int32_t* __restrict__ cols,
                                                       const int4* __restrict__ desc,
                                                       const int32_t* __restrict__ srp,
                                                       const int32_t* __restrict__ rso, int64_t n_chunks,
                                                       int shift, int32_t nb, int32_t* __restrict__ pieces,
                                                       int32_t* __restrict__ kind,
                                                       int32_t* __restrict__ blk_cnt) {
    const int64_t j = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (j >= n_chunks) return;
    const int lane = threadIdx.x & 31;
    const Chunk c = ov_chunk(desc, srp, rso, j);
    bool sorted = false;
    if (c.heavy) {
        const int32_t prev = prev_entry(cols, desc, srp, j, c);
        sorted = walk_chunk(cols, c, prev, shift, [&](int32_t, int32_t, bool) {});
    }
    if (!sorted) {
        if (lane == 0) {
            pieces[j] = 1;
            kind[j] = 0;
            atomicAdd(&blk_cnt[nb], 1);
        }
        return;
    }
    int32_t seen = 0;  // boundaries so far; the first kMaxPieces start pieces
    walk_chunk(cols, c, INT32_MIN, shift, [&](int32_t, int32_t blk, bool bnd) {
        const unsigned m = __ballot_sync(0xffffffffu, bnd);
        const int rank = seen + __popc(m & ((1u << lane) - 1u));
        if (bnd && rank < kMaxPieces) atomicAdd(&blk_cnt[blk], 1);
        seen += __popc(m);
    });
    if (lane == 0) {
        pieces[j] = min(seen, kMaxPieces);
        kind[j] = 1;
    }
}

// the lowest k set bits of m
__device__ __forceinline__ unsigned lowest_bits(unsigned m, int k) {
    while (__popc(m) > k) m &= ~(1u << (31 - __clz(m)));
    return m;
}

// Pass B: emit the pieces {-1 - slot, first entry, 0, length} at block-major positions.
__global__ void __launch_bounds__(kThreads) k_seg_emit(const int32_t* __restrict__ cols,
                                                      const int4* __restrict__ desc,
                                                      const int32_t* __restrict__ srp,
                                                      const int32_t* __restrict__ rso, int64_t n_chunks,
                                                      int shift, int32_t nb, const int32_t* __restrict__ pieces,
                                                      const int32_t* __restrict__ kind,
                                                      const int32_t* __restrict__ slot0,
                                                      const int32_t* __restrict__ blk_start,
                                                      int32_t* __restrict__ blk_cursor, int4* __restrict__ seg) {
    const int64_t j = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (j >= n_chunks) return;
    const int lane = threadIdx.x & 31;
    const Chunk c = ov_chunk(desc, srp, rso, j);
    const int32_t s0 = slot0[j], np = pieces[j];
    if (kind[j] == 0) {  // the whole chunk (lighter row or unsorted): bucket nb
        if (lane == 0) {
            const int32_t pos = blk_start[nb] + atomicAdd(&blk_cursor[nb], 1);
            seg[pos] = make_int4(-1 - s0, c.base, 0, c.len);
        }
        return;
    }
    // the first np boundaries start pieces; piece r ends where piece r + 1 starts
    int32_t seen = 0, p_start = -1, p_blk = 0;
    auto emit = [&](int32_t start, int32_t end, int32_t blk, int32_t r) {
        const int32_t pos = blk_start[blk] + atomicAdd(&blk_cursor[blk], 1);
        seg[pos] = make_int4(-1 - (s0 + r), c.base + start, 0, end - start);
    };
    walk_chunk(cols, c, INT32_MIN, shift, [&](int32_t e, int32_t blk, bool bnd) {
        const unsigned m = lowest_bits(__ballot_sync(0xffffffffu, bnd), max(0, np - seen));
        if (m == 0) return;
        const int first = __ffs(m) - 1;
        const int32_t e_first = __shfl_sync(0xffffffffu, e, first);
        if (lane == 0 && p_start >= 0) emit(p_start, e_first, p_blk, seen - 1);  // close pending
        if ((m >> lane) & 1u) {
            const unsigned later = m & ~((2u << lane) - 1u);
            const int r = seen + __popc(m & ((1u << lane) - 1u));
            if (later) emit(e, e + (__ffs(later) - 1 - lane), blk, r);
        }
        const int last = 31 - __clz(m);
        p_start = __shfl_sync(0xffffffffu, e, last);
        p_blk = __shfl_sync(0xffffffffu, blk, last);
        seen += __popc(m);
    });
    if (lane == 0 && p_start >= 0) emit(p_start, c.len, p_blk, np - 1);
}

// slot range of oversized row k: [slot0[chunk_start[k]], slot0[chunk_start[k + 1]])
__global__ void k_row_slots(const int32_t* __restrict__ chunk_start, const int32_t* __restrict__ slot0,
                            int64_t n_ov, int32_t* __restrict__ row_slot) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k <= n_ov) row_slot[k] = slot0[chunk_start[k]];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

void free_col_sched(ColSched& cs, cudaStream_t s) {
    dfree(cs.seg, s);
    dfree(cs.slot_base, s);
    dfree(cs.partial, s);
    cs = ColSched{};
}

// Column-block width for F: the largest power of two 2^shift with 2^shift * 4F <= target
// bytes; -1 when blocking does not apply (X already fits that slice, or no heavy rows).
int col_sched_shift(const agcn_plan_s* p, int32_t F, double target_bytes) {
    if (p->ov_chunks_heavy == 0 || target_bytes <= 0) return -1;
    const double x_bytes = 4.0 * (double)p->x_rows * F;
    if (x_bytes <= target_bytes) return -1;
    int shift = 0;
    while (shift < 30 && (double)(int64_t(1) << (shift + 1)) * 4.0 * F <= target_bytes) ++shift;
    return shift;
}

void build_col_sched(agcn_plan_s* p, int shift, int32_t F, cudaStream_t s) {
    ColSched& cs = p->sched;
    const int64_t n_ov = p->n_ov, n_chunks = p->ov_chunks;
    const int32_t nb = (int32_t)((p->x_rows + (int64_t(1) << shift) - 1) >> shift);  // column blocks
    const int64_t cap = p->ov_chunks + (int64_t)(kMaxPieces - 1) * p->ov_chunks_heavy;
    AGCN_CHECK(cap < (1ll << 31), AGCN_ERR_OVERFLOW, "too many column-block pieces");
    if (!cs.seg || cs.cap < cap) {
        dfree(cs.seg, s);
        dfree(cs.slot_base, s);
        cs.seg = dalloc<int4>(cap, s);
        cs.slot_base = dalloc<int32_t>(n_ov + 1, s);
        cs.cap = cap;
    }
    cs.shift = shift;
    cs.nb = nb;
    Scratch tmp(s);
    int32_t* slot0 = tmp.alloc<int32_t>(n_chunks + 1);     // pieces -> first slot per chunk
    int32_t* pieces = tmp.alloc<int32_t>(n_chunks + 1);
    int32_t* kind = tmp.alloc<int32_t>(n_chunks + 1);
    int32_t* blk = tmp.alloc<int32_t>(2 * (nb + 2));      // counts -> starts, cursors
    int32_t* blk_start = blk;
    int32_t* blk_cursor = blk + (nb + 2);
    AGCN_CUDA(cudaMemsetAsync(blk, 0, sizeof(int32_t) * 2 * (nb + 2), s));
    const unsigned g = blocks_for(n_chunks, kWarps);
    const int4* ovd = p->desc + p->nb_small;
    k_seg_count<<<g, kThreads, 0, s>>>(p->cols, ovd, p->sorted_rowptr, p->row_src_off, n_chunks, shift, nb,
                                       pieces, kind, blk_start);
    post_launch();
    exclusive_scan_i32(pieces, slot0, n_chunks, s);
    exclusive_scan_i32(blk_start, blk_start, nb + 1, s);
    k_seg_emit<<<g, kThreads, 0, s>>>(p->cols, ovd, p->sorted_rowptr, p->row_src_off, n_chunks, shift, nb,
                                      pieces, kind, slot0, blk_start, blk_cursor, cs.seg);
    post_launch();
    k_row_slots<<<blocks_for(n_ov + 1, 256), 256, 0, s>>>(p->ov_chunk_start, slot0, n_ov, cs.slot_base);
    post_launch();
    // the piece count (= slot_base[n_ov]) is read by the SpMM on the device
    cs.partial_need = (size_t)cap * (size_t)F;
    if (cs.partial_need > cs.partial_floats) {
        dfree(cs.partial, s);
        cs.partial = dalloc<float>(cs.partial_need, s);
        cs.partial_floats = cs.partial_need;
    }
    cs.F = F;
}

}  // namespace agcn
