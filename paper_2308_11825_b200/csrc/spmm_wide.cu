// spmm_wide.cu -- the occupancy-first SpMM kernel for F = 8 L <= 256 (L lanes of 32 B per X row).
//
// Same work decomposition and results contract as k_spmm_block (spmm.cu): one 128-bit
// descriptor {deg, loc, row, info} per warp at a time, a "combined warp"
// of L = F/8 lanes per X row, G = 32/L of them per warp.  What changes is how the
// kernel reaches the L2->SM gather roof on B200 (tools/gather_probe.cu: ~18-19 TB/s random
// row gathers need 64 resident warps per SM, i.e. <= 32 registers and no shared memory):
//  * every lane moves 32 bytes per X row with one 256-bit load (LDG.E.256), so a warp issues
//    G rows per load instruction;
//  * no shared-memory staging: a combined warp loads L (colidx, val) pairs with one
//    coalesced load per lane and broadcasts them with shuffles;
//  * rows are whole units of a combined warp: a descriptor's R rows go round-robin to
//    groups of K combined warps (K = the largest power of two with K*R <= G); the K
//    members of a group split the row's nonzeros into contiguous parts and add their
//    partial rows with a fixed xor-shuffle tree.  The paper's level-2 merge
//    (atomicAdd_block) becomes that deterministic shuffle tree; level 3
//    (rows with degree > deg_bound) writes per-chunk partial rows summed by k_ov_reduce.
//  * the row offsets / output rows of the descriptor (<= 32 rows) are fetched once per
//    descriptor, one per lane, and shuffled to the combined warps.
//  * colidx / vals are read straight from the caller's CSR through row_src_off (the plan
//    never copies them), one batch of pairs ahead (prefetch); both are evict-first streams
//    (ld.global.cs).  When X fits in L2 its rows are loaded with an evict_last hint.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

struct f8 {
    float4 a, b;
};

__device__ __forceinline__ void ld8(f8& r, const float* p, int hint) {
    // hint: 0 plain, 1 evict_last (hot), 2 evict_first (cold)
    if (hint == 1)
        asm("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else if (hint == 2)
        asm("ld.global.nc.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else
        asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
}

__device__ __forceinline__ void fma8(f8& acc, float v, const f8& x) {
    acc.a.x = fmaf(v, x.a.x, acc.a.x);
    acc.a.y = fmaf(v, x.a.y, acc.a.y);
    acc.a.z = fmaf(v, x.a.z, acc.a.z);
    acc.a.w = fmaf(v, x.a.w, acc.a.w);
    acc.b.x = fmaf(v, x.b.x, acc.b.x);
    acc.b.y = fmaf(v, x.b.y, acc.b.y);
    acc.b.z = fmaf(v, x.b.z, acc.b.z);
    acc.b.w = fmaf(v, x.b.w, acc.b.w);
}

__device__ __forceinline__ void st8(float* p, const f8& v) {
    __stcs(reinterpret_cast<float4*>(p), v.a);
    __stcs(reinterpret_cast<float4*>(p) + 1, v.b);
}

__device__ __forceinline__ float shfl_xor_add(float v, int o) {
    return v + __shfl_xor_sync(0xffffffffu, v, o);
}

struct WideArgs {
    const int4* desc;
    int64_t n_desc;       // descriptors executed from desc (nblocks, or nb_small with pieces)
    int64_t first_ov;     // descriptor index of the first oversized chunk
    int64_t n_zero;       // sorted rows [0, n_zero) have degree 0
    const int32_t* cols;  // column indices, indexed like vals (rowptr-relative)
    const int32_t* srp;   // sorted rowptr
    const int32_t* rso;   // row_src_off
    const int32_t* perm;  // sorted -> original row
    const float* vals;    // caller vals, offset by rowptr[0]
    const float* X;
    float* Y;
    float* ovp;           // oversized partial rows [ov_chunks][F]
    int32_t db;           // deg_bound
    const int4* pieces;   // column-blocked pieces of the oversized rows (sched.cu), or NULL
    const int32_t* n_pieces;  // device: number of pieces
    float* piece_partial; // [pieces][F] partial rows (slot-indexed)
    int64_t piece_cap;    // upper bound of the piece count (grid sizing)
    Epi epi;              // output epilogue (EPI)
    int32_t L;            // lanes per X row (F / 8); used when the kernel's LT is 0
    int32_t zero_last;    // write the degree-0 rows after the descriptors (A/B: AGCN_ZERO_LAST)
    int32_t fuse_ov;      // level 3 of rows of <= kHeavyChunks chunks done by the last warp
    const int32_t* ov_cs; // [n_ov + 1] first chunk of oversized row k
    int32_t* ov_cnt;      // [n_ov] chunks of row k finished (zero between launches)
    int64_t ov_start;     // sorted position of the first oversized row
    int32_t lean;         // auto shape choice: U 2 at 4 CTAs/SM (see launch<L>)
};


// a finished output row slice of 8 floats at column c of original row orow (degree deg)
template <bool EPI>
__device__ __forceinline__ void store_row(float* Y, int64_t orow, int32_t c, int32_t F, int32_t deg, f8 v,
                                          const Epi& e) {
    if (EPI) {
        v.a = epi4(v.a, deg, orow, c, e);
        v.b = epi4(v.b, deg, orow, c + 4, e);
    }
    st8(Y + orow * F + c, v);
    if (EPI) {
        fanout4(e, orow * F + c, v.a);
        fanout4(e, orow * F + c + 4, v.b);
    }
}

// Level 3 fused (deterministic): after a warp has written the partial row of an
// oversized chunk, it counts the chunk in; the warp that completes a row of at most
// kHeavyChunks chunks sums that row's partials in chunk order (L2 loads: they were written by
// other SMs), applies the epilogue, stores the output row and re-arms the counter.  Heavier rows
// keep their CTA-wide reduction kernel.
template <bool EPI>
__device__ __noinline__ void ov_finish(const WideArgs& a, int32_t row, int32_t deg, int32_t F, int lane,
                                       int s, int li) {
    __threadfence();                 // publish this warp's partial-row stores
    __syncwarp();
    const int64_t k = row - a.ov_start;
    const int32_t c0 = __ldg(a.ov_cs + k), nc = __ldg(a.ov_cs + k + 1) - c0;
    if (nc > kHeavyChunks) return;
    int last = 0;
    if (lane == 0) last = atomicAdd(a.ov_cnt + k, 1) == nc - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();                 // the other chunks' partials are visible from here on
    if (s == 0) {
        f8 acc;
        acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
        const float* base = a.ovp + (int64_t)c0 * F + li * 8;
#pragma unroll 4
        for (int32_t j = 0; j < nc; ++j) {
            const float4 x0 = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)j * F));
            const float4 x1 = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)j * F) + 1);
            acc.a.x += x0.x; acc.a.y += x0.y; acc.a.z += x0.z; acc.a.w += x0.w;
            acc.b.x += x1.x; acc.b.y += x1.y; acc.b.z += x1.z; acc.b.w += x1.w;
        }
        store_row<EPI>(a.Y, __ldg(a.perm + row), li * 8, F, deg, acc, a.epi);
    }
    if (lane == 0) a.ov_cnt[k] = 0;
}

// L lanes per X row (F = 8 L), U X rows in flight per lane, MINB resident CTAs per SM
// (register budget), KEEP: X-row loads carry an L2 evict_last hint.
// LT = 0: L is a runtime value (a.L), for the F = 8 L with L not a power of two.
template <int LT, int U, int MINB, bool KEEP, bool PIECES, bool EPI>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_wide(const __grid_constant__ WideArgs a) {
    const int L = LT ? LT : a.L;
    const int G = 32 / L;                     // combined warps per warp; lanes >= G L idle
    const int F = 8 * L;
    constexpr bool UDIV = LT && LT % U == 0;  // else the last round of a batch may be partial
    constexpr bool FULL = LT && 32 % LT == 0; // every lane in a combined warp
    constexpr bool POW2 = LT && (LT & (LT - 1)) == 0;
    const int lane = threadIdx.x & 31;
    const int s = lane / L, li = lane % L;
    const bool act = FULL || s < G;           // an idle lane (s == G) only joins the shuffles
    const int32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int32_t W = gridDim.x * kWarps;

    // degree-0 rows: Y row = 0 (reading Q16); 32 rows per warp step, one perm load per lane.
    // Before the descriptors, or after them (a.zero_last: the stores then fill the tail left by
    // the last, longest descriptors instead of preceding the gathers)
    auto zero_rows = [&]() {
        f8 z;
        z.a = z.b = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t r0 = (int64_t)gw * 32; r0 < a.n_zero; r0 += (int64_t)W * 32) {
            const int32_t pr = r0 + lane < a.n_zero ? __ldg(a.perm + r0 + lane) : -1;
#pragma unroll 4
            for (int i = 0; i < 32; i += G) {
                const int32_t o = __shfl_sync(0xffffffffu, pr, FULL ? i + s : (i + s) & 31);
                if (act && (FULL || i + s < 32) && o >= 0) store_row<EPI>(a.Y, o, li * 8, F, 0, z, a.epi);
            }
        }
    };
    if (!a.zero_last) zero_rows();

    // execution list: the plan's descriptors [0, n_desc), then (when the column-blocked
    // schedule replaces the oversized chunks) its pieces, block-major
    const int32_t n_desc = (int32_t)a.n_desc;
    const int32_t n_exec = n_desc + (PIECES ? __ldg(a.n_pieces) : 0);
    for (int32_t b = gw; b < n_exec; b += W) {
        const bool piece = PIECES && b >= n_desc;
        const int4 m = piece ? __ldg(a.pieces + (b - n_desc)) : __ldg(a.desc + b);
        const bool ov = piece || m.x > a.db;
        const int32_t R = ov ? 1 : (m.w & 0xffff);      // rows of the descriptor (<= 32)
        const int32_t d = ov ? m.w : m.x;               // nonzeros per row (chunk / piece size if ov)
        const int32_t slot = PIECES ? -1 - m.x : 0;     // a piece's partial row
        // per-row data, one row per lane: where the row's entries start in the caller's
        // colidx / vals (P:295 step (3) row-pointer update), and its output row
        int32_t rso_l = 0, dst_l = 0;
        if (lane < R) {
            if (piece) {
                rso_l = m.y;
            } else {
                rso_l = __ldg(a.rso + m.z + lane);
                if (ov)
                    rso_l += m.y - __ldg(a.srp + m.z);  // chunk offset inside the row
                else
                    dst_l = __ldg(a.perm + m.z + lane);
            }
        }
        int K = 1;                                       // combined warps per row
        while (2 * K * R <= G) K *= 2;
        f8 acc;
        acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (K == 1) {
            // ---- whole rows per combined warp: sub-warp s owns rows s, s+G, s+2G, ... and
            // streams their entries back to back (so short rows keep U gathers in flight),
            // flushing the accumulator at every row boundary (all rows have d entries, so the
            // boundaries are warp-uniform).
            const int32_t T = ((R + G - 1) / G) * d;              // sub-warp 0's entries (bound)
            const int32_t Ts = act && s < R ? ((R - s + G - 1) / G) * d : 0;
            int32_t c, cn;
            float v, vn;
            auto pair = [&](int32_t t, int32_t& cc, float& vv) {  // entry t of this sub-warp
                const int32_t ri = t / d;
                const int32_t e = __shfl_sync(0xffffffffu, rso_l, min(s + ri * G, 31)) + (t - ri * d);
                cc = 0;
                vv = 0.f;
                if (t < Ts) {
                    cc = __ldg(a.cols + e);
                    vv = __ldg(a.vals + e);
                }
            };
            pair(li, c, v);
            int32_t left = d, rowi = 0;
            for (int32_t base = 0; base < T; base += L) {        // warp-uniform trip count
                pair(base + L + li, cn, vn);                      // next batch (prefetch)
                const int32_t nb = Ts - base;                     // valid entries in this batch
                const int32_t nbu = min(L, T - base);             // warp-uniform bound
#pragma unroll 1
                for (int q = 0; q < L; q += U) {
                    if (q >= nbu) break;
                    f8 x[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t cu = __shfl_sync(0xffffffffu, c, FULL ? s * L + q + u : (s * L + q + u) & 31);
                        if (q + u < nb && (UDIV || q + u < L))
                            ld8(x[u], a.X + ((int64_t)cu * F + li * 8), KEEP ? 1 : 0);
                        else
                            x[u].a = x[u].b = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const float vu = __shfl_sync(0xffffffffu, v, FULL ? s * L + q + u : (s * L + q + u) & 31);
                        fma8(acc, UDIV || q + u < L ? vu : 0.f, x[u]);
                        if (q + u < nbu && --left == 0) {         // row boundary: store, restart
                            const int32_t r = s + rowi * G;
                            const int32_t o = __shfl_sync(0xffffffffu, dst_l, min(r, 31));
                            if (act && r < R) {
                                if (!ov)
                                    store_row<EPI>(a.Y, o, li * 8, F, d, acc, a.epi);
                                else
                                    st8((piece ? a.piece_partial + (int64_t)slot * F
                                               : a.ovp + (int64_t)(b - a.first_ov) * F) + li * 8, acc);
                            }
                            acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
                            left = d;
                            ++rowi;
                        }
                    }
                }
                c = cn;
                v = vn;
            }
            if (ov && !piece && a.fuse_ov) ov_finish<EPI>(a, m.z, m.x, F, lane, s, li);
            continue;
        }
        // ---- rows split over K combined warps (R <= G/2): contiguous parts, xor-tree merge
        const int NG = G / K;                            // row groups per warp
        const int g = s / K, k = s - g * K;
        const int32_t part = (d + K - 1) / K;            // nonzeros per group member
        const int32_t p0 = k * part;
        const int32_t len_k = max(0, min(d, p0 + part) - p0);
        for (int32_t r0 = 0; r0 < R; r0 += NG) {
            const int32_t r = r0 + g;
            const bool gact = (FULL || g < NG) && r < R;           // idle groups / lanes: no work
            const int32_t mylen = gact ? len_k : 0;
            const int32_t e0 = __shfl_sync(0xffffffffu, rso_l, r & 31) + p0;  // first entry
            acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
            // (colidx, val) pairs, L per batch, one per lane; the next batch is prefetched
            int32_t c = 0;
            float v = 0.f;
            if (li < mylen) {
                c = __ldg(a.cols + e0 + li);
                v = __ldg(a.vals + e0 + li);
            }
            for (int32_t base = 0; base < part; base += L) {     // warp-uniform trip count
                const int32_t jn = base + L + li;
                int32_t cn = 0;
                float vn = 0.f;
                if (jn < mylen) {
                    cn = __ldg(a.cols + e0 + jn);
                    vn = __ldg(a.vals + e0 + jn);
                }
                const int32_t nb = mylen - base;                 // valid pairs in this batch (may be <= 0)
                const int32_t nbu = min(L, part - base);         // warp-uniform bound
#pragma unroll 1
                for (int q = 0; q < L; q += U) {
                    if (q >= nbu) break;
                    f8 x[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t cu = __shfl_sync(0xffffffffu, c, FULL ? s * L + q + u : (s * L + q + u) & 31);
                        if (q + u < nb && (UDIV || q + u < L))
                            ld8(x[u], a.X + ((int64_t)cu * F + li * 8), KEEP ? 1 : 0);
                        else
                            x[u].a = x[u].b = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const float vu = __shfl_sync(0xffffffffu, v, FULL ? s * L + q + u : (s * L + q + u) & 31);
                        fma8(acc, UDIV || q + u < L ? vu : 0.f, x[u]);
                    }
                }
                c = cn;
                v = vn;
            }
            // combine the K partial rows of a group (fixed tree: deterministic).  Power-of-two
            // L: xor butterflies; otherwise member k adds member k + o's partial (member 0
            // ends with ((p0 + p1) + (p2 + p3)) ..., the same order as the butterfly).
            if (POW2) {
                for (int o = L; o < K * L; o <<= 1) {
                    acc.a.x = shfl_xor_add(acc.a.x, o);
                    acc.a.y = shfl_xor_add(acc.a.y, o);
                    acc.a.z = shfl_xor_add(acc.a.z, o);
                    acc.a.w = shfl_xor_add(acc.a.w, o);
                    acc.b.x = shfl_xor_add(acc.b.x, o);
                    acc.b.y = shfl_xor_add(acc.b.y, o);
                    acc.b.z = shfl_xor_add(acc.b.z, o);
                    acc.b.w = shfl_xor_add(acc.b.w, o);
                }
            } else {
                for (int o = L; o < K * L; o <<= 1) {
                    acc.a.x += __shfl_down_sync(0xffffffffu, acc.a.x, o);
                    acc.a.y += __shfl_down_sync(0xffffffffu, acc.a.y, o);
                    acc.a.z += __shfl_down_sync(0xffffffffu, acc.a.z, o);
                    acc.a.w += __shfl_down_sync(0xffffffffu, acc.a.w, o);
                    acc.b.x += __shfl_down_sync(0xffffffffu, acc.b.x, o);
                    acc.b.y += __shfl_down_sync(0xffffffffu, acc.b.y, o);
                    acc.b.z += __shfl_down_sync(0xffffffffu, acc.b.z, o);
                    acc.b.w += __shfl_down_sync(0xffffffffu, acc.b.w, o);
                }
            }
            const int32_t rd = __shfl_sync(0xffffffffu, dst_l, r & 31);
            if (k == 0 && gact) {
                if (!ov)
                    store_row<EPI>(a.Y, rd, li * 8, F, d, acc, a.epi);
                else
                    st8((piece ? a.piece_partial + (int64_t)slot * F
                               : a.ovp + (int64_t)(b - a.first_ov) * F) + li * 8, acc);
            }
        }
        if (ov && !piece && a.fuse_ov) ov_finish<EPI>(a, m.z, m.x, F, lane, s, li);
    }
    if (a.zero_last) zero_rows();
}

template <int L, int U, int MINB, bool KEEP, bool PIECES, bool EPI>
void launch_t(const WideArgs& a, cudaStream_t s) {
    auto kern = k_spmm_wide<L, U, MINB, KEEP, PIECES, EPI>;
    static int occ = -1;
    if (occ < 0) {
        AGCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
        if (occ < 1) occ = 1;
    }
    const int G = 32 / (L ? L : a.L);
    const int64_t work = std::max<int64_t>(a.n_desc + (a.pieces ? a.piece_cap : 0), (a.n_zero + G - 1) / G);
    const int64_t want = (work + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * occ));
    kern<<<(unsigned)grid, kThreads, 0, s>>>(a);
    post_launch();
}

int env_int(const char* name, int dflt) {  // experiment switch
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <int L, int U, int MINB, bool EPI>
void launch_e(const WideArgs& a, bool keep, cudaStream_t s) {
    if (a.pieces)
        keep ? launch_t<L, U, MINB, true, true, EPI>(a, s) : launch_t<L, U, MINB, false, true, EPI>(a, s);
    else
        keep ? launch_t<L, U, MINB, true, false, EPI>(a, s) : launch_t<L, U, MINB, false, false, EPI>(a, s);
}

template <int L, int U, int MINB>
void launch_k(const WideArgs& a, bool keep, cudaStream_t s) {
    if (a.epi.active())
        launch_e<L, U, MINB, true>(a, keep, s);
    else
        launch_e<L, U, MINB, false>(a, keep, s);
}

template <int L>
void launch(const WideArgs& a, bool keep, cudaStream_t s) {
    // register budget vs rows in flight (AGCN_WIDE_VARIANT, A/B only; profiles/r01k_wide_ab.md,
    // r01bc_kernel_shapes.md; the measured-and-dropped shapes -- U 4 at 4 CTAs/SM with spills,
    // U 2 at 5 CTAs/SM, U 8 at 2 CTAs/SM -- are no longer instantiated):
    //   0: U 4 at 3 CTAs/SM (80 regs)   4: U 2 at 4 CTAs/SM (64 regs)
    //  -1 (default): 4 for mid-size graphs at F <= 64 (a.lean: C3 F32/F64 -5..9 %), else 0
    static const int venv = env_int("AGCN_WIDE_VARIANT", -1);
    const int variant = venv >= 0 ? venv : (a.lean ? 4 : 0);
    constexpr int U4 = L >= 4 ? 4 : L, U2 = L >= 2 ? 2 : L;
    if (variant == 4)
        launch_k<L, U2, 4>(a, keep, s);
    else
        launch_k<L, U4, 3>(a, keep, s);
}

}  // namespace

bool wide_supported(const agcn_plan_s* p, const float* X, const float* Y, int32_t F) {
    const bool shape = F >= 8 && F <= 256 && F % 8 == 0;   // L = F / 8 lanes of 32 bytes per row
    const bool al = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 31u) == 0;
    return shape && al && p->mbw <= 32;
}

void launch_wide(agcn_plan_s* p, const float* vals, const float* X, int32_t F, float* Y,
                 bool l2_keep, bool blocked, bool fuse_ov, const Epi& epi, cudaStream_t s) {
    const ColSched& cs = p->sched;
    WideArgs a{p->desc, blocked ? p->nb_small : p->nblocks, p->nb_small, p->n_zero, p->cols,
               p->sorted_rowptr, p->row_src_off, p->perm, vals + p->rp_base, X, Y, p->ov_partial,
               p->deg_bound, blocked ? cs.seg : nullptr, blocked ? cs.slot_base + p->n_ov : nullptr,
               blocked ? cs.partial : nullptr, blocked ? cs.cap : 0, epi};
    AGCN_CHECK(a.n_desc + a.piece_cap < (1ll << 31), AGCN_ERR_OVERFLOW, "too many descriptors");
    a.L = F / 8;
    static const int zero_last = env_int("AGCN_ZERO_LAST", 1);  // C5 -1 %, C3/C4 even (profiles r01bj)
    a.zero_last = zero_last;
    a.fuse_ov = fuse_ov && !blocked && p->n_ov > 0 && p->ov_cnt != nullptr;
    a.ov_cs = p->ov_chunk_start;
    a.ov_cnt = p->ov_cnt;
    a.ov_start = p->ov_start;
    {   // nnz per resident warp of the default shape: mid-size graphs (C3: 328) are latency-
        // bound with few descriptors per warp, where 32 warps/SM at U 2 win (profiles r01bl)
        const double share = (double)p->nnz / ((double)num_sms() * 24.0);
        a.lean = F <= 64 && share >= 100.0 && share <= 4000.0;
    }
    switch (F) {
        case 8: launch<1>(a, l2_keep, s); break;
        case 16: launch<2>(a, l2_keep, s); break;
        case 32: launch<4>(a, l2_keep, s); break;
        case 64: launch<8>(a, l2_keep, s); break;
        case 128: launch<16>(a, l2_keep, s); break;
        case 256: launch<32>(a, l2_keep, s); break;
        default: {  // F = 8 L, L not a power of two: one kernel with L at run time
            static const int minb = env_int("AGCN_WIDE_RT_MINB", 3);
            minb == 2 ? launch_k<0, 4, 2>(a, l2_keep, s) : launch_k<0, 4, 3>(a, l2_keep, s);
            break;
        }
    }
}

}  // namespace agcn
