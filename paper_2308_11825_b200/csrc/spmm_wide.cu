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
//  * column indices come from the plan's copy of colidx and vals from the caller's array, both
//    indexed like the caller's CSR (a sorted row starts at row_src_off), one batch of pairs
//    ahead (prefetch), through the read-only path (ld.global.nc).
//  * X residency in L2 (agcn_l2_hint_t, template XM): 0 plain loads; 1 evict_last on every X
//    row (X fits in L2); 2 the plan's hot columns (-1 - slot) read the compact hot buffer Xh --
//    under the launch's persisting access-policy window in HOT_WINDOW mode; 3 as 2 with hot
//    loads evict_last and cold loads evict_first.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

struct f8 {
    float4 a, b;
};

// X-row slice loads bypass L1 allocation (L1::no_allocate): the gathered rows are not reused
// from L1 (hit rate ~1 %), and not allocating them keeps the CSR stream's lines, which the next
// batch of the same warp reads again, resident (C5 -2 %, C3 / C4 neutral; profiles/r02ba_*).
__device__ __forceinline__ void ld8(f8& r, const float* p, int hint) {
    // hint: 0 plain, 1 evict_last (hot), 2 evict_first (cold)
    if (hint == 1)
        asm("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else if (hint == 2)
        asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else
        asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
}

// acc += v * x over 8 floats as four packed fp32x2 FMAs (FFMA2, sm_100): per element the same
// fma.rn as a scalar FFMA (bitwise identical results), half the FMA instructions
__device__ __forceinline__ void fma8(f8& acc, float v, const f8& x) {
    asm("{\n\t.reg .b64 vv, a0, a1, a2, a3, x0, x1, x2, x3;\n\t"
        "mov.b64 vv, {%8, %8};\n\t"
        "mov.b64 a0, {%0, %1};\n\tmov.b64 a1, {%2, %3};\n\t"
        "mov.b64 a2, {%4, %5};\n\tmov.b64 a3, {%6, %7};\n\t"
        "mov.b64 x0, {%9, %10};\n\tmov.b64 x1, {%11, %12};\n\t"
        "mov.b64 x2, {%13, %14};\n\tmov.b64 x3, {%15, %16};\n\t"
        "fma.rn.f32x2 a0, vv, x0, a0;\n\tfma.rn.f32x2 a1, vv, x1, a1;\n\t"
        "fma.rn.f32x2 a2, vv, x2, a2;\n\tfma.rn.f32x2 a3, vv, x3, a3;\n\t"
        "mov.b64 {%0, %1}, a0;\n\tmov.b64 {%2, %3}, a1;\n\t"
        "mov.b64 {%4, %5}, a2;\n\tmov.b64 {%6, %7}, a3;\n\t}"
        : "+f"(acc.a.x), "+f"(acc.a.y), "+f"(acc.a.z), "+f"(acc.a.w), "+f"(acc.b.x), "+f"(acc.b.y),
          "+f"(acc.b.z), "+f"(acc.b.w)
        : "f"(v), "f"(x.a.x), "f"(x.a.y), "f"(x.a.z), "f"(x.a.w), "f"(x.b.x), "f"(x.b.y), "f"(x.b.z),
          "f"(x.b.w));
}

// (a 256-bit st.global.cs.v8.f32 here measured -0.2 % but broke the in-kernel level-3 merge's
// reads of the partial rows -- parity failures on C2 / C3, profiles/r02bb: not used)
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
    const int32_t* cols;  // the plan's colidx copy, indexed like vals (hot columns -1 - slot)
    const int32_t* srp;   // sorted rowptr
    const int32_t* rso;   // row_src_off
    const int32_t* perm;  // sorted -> original row
    const float* vals;    // caller vals, offset by rowptr[0]
    const float* X;
    const float* Xh;      // hot rows [n_hot][F] (XM >= 2)
    float* Y;
    float* ovp;           // oversized partial rows [ov_chunks][F]
    const int32_t* ov_order;  // execution order of the oversized chunks, or NULL (descriptor order)
    int32_t db;           // deg_bound
    Epi epi;              // output epilogue (EPI)
    int32_t L;            // lanes per X row (F / 8); used when the kernel's LT is 0
    int32_t fuse_ov;      // level 3 of rows of <= kHeavyChunks chunks done by the last warp
    const int32_t* ov_cs; // [n_ov + 1] first chunk of oversized row k
    int32_t* ov_cnt;      // [n_ov] chunks of row k finished (zero between launches)
    int64_t ov_start;     // sorted position of the first oversized row
    int32_t zero_in_chunks;  // k_spmm_chunks writes the degree-0 rows (k_spmm_wide then skips them)
};

// one X-row slice of 8 floats for column code c (XM: see the file comment)
template <int XM>
__device__ __forceinline__ void ldx8(f8& r, const WideArgs& a, int32_t c, int32_t F, int li) {
    // (XM 0 / 1 keep the c < 0 test although it is never true there: the same code shape as the
    // hot modes, which ptxas allocates without spills at 80 registers)
    if (c < 0) {
        ld8(r, a.Xh + ((int64_t)(-1 - c) * F + li * 8), XM == 3 ? 1 : 0);
    } else {
        ld8(r, a.X + ((int64_t)c * F + li * 8), XM == 1 ? 1 : (XM == 3 ? 2 : 0));
    }
}


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
// (register budget), XM: X residency mode (file comment).
// LT = 0: L is a runtime value (a.L), for the F = 8 L with L not a power of two.
template <int LT, int U, int MINB, int XM, bool EPI>
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

    // degree-0 rows: Y row = 0 (reading Q16); 32 rows per warp step, one perm load per lane,
    // after the descriptors (the stores fill the tail left by the last, longest descriptors;
    // C5 -1 %, profiles/r01bj_zero_rows_last.md)
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

    const int32_t n_desc = (int32_t)a.n_desc;
    for (int32_t b0 = gw; b0 < n_desc; b0 += W) {
        // the oversized chunks [first_ov, n_desc) run in the plan's execution order
        const int32_t b = a.ov_order && b0 >= a.first_ov ? (int32_t)a.first_ov + __ldg(a.ov_order + (b0 - a.first_ov)) : b0;
        const int4 m = __ldg(a.desc + b);
        const bool ov = m.x > a.db;
        const int32_t R = ov ? 1 : (m.w & 0xffff);      // rows of the descriptor (<= 32)
        const int32_t d = ov ? m.w : m.x;               // nonzeros per row (chunk size if ov)
        // per-row data, one row per lane: where the row's entries start in the caller's vals
        // (P:295 step (3) row-pointer update), and its output row
        int32_t rso_l = 0, dst_l = 0;
        if (lane < R) {
            rso_l = __ldg(a.rso + m.z + lane);
            if (ov)
                rso_l += m.y - __ldg(a.srp + m.z);  // chunk offset inside the row
            else
                dst_l = __ldg(a.perm + m.z + lane);
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
            // t / d through a float reciprocal: exact here ((t + 0.5) / d is >= 0.5 / d away from an
            // integer and t < 2^15, so the rounding error of the product, < (t + 0.5) / d * 2^-22,
            // cannot cross it)
            const float rd = __frcp_rn((float)d);
            auto pair = [&](int32_t t, int32_t& cc, float& vv) {  // entry t of this sub-warp
                const int32_t ri = __float2int_rz(__fmul_rn((float)t + 0.5f, rd));
                const int32_t j = t - ri * d, r = s + ri * G;     // row r of the descriptor
                const int32_t e = __shfl_sync(0xffffffffu, rso_l, min(r, 31)) + j;
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
                            ldx8<XM>(x[u], a, cu, F, li);
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
                                    st8(a.ovp + (int64_t)(b - a.first_ov) * F + li * 8, acc);
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
            if (ov && a.fuse_ov) ov_finish<EPI>(a, m.z, m.x, F, lane, s, li);
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
            const int32_t e0 = __shfl_sync(0xffffffffu, rso_l, r & 31) + p0;  // first entry (vals)
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
                            ldx8<XM>(x[u], a, cu, F, li);
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
                    st8(a.ovp + (int64_t)(b - a.first_ov) * F + li * 8, acc);
            }
        }
        if (ov && a.fuse_ov) ov_finish<EPI>(a, m.z, m.x, F, lane, s, li);
    }
    zero_rows();
}

// 32 degree-0 rows (sorted positions [32 zb, 32 zb + 32)) written as zero rows of Y, one per
// combined warp and step (reading Q16)
template <int L>
__device__ __forceinline__ void zero_batch(const WideArgs& a, int64_t zb, int lane, int s, int li) {
    constexpr int G = 32 / L, F = 8 * L;
    const int64_t r0 = zb * 32;
    if (r0 >= a.n_zero) return;
    const int32_t pr = r0 + lane < a.n_zero ? __ldg(a.perm + r0 + lane) : -1;
    f8 z;
    z.a = z.b = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int i = 0; i < 32; i += G) {
        const int32_t o = __shfl_sync(0xffffffffu, pr, i + s);
        if (o >= 0) st8(a.Y + (int64_t)o * F + li * 8, z);
    }
}

// The oversized-row chunks {deg, loc, row, nnz <= deg_bound} on their own: all G
// combined warps of a warp split one chunk into contiguous parts (the main kernel's R = 1 case,
// same split and the same xor-tree merge, so bitwise the same partial rows) with nothing else
// live -- no row boundaries, no epilogue, no output-row bookkeeping -- so the register budget
// goes to occupancy: U rows in flight per lane at MINB CTAs of 8 warps per SM.  Level 3 (the
// chunk partials summed in order) stays with k_ov_reduce_h.
template <int L, int U, int MINB, int XM>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_chunks(const __grid_constant__ WideArgs a) {
    constexpr int G = 32 / L;
    constexpr int F = 8 * L;
    const int lane = threadIdx.x & 31;
    const int s = lane / L, li = lane % L;
    const int32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int32_t W = gridDim.x * kWarps;
    const int32_t nch = (int32_t)(a.n_desc - a.first_ov);
    for (int32_t i0 = gw; i0 < nch; i0 += W) {
        const int32_t i = a.ov_order ? __ldg(a.ov_order + i0) : i0;   // the plan's execution order
        const int4 m = __ldg(a.desc + a.first_ov + i);
        const int32_t len = m.w;
        const int32_t vb = __ldg(a.rso + m.z) + (m.y - __ldg(a.srp + m.z));  // chunk start in vals
        const int32_t part = (len + G - 1) / G;
        const int32_t p0 = s * part;
        const int32_t mylen = max(0, min(len - p0, part));
        const int32_t vbb = vb + p0;
        f8 acc;
        acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
        int32_t c = 0;
        float v = 0.f;
        if (li < mylen) {
            c = __ldg(a.cols + vbb + li);
            v = __ldg(a.vals + vbb + li);
        }
        for (int32_t base = 0; base < part; base += L) {  // warp-uniform trip count
            const int32_t jn = base + L + li;
            int32_t cn = 0;
            float vn = 0.f;
            if (jn < mylen) {
                cn = __ldg(a.cols + vbb + jn);
                vn = __ldg(a.vals + vbb + jn);
            }
            const int32_t nb = mylen - base;
            const int32_t nbu = min(L, part - base);
#pragma unroll 1
            for (int q = 0; q < L; q += U) {
                if (q >= nbu) break;
                f8 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int32_t cu = __shfl_sync(0xffffffffu, c, s * L + q + u);
                    if (q + u < nb)
                        ldx8<XM>(x[u], a, cu, F, li);
                    else
                        x[u].a = x[u].b = make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) fma8(acc, __shfl_sync(0xffffffffu, v, s * L + q + u), x[u]);
            }
            c = cn;
            v = vn;
        }
#pragma unroll
        for (int o = L; o < 32; o <<= 1) {
            acc.a.x = shfl_xor_add(acc.a.x, o);
            acc.a.y = shfl_xor_add(acc.a.y, o);
            acc.a.z = shfl_xor_add(acc.a.z, o);
            acc.a.w = shfl_xor_add(acc.a.w, o);
            acc.b.x = shfl_xor_add(acc.b.x, o);
            acc.b.y = shfl_xor_add(acc.b.y, o);
            acc.b.z = shfl_xor_add(acc.b.z, o);
            acc.b.w = shfl_xor_add(acc.b.w, o);
        }
        if (s == 0) st8(a.ovp + (int64_t)i * F + li * 8, acc);
        // the degree-0 rows, one batch of 32 after every chunk: their DRAM writes overlap this
        // kernel's L2-bound gathers instead of forming a write-bound tail of k_spmm_wide
        if (a.zero_in_chunks) zero_batch<L>(a, (int64_t)i0, lane, s, li);
    }
    if (a.zero_in_chunks)
        for (int64_t zb = (int64_t)nch + gw; zb * 32 < a.n_zero; zb += W) zero_batch<L>(a, zb, lane, s, li);
}

// launch `kern` on a persistent grid (SMs x occupancy, capped by the work) with the hot
// buffer under a persisting L2 access-policy window when win > 0 (launch attribute)
template <class K>
void launch_grid(K kern, int& occ, int64_t work_warps, const WideArgs& a, size_t win, cudaStream_t s) {
    if (occ <= 0) {
        AGCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
        if (occ < 1) occ = 1;
    }
    const int64_t want = (work_warps + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * occ));
    if (win == 0) {
        kern<<<(unsigned)grid, kThreads, 0, s>>>(a);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(kThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeAccessPolicyWindow;
        at[0].val.accessPolicyWindow.base_ptr = const_cast<float*>(a.Xh);
        at[0].val.accessPolicyWindow.num_bytes = win;
        at[0].val.accessPolicyWindow.hitRatio = 1.0f;
        at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        AGCN_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    }
    post_launch();
}

int dev_index() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < 64 ? dev : 0;
}

template <int L, int U, int MINB, int XM, bool EPI>
void launch_t(const WideArgs& a, size_t win, cudaStream_t s) {
    static int occ[64] = {};  // per device; a benign race (every thread computes the same value)
    const int G = 32 / (L ? L : a.L);
    launch_grid(k_spmm_wide<L, U, MINB, XM, EPI>, occ[dev_index()], std::max<int64_t>(a.n_desc, (a.n_zero + G - 1) / G),
                a, win, s);
}

template <int L, int U, int MINB, int XM>
void launch_c(const WideArgs& a, size_t win, cudaStream_t s) {
    static int occ[64] = {};
    launch_grid(k_spmm_chunks<L, U, MINB, XM>, occ[dev_index()], a.n_desc - a.first_ov, a, win, s);
}

// the chunk kernel's shapes (agcn_spmm_opts_t.chunk_shape)
template <int L, int XM>
void launch_chunks(const WideArgs& a, int shape, size_t win, cudaStream_t s) {
    constexpr int U4 = L >= 4 ? 4 : L, U2 = L >= 2 ? 2 : L;
    if (shape == 3)
        launch_c<L, U4, 3, XM>(a, win, s);
    else if (shape == 6)
        launch_c<L, U2, 6, XM>(a, win, s);
    else
        launch_c<L, U4, 4, XM>(a, win, s);
}

template <int L, int U, int MINB, int XM>
void launch_e(const WideArgs& a, size_t win, cudaStream_t s) {
    if (a.epi.active())
        launch_t<L, U, MINB, XM, true>(a, win, s);
    else
        launch_t<L, U, MINB, XM, false>(a, win, s);
}

// register budget vs rows in flight (profiles/r01k_wide_ab.md, r01bc_kernel_shapes.md,
// r01bl_auto_shape.md): U 4 at 3 CTAs/SM (80 registers) by default; U 2 at 4 CTAs/SM (64
// registers) for mid-size graphs at F <= 64 (lean: C3 F32/F64 -5..9 %).  Hot-row plans (large
// graphs) always take the default shape.
template <int L>
void launch(const WideArgs& a, int xm, bool lean, size_t win, int chunks, cudaStream_t s) {
    constexpr int U4 = L >= 4 ? 4 : (L ? L : 4), U2 = L >= 2 ? 2 : (L ? L : 2);
    if (L && chunks) {  // the oversized chunks first, then the rest (n_desc = nb_small)
        switch (xm) {
            case 0: launch_chunks<L ? L : 1, 0>(a, chunks, 0, s); break;
            case 1: launch_chunks<L ? L : 1, 1>(a, chunks, 0, s); break;
            case 2: launch_chunks<L ? L : 1, 2>(a, chunks, win, s); break;
            default: launch_chunks<L ? L : 1, 3>(a, chunks, win, s); break;
        }
    }
    WideArgs b = a;
    if (L && chunks) {
        b.n_desc = a.first_ov;
        if (a.zero_in_chunks) b.n_zero = 0;   // written by k_spmm_chunks
    }
    switch (xm) {
        case 0: lean ? launch_e<L, U2, 4, 0>(b, 0, s) : launch_e<L, U4, 3, 0>(b, 0, s); break;
        case 1: lean ? launch_e<L, U2, 4, 1>(b, 0, s) : launch_e<L, U4, 3, 1>(b, 0, s); break;
        case 2: launch_e<L, U4, 3, 2>(b, win, s); break;
        default: launch_e<L, U4, 3, 3>(b, win, s); break;
    }
}

}  // namespace

bool wide_supported(const agcn_plan_s* p, const float* X, const float* Y, int32_t F) {
    const bool shape = F >= 8 && F <= 256 && F % 8 == 0;   // L = F / 8 lanes of 32 bytes per row
    const bool al = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 31u) == 0;
    return shape && al && p->mbw <= 32;
}

void launch_wide(agcn_plan_s* p, const float* vals, const float* X, const float* Xh, int32_t F, float* Y,
                 int l2, size_t win, bool fuse_ov, int chunk_shape, bool chunk_order, const Epi& epi,
                 cudaStream_t s) {
    WideArgs a{p->desc, p->nblocks, p->nb_small, p->n_zero, p->cols_copy, p->sorted_rowptr, p->row_src_off,
               p->perm, vals + p->rp_base, X, Xh, Y, p->ov_partial, chunk_order ? p->ov_order : nullptr,
               p->deg_bound, epi};
    AGCN_CHECK(a.n_desc < (1ll << 31), AGCN_ERR_OVERFLOW, "too many descriptors");
    a.L = F / 8;
    a.fuse_ov = fuse_ov && p->n_ov > 0 && p->ov_cnt != nullptr;
    a.ov_cs = p->ov_chunk_start;
    a.ov_cnt = p->ov_cnt;
    a.ov_start = p->ov_start;
    // X residency mode: plans with hot rows always decode hot columns (2, or 3 with hints)
    const int xm = p->n_hot > 0 ? (l2 == AGCN_L2_HOT_HINTS ? 3 : 2) : (l2 == AGCN_L2_KEEP_ALL ? 1 : 0);
    if (xm < 2) win = 0;
    // nnz per resident warp of the default shape: mid-size graphs (C3: 328) are latency-
    // bound with few descriptors per warp, where 32 warps/SM at U 2 win (profiles r01bl)
    const double share = (double)p->nnz / ((double)num_sms() * 24.0);
    const bool lean = F <= 64 && share >= 100.0 && share <= 4000.0;
    // the chunk kernel: plans whose oversized chunks are not merged in-kernel (level 3 by
    // k_ov_reduce_h), power-of-two L
    // auto: F >= 32 (C4 F128 -13 %; since the X loads skip L1 (r02ba) also C5 F64 -2.3 %, C5 F32
    // -2.9 %, C4 F64 -4.4 %, profiles/r02be_chunk_kernel.txt; F < 32 not measured)
    const int chunks = (!a.fuse_ov && p->ov_chunks > 0 && chunk_shape >= 0 && (chunk_shape || F >= 32))
                           ? (chunk_shape ? chunk_shape : 4) : 0;
    a.zero_in_chunks = chunks && (F & (F - 1)) == 0 && !epi.active();
    switch (F) {
        case 8: launch<1>(a, xm, lean, win, chunks, s); break;
        case 16: launch<2>(a, xm, lean, win, chunks, s); break;
        case 32: launch<4>(a, xm, lean, win, chunks, s); break;
        case 64: launch<8>(a, xm, lean, win, chunks, s); break;
        case 128: launch<16>(a, xm, lean, win, chunks, s); break;
        case 256: launch<32>(a, xm, lean, win, chunks, s); break;
        default: launch<0>(a, xm, false, win, 0, s); break;  // F = 8 L, L not a power of two (run-time L)
    }
}

}  // namespace agcn
