// spmm.cu -- agcn_spmm: Y = A.X over the block-level partition (Accel-GCN section III-D).
//
// Mapping on sm_100a:
//  * One 128-bit descriptor {deg, loc, row, info} is the unit of work.  A
//    persistent grid of 8-warp CTAs walks the descriptor array; each WARP owns one
//    descriptor at a time (the paper gives one CTA of max_block_warps warps; on B200 the
//    block-level merge then needs no CTA barrier, see below).
//  * Combined warp: the F columns of one X row are covered by L consecutive
//    lanes with float4 loads (L*T float4 = the paper's round_dim, lanes past F truncated,
//    P:493); a warp holds G = 32/L such "combined warps" (sub-warps), which split the
//    descriptor's contiguous nonzeros evenly (per-sub-warp nnz differ by at most 4).
//  * The descriptor's colidx (the plan's copy) and vals (the caller's array), one contiguous
//    run per row at row_src_off, are staged in shared memory once per descriptor.  Hot columns
//    (-1 - slot) read the plan's compact hot rows.
//  * Three-level accumulation made deterministic: (1) registers, (2) the
//    partial rows of sub-warps that share a row are merged in fixed sub-warp order through
//    shared memory (replaces atomicAdd_block), (3) rows with degree > deg_bound are split
//    into chunks whose partial sums go to a scratch buffer and are summed in chunk order by
//    a second kernel (replaces global atomics).
//  * Rows are restored to the original order in the store: Y[perm[row]] (reading S:142-150).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kWarpsPerCta = 8;
constexpr double kL2KeepBytes = 128.0 * 1024 * 1024;  // X up to ~L2 size gets evict_last hints

constexpr int kCtaThreads = kWarpsPerCta * 32;

template <bool V4>
struct VecT;
template <>
struct VecT<true> {
    using T = float4;
};
template <>
struct VecT<false> {
    using T = float;
};

__device__ __forceinline__ float4 vzero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vzero(float4& a) { a = vzero4(); }
__device__ __forceinline__ void vzero(float& a) { a = 0.f; }
__device__ __forceinline__ void vfma(float4& a, float v, const float4& x) {
    a.x = fmaf(v, x.x, a.x);
    a.y = fmaf(v, x.y, a.y);
    a.z = fmaf(v, x.z, a.z);
    a.w = fmaf(v, x.w, a.w);
}
__device__ __forceinline__ void vfma(float& a, float v, float x) { a = fmaf(v, x, a); }
__device__ __forceinline__ void vadd(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}
__device__ __forceinline__ void vadd(float& a, float b) { a += b; }

// X-row gather loads (read-only path); with keep, an L2 evict_last cache-policy hint (X fits
// in L2).  pol comes from policy_evict_last().
__device__ __forceinline__ float4 ldx(const float4* p, bool keep, uint64_t pol) {
    float4 v;
    if (keep)
        asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
            : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    else
        v = __ldg(p);
    return v;
}
__device__ __forceinline__ float ldx(const float* p, bool keep, uint64_t pol) {
    float v;
    if (keep)
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else
        v = __ldg(p);
    return v;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// Y / partial stores: streaming (written once)
__device__ __forceinline__ void sty(float4* p, const float4& v) { __stcs(p, v); }
__device__ __forceinline__ void sty(float* p, float v) { __stcs(p, v); }
// CSR streams: read once (evict-first)
__device__ __forceinline__ int32_t ldcs_i(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float ldcs_f(const float* p) { return __ldcs(p); }

struct BlockArgs {
    const int4* desc;
    int64_t nblocks;
    int64_t first_ov;       // descriptor index of the first oversized chunk (== nb_small)
    int32_t db;             // deg_bound
    int32_t stage;          // shared-memory entries per warp (>= db + 8, multiple of 4)
    int32_t rso_stage;      // shared-memory row offsets per warp (>= max_block_warps)
    const int32_t* cols;    // the plan's colidx copy, indexed like vals (hot columns -1 - slot)
    const int32_t* srp;     // sorted rowptr
    const int32_t* rso;     // row_src_off
    const int32_t* perm;    // sorted -> original row
    const float* vals;      // caller vals, already offset by rowptr[0]
    const float* X;
    const float* Xh;        // hot rows [n_hot][FV] (plans with hot rows)
    float* Y;
    float* ovp;             // oversized partials [ov_chunks][FV]
    int64_t n_zero;         // sorted rows [0, n_zero) have degree 0
    int32_t FV;             // vectors per row (F/4 on the float4 path, F otherwise)
    int32_t keep;           // X loads with an L2 evict_last hint
};

template <int L, int T, bool V4, int U>
__global__ void __launch_bounds__(kCtaThreads, 4) k_spmm_block(const __grid_constant__ BlockArgs a) {
    using VT = typename VecT<V4>::T;
    constexpr int G = 32 / L;
    static_assert(U % 4 == 0, "U must be a multiple of 4 (LDS.128 of staged colidx / vals)");
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = lane / L, li = lane % L;
    int32_t* s_col = reinterpret_cast<int32_t*>(smem) + warp * (2 * a.stage + a.rso_stage);
    float* s_val = reinterpret_cast<float*>(s_col + a.stage);
    int32_t* s_rso = s_col + 2 * a.stage;
    VT* s_part = reinterpret_cast<VT*>(smem + (size_t)kWarpsPerCta * (2 * a.stage + a.rso_stage) * 4) +
                 warp * (G * 2 * T * L);
    const VT* __restrict__ X = reinterpret_cast<const VT*>(a.X);
    const VT* __restrict__ XH = reinterpret_cast<const VT*>(a.Xh);
    VT* __restrict__ Y = reinterpret_cast<VT*>(a.Y);
    VT* __restrict__ OVP = reinterpret_cast<VT*>(a.ovp);
    const int32_t FV = a.FV;
    const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + warp;
    const int64_t W = (int64_t)gridDim.x * kWarpsPerCta;
    const bool keep = a.keep;
    const uint64_t pol = policy_evict_last();

    // degree-0 rows: Y row = 0 (reading Q16)
    for (int64_t r = gw * G + s; r < a.n_zero; r += W * G) {
        const int64_t orow = a.perm[r];
        VT z;
        vzero(z);
        for (int32_t c = li; c < FV; c += L) sty(Y + orow * FV + c, z);
    }

    int4 m_next = gw < a.nblocks ? __ldg(a.desc + gw) : make_int4(0, 0, 0, 0);
    for (int64_t b = gw; b < a.nblocks; b += W) {
        const int4 m = m_next;
        if (b + W < a.nblocks) m_next = __ldg(a.desc + b + W);  // prefetch the next descriptor
        const bool ov = m.x > a.db;
        const int32_t d = m.x, loc = m.y, row0 = m.z;
        const int32_t R = ov ? 1 : (m.w & 0xffff);
        const int32_t total = ov ? m.w : R * d;
        const int32_t seg = ov ? total : d;  // row-segment length inside the descriptor

        // ---- stage colidx / vals of the descriptor in shared memory.  Rows are read from the
        // caller's CSR through row_src_off (the O(n) row-pointer update of P:295 (3)).
        __syncwarp();
        int32_t vbase0 = 0;
        if (ov) {
            vbase0 = __ldg(a.rso + row0) + (loc - __ldg(a.srp + row0));
        } else {
            for (int32_t r = lane; r < R; r += 32) s_rso[r] = __ldg(a.rso + row0 + r);
            __syncwarp();
        }
#pragma unroll 4
        for (int32_t e = lane; e < total; e += 32) {
            int32_t off;
            if (ov) {
                off = vbase0 + e;
            } else {
                const int32_t r = e / d;
                off = s_rso[r] + (e - r * d);
            }
            s_col[e] = ldcs_i(a.cols + off);
            s_val[e] = ldcs_f(a.vals + off);
        }
        __syncwarp();

        // ---- even split of [0, total) over the G sub-warps (multiples of 4 entries)
        const int32_t Q = (((total + G - 1) / G) + 3) & ~3;
        const int32_t q0 = min(s * Q, total), q1 = min(q0 + Q, total);

        for (int32_t cc = 0; cc < FV; cc += T * L) {
            VT acc[T];
#pragma unroll
            for (int t = 0; t < T; ++t) vzero(acc[t]);
            int32_t rs = (q0 / seg) * seg;  // current row segment [rs, re)
            int32_t re = rs + seg;
            bool fin = false;               // this sub-warp finishes a row begun earlier
            int32_t fin_rs = 0;

            auto store_row = [&](int32_t rstart, VT* v) {
                VT* dst;
                if (ov)
                    dst = OVP + (b - a.first_ov) * (int64_t)FV;
                else
                    dst = Y + (int64_t)a.perm[row0 + rstart / seg] * FV;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const int32_t c = cc + li + t * L;
                    if (c < FV) sty(dst + c, v[t]);
                }
            };

            for (int32_t q = q0; q < q1; q += U) {
                int32_t col[U];
                float val[U];
#pragma unroll
                for (int u = 0; u < U; u += 4) {
                    const int4 c4 = *reinterpret_cast<const int4*>(s_col + q + u);
                    const float4 v4 = *reinterpret_cast<const float4*>(s_val + q + u);
                    col[u] = c4.x; col[u + 1] = c4.y; col[u + 2] = c4.z; col[u + 3] = c4.w;
                    val[u] = v4.x; val[u + 1] = v4.y; val[u + 2] = v4.z; val[u + 3] = v4.w;
                }
                VT xv[U][T];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool ok = q + u < q1;
                    const VT* xr = col[u] >= 0 ? X + (int64_t)col[u] * FV : XH + (int64_t)(-1 - col[u]) * FV;
#pragma unroll
                    for (int t = 0; t < T; ++t) {
                        const int32_t c = cc + li + t * L;
                        if (ok && c < FV)
                            xv[u][t] = ldx(xr + c, keep, pol);
                        else
                            vzero(xv[u][t]);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (q + u < q1) {
#pragma unroll
                        for (int t = 0; t < T; ++t) vfma(acc[t], val[u], xv[u][t]);
                        if (q + u + 1 == re) {  // row segment ends inside this range
                            if (rs >= q0) {
                                store_row(rs, acc);  // whole row is ours
                            } else {                 // head partial: we finish the row
#pragma unroll
                                for (int t = 0; t < T; ++t) s_part[(s * 2 + 0) * T * L + t * L + li] = acc[t];
                                fin = true;
                                fin_rs = rs;
                            }
#pragma unroll
                            for (int t = 0; t < T; ++t) vzero(acc[t]);
                            rs = re;
                            re += seg;
                        }
                    }
                }
            }
            // range ended inside a row: tail partial (row began here) or middle partial
            if (q1 > q0 && q1 > rs && q1 < re) {
                const int slot = rs >= q0 ? 1 : 0;
#pragma unroll
                for (int t = 0; t < T; ++t) s_part[(s * 2 + slot) * T * L + t * L + li] = acc[t];
            }
            __syncwarp();
            if (fin) {  // sum the row's partials in sub-warp order: tail, middles, own head
                const int s_first = fin_rs / Q;
                VT sum[T];
#pragma unroll
                for (int t = 0; t < T; ++t) sum[t] = s_part[(s_first * 2 + 1) * T * L + t * L + li];
                for (int s2 = s_first + 1; s2 <= s; ++s2) {
#pragma unroll
                    for (int t = 0; t < T; ++t) vadd(sum[t], s_part[(s2 * 2 + 0) * T * L + t * L + li]);
                }
                store_row(fin_rs, sum);
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ float shfl_vt(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ float4 shfl_vt(float4 v, int src) {
    return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                       __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

__device__ __forceinline__ void fanout_v(const Epi& e, int64_t vec_off, const float4& v) {
    fanout4(e, 4 * vec_off, v);  // vec_off counts float4 vectors
}
__device__ __forceinline__ void fanout_v(const Epi& e, int64_t off, float v) { fanout1(e, off, v); }

__device__ __forceinline__ float4 epi_v(float4 y, int32_t deg, int64_t orow, int32_t c, const Epi& e) {
    return epi4(y, deg, orow, 4 * c, e);  // c counts float4 vectors
}
__device__ __forceinline__ float epi_v(float y, int32_t deg, int64_t orow, int32_t c, const Epi& e) {
    return epi1(y, deg, orow, c, e);
}

// Output epilogue as its own pass (kernels without the fused one), in place on Y, for rows
// [k0, k1): sorted rows (perm != NULL, degree from the sorted rowptr) or original rows
// (perm == NULL, degree from rp).  One thread per element.
__global__ void k_epilogue(float* __restrict__ Y, int64_t k0, int64_t k1, int32_t F,
                           const int32_t* __restrict__ perm, const int32_t* __restrict__ rp, const Epi epi) {
    const int64_t total = (k1 - k0) * (int64_t)F;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = k0 + i / F;
        const int32_t c = (int32_t)(i % F);
        const int64_t orow = perm ? perm[k] : k;
        float* y = Y + orow * F + c;
        const float v = epi1(*y, rp[k + 1] - rp[k], orow, c, epi);
        *y = v;
        fanout1(epi, orow * F + c, v);
    }
}

// Level-3 merge (deterministic), sized to the chunk counts (C5: median 3 chunks per oversized row, the
// heaviest 633).  Oversized rows sit in ascending degree order, so the n_heavy rows with more
// than kHeavyChunks chunks are the suffix: CTAs [0, n_heavy) take one of them each, heaviest
// first, with all 256 threads; the other CTAs take 8 rows each, one warp per row.  Lane or
// thread (g, c) sums chunks c0+g, c0+g+NG, ... of vector column c into its own accumulator in
// chunk order; the NG group sums are then added in group order (shuffles / shared memory).
// Every summation order is a function of the plan alone: deterministic.
constexpr int kReduceWarps = 8;
constexpr int64_t kFuseOvMaxChunks = 16384;  // fused level 3 up to this many oversized chunks
template <bool V4>
__global__ void __launch_bounds__(kReduceWarps * 32) k_ov_reduce_h(
    const float* __restrict__ ovp_f, const int32_t* __restrict__ chunk_start,
    const int32_t* __restrict__ perm, int64_t ov_start, int64_t n_ov, int64_t n_heavy,
    float* __restrict__ Y_f, int32_t FV, const int32_t* __restrict__ srp, const Epi epi) {
    using VT = typename VecT<V4>::T;
    const VT* ovp = reinterpret_cast<const VT*>(ovp_f);
    VT* Y = reinterpret_cast<VT*>(Y_f);
    const bool cta = blockIdx.x < n_heavy;
    const int nthr = cta ? kReduceWarps * 32 : 32;
    const int t = cta ? threadIdx.x : (threadIdx.x & 31);
    const int64_t k = cta ? n_ov - 1 - blockIdx.x
                          : (int64_t)(blockIdx.x - n_heavy) * kReduceWarps + (threadIdx.x >> 5);
    if (!cta && k >= n_ov - n_heavy) return;   // whole warps only: no CTA barrier below
    __shared__ VT part[kReduceWarps * 32];
    const int32_t c0 = chunk_start[k], c1 = chunk_start[k + 1];
    const int64_t orow = perm[ov_start + k];
    const int FVc = FV < nthr ? FV : nthr;   // vector columns per pass
    const int NG = nthr / FVc;               // chunk groups
    const int g = t / FVc, cl = t - g * FVc;
    for (int32_t cb = 0; cb < FV; cb += FVc) {
        const int32_t c = cb + cl;
        VT acc;
        vzero(acc);
        if (g < NG && c < FV) {
            int32_t j = c0 + g;
            for (; j + 3 * NG < c1; j += 4 * NG) {
                const VT x0 = ovp[(int64_t)j * FV + c], x1 = ovp[(int64_t)(j + NG) * FV + c];
                const VT x2 = ovp[(int64_t)(j + 2 * NG) * FV + c], x3 = ovp[(int64_t)(j + 3 * NG) * FV + c];
                vadd(acc, x0);
                vadd(acc, x1);
                vadd(acc, x2);
                vadd(acc, x3);
            }
            for (; j < c1; j += NG) vadd(acc, ovp[(int64_t)j * FV + c]);
        }
        if (cta) {
            part[t] = acc;
            __syncthreads();
            if (g == 0) {
                for (int gg = 1; gg < NG; ++gg) vadd(acc, part[gg * FVc + cl]);
            }
            __syncthreads();
        } else {
            for (int gg = 1; gg < NG; ++gg) {  // group 0 adds groups 1.. in order
                const VT o = shfl_vt(acc, cl + gg * FVc);
                if (g == 0) vadd(acc, o);
            }
        }
        if (g == 0 && c < FV) {
            if (epi.active()) acc = epi_v(acc, srp[ov_start + k + 1] - srp[ov_start + k], orow, c, epi);
            sty(Y + orow * FV + c, acc);
            if (epi.npeer) fanout_v(epi, orow * FV + c, acc);
        }
    }
}

// ---------------------------------------------------------------- ablation arm (Fig. 3(b))
struct WarpArgs {
    const int4* tasks;
    int64_t ntasks;
    const int32_t* rp;      // rowptr rebased to 0
    const int32_t* ci;      // colidx copy (rebased)
    const float* vals;      // caller vals offset by rowptr[0]
    const float* X;
    float* Y;               // zeroed before the launch
    int32_t FV;
};

__device__ __forceinline__ void vatomic(float4* p, const float4& v) { atomicAdd(p, v); }
__device__ __forceinline__ void vatomic(float* p, float v) { atomicAdd(p, v); }

// One warp-level task {row, col, len} per combined warp (sub-warp of L lanes); rows that
// span several tasks are merged with global atomics (GNNAdvisor-style).
template <int L, int T, bool V4, int U>
__global__ void __launch_bounds__(kCtaThreads) k_spmm_warp(const WarpArgs a) {
    using VT = typename VecT<V4>::T;
    constexpr int G = 32 / L;
    const int lane = threadIdx.x & 31, s = lane / L, li = lane % L;
    const VT* __restrict__ X = reinterpret_cast<const VT*>(a.X);
    VT* __restrict__ Y = reinterpret_cast<VT*>(a.Y);
    const int64_t gs = ((int64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5)) * G + s;
    const int64_t S = (int64_t)gridDim.x * kWarpsPerCta * G;
    const int32_t FV = a.FV;
    for (int64_t t = gs; t < a.ntasks; t += S) {
        const int4 task = __ldg(a.tasks + t);
        const int32_t row = task.x, len = task.z;
        const int32_t start = a.rp[row] + task.y;
        const bool whole = len == a.rp[row + 1] - a.rp[row];
        for (int32_t cc = 0; cc < FV; cc += T * L) {
            VT acc[T];
#pragma unroll
            for (int i = 0; i < T; ++i) vzero(acc[i]);
            for (int32_t q = 0; q < len; q += U) {
                int32_t col[U];
                float val[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool ok = q + u < len;
                    col[u] = ok ? __ldg(a.ci + start + q + u) : 0;
                    val[u] = ok ? __ldg(a.vals + start + q + u) : 0.f;
                }
                VT xv[U][T];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int i = 0; i < T; ++i) {
                        const int32_t c = cc + li + i * L;
                        if (q + u < len && c < FV)
                            xv[u][i] = ldx(X + (int64_t)col[u] * FV + c, false, 0);
                        else
                            vzero(xv[u][i]);
                    }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int i = 0; i < T; ++i) vfma(acc[i], val[u], xv[u][i]);
            }
#pragma unroll
            for (int i = 0; i < T; ++i) {
                const int32_t c = cc + li + i * L;
                if (c < FV) {
                    if (whole)
                        sty(Y + (int64_t)row * FV + c, acc[i]);
                    else
                        vatomic(Y + (int64_t)row * FV + c, acc[i]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- dispatch
struct Shape {
    int L, T;
};

// Combined-warp shape: L lanes (power of two) x T vectors per lane cover FV vectors in one
// pass if FV <= 128 (fewest lane slots, then fewest vectors per lane); wider rows loop over
// column chunks of 32 x 4 vectors.
Shape pick_shape(int32_t FV) {
    if (FV > 128) return {32, 4};
    Shape best{32, 4};
    int best_slots = 1 << 30;
    for (int T = 1; T <= 4; ++T)
        for (int L = 1; L <= 32; L <<= 1)
            if (L * T >= FV) {
                int slots = L * T;
                if (slots < best_slots) {
                    best_slots = slots;
                    best = {L, T};
                }
                break;
            }
    return best;
}

void launch_epilogue(float* Y, int64_t k0, int64_t k1, int32_t F, const int32_t* perm, const int32_t* rp,
                     const Epi& epi, cudaStream_t s) {
    if (k1 <= k0) return;
    const int64_t total = (k1 - k0) * (int64_t)F;
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_epilogue<<<grid, 256, 0, s>>>(Y, k0, k1, F, perm, rp, epi);
    post_launch();
}

// After an SpMM that read the hot buffer under a persisting window: drop its lines from L2
// (discard.global.L2: invalidate without write-back -- the buffer is re-gathered by every call),
// so they do not keep occupying the persisting set-aside for whatever runs next.
__global__ void k_l2_discard(const float* __restrict__ p, int64_t lines) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < lines; i += (int64_t)gridDim.x * blockDim.x)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + i * 32) : "memory");
}

// Per-device launch facts (a process may drive several devices): SM count and, per kernel
// instantiation and shared-memory size, the occupancy after the shared-memory opt-in.
constexpr int kMaxDev = 64;
int cur_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDev ? dev : 0;
}

template <class K>
int occupancy(K kern, int threads, size_t smem, size_t optin) {
    static std::mutex mu;
    static int occ[kMaxDev] = {};
    static size_t occ_smem[kMaxDev] = {};
    const int dev = cur_device();
    std::lock_guard<std::mutex> lock(mu);
    if (occ[dev] <= 0 || occ_smem[dev] != smem) {
        if (optin) AGCN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)optin));
        AGCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev], kern, threads, smem));
        if (occ[dev] < 1) occ[dev] = 1;
        occ_smem[dev] = smem;
    }
    return occ[dev];
}

template <int L, int T, bool V4, int U>
void launch_block_u(const BlockArgs& a, cudaStream_t s, size_t smem) {
    auto kern = k_spmm_block<L, T, V4, U>;
    const int occ = occupancy(kern, kCtaThreads, smem, 200 * 1024);
    const int64_t work = std::max<int64_t>(a.nblocks, (a.n_zero + 31) / 32);
    const int64_t want = (work + kWarpsPerCta - 1) / kWarpsPerCta;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * occ));
    kern<<<(unsigned)grid, kCtaThreads, smem, s>>>(a);
    post_launch();
}

// X-row loads in flight per lane: 4 (register budget; U 8 at one vector per lane measured no
// better, r01).
template <int L, int T, bool V4>
void launch_block(const BlockArgs& a, cudaStream_t s, size_t smem) {
    launch_block_u<L, T, V4, 4>(a, s, smem);
}

template <int L, int T, bool V4>
void launch_warp(const WarpArgs& a, cudaStream_t s) {
    auto kern = k_spmm_warp<L, T, V4, 4>;
    const int occ = occupancy(kern, kCtaThreads, 0, 0);
    constexpr int G = 32 / L;
    const int64_t want = (a.ntasks + kWarpsPerCta * G - 1) / (kWarpsPerCta * G);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * occ));
    kern<<<(unsigned)grid, kCtaThreads, 0, s>>>(a);
    post_launch();
}

// Xh[k] = X[hot_cols[k]] for k < H: the hot rows (the H highest-degree vertices) in a compact
// buffer; one thread per 16-byte vector of the flattened [H][F / 4] output (fully coalesced
// stores, row-contiguous loads), 4 vectors in flight per thread; scalar lanes when F % 4 != 0
template <bool V4>
__global__ void k_gather_hot(const float* __restrict__ X, const int32_t* __restrict__ hot_cols,
                             int64_t H, int32_t F, float* __restrict__ Xh) {
    const int32_t FV = V4 ? F / 4 : F;
    const int64_t total = H * FV, T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 4 * T) {
        if (V4) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = i0 + u * T;
                if (i < total) {
                    const int64_t k = i / FV, c = i - k * FV;
                    v[u] = __ldg(reinterpret_cast<const float4*>(X + (int64_t)__ldg(hot_cols + k) * F) + c);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * T < total) reinterpret_cast<float4*>(Xh)[i0 + u * T] = v[u];
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = i0 + u * T;
                if (i < total) {
                    const int64_t k = i / FV, c = i - k * FV;
                    Xh[i] = __ldg(X + (int64_t)__ldg(hot_cols + k) * F + c);
                }
            }
        }
    }
}

#define AGCN_DISPATCH_LT(SHAPE, FN, ...)                                             \
    do {                                                                             \
        switch ((SHAPE).L * 8 + (SHAPE).T) {                                         \
            case 1 * 8 + 1: FN<1, 1>(__VA_ARGS__); break;                            \
            case 1 * 8 + 2: FN<1, 2>(__VA_ARGS__); break;                            \
            case 1 * 8 + 3: FN<1, 3>(__VA_ARGS__); break;                            \
            case 1 * 8 + 4: FN<1, 4>(__VA_ARGS__); break;                            \
            case 2 * 8 + 1: FN<2, 1>(__VA_ARGS__); break;                            \
            case 2 * 8 + 2: FN<2, 2>(__VA_ARGS__); break;                            \
            case 2 * 8 + 3: FN<2, 3>(__VA_ARGS__); break;                            \
            case 2 * 8 + 4: FN<2, 4>(__VA_ARGS__); break;                            \
            case 4 * 8 + 1: FN<4, 1>(__VA_ARGS__); break;                            \
            case 4 * 8 + 2: FN<4, 2>(__VA_ARGS__); break;                            \
            case 4 * 8 + 3: FN<4, 3>(__VA_ARGS__); break;                            \
            case 4 * 8 + 4: FN<4, 4>(__VA_ARGS__); break;                            \
            case 8 * 8 + 1: FN<8, 1>(__VA_ARGS__); break;                            \
            case 8 * 8 + 2: FN<8, 2>(__VA_ARGS__); break;                            \
            case 8 * 8 + 3: FN<8, 3>(__VA_ARGS__); break;                            \
            case 8 * 8 + 4: FN<8, 4>(__VA_ARGS__); break;                            \
            case 16 * 8 + 1: FN<16, 1>(__VA_ARGS__); break;                          \
            case 16 * 8 + 2: FN<16, 2>(__VA_ARGS__); break;                          \
            case 16 * 8 + 3: FN<16, 3>(__VA_ARGS__); break;                          \
            case 16 * 8 + 4: FN<16, 4>(__VA_ARGS__); break;                          \
            case 32 * 8 + 1: FN<32, 1>(__VA_ARGS__); break;                          \
            case 32 * 8 + 2: FN<32, 2>(__VA_ARGS__); break;                          \
            case 32 * 8 + 3: FN<32, 3>(__VA_ARGS__); break;                          \
            case 32 * 8 + 4: FN<32, 4>(__VA_ARGS__); break;                          \
            default: throw Error{AGCN_ERR_CUDA, "internal: bad combined-warp shape"}; \
        }                                                                            \
    } while (0)

template <int L, int T>
void block_v4(const BlockArgs& a, cudaStream_t s, size_t smem) { launch_block<L, T, true>(a, s, smem); }
template <int L, int T>
void block_v1(const BlockArgs& a, cudaStream_t s, size_t smem) { launch_block<L, T, false>(a, s, smem); }
template <int L, int T>
void warp_v4(const WarpArgs& a, cudaStream_t s) { launch_warp<L, T, true>(a, s); }
template <int L, int T>
void warp_v1(const WarpArgs& a, cudaStream_t s) { launch_warp<L, T, false>(a, s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int num_sms() {
    static std::atomic<int> sms[kMaxDev] = {};
    const int dev = cur_device();
    int v = sms[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

size_t ensure_persisting_l2(size_t bytes) {
    static std::mutex mu;
    static size_t set[kMaxDev] = {};
    static int maxp[kMaxDev] = {}, maxw[kMaxDev] = {};
    const int dev = cur_device();
    std::lock_guard<std::mutex> lock(mu);
    if (maxp[dev] == 0) {
        if (cudaDeviceGetAttribute(&maxp[dev], cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess) maxp[dev] = -1;
        if (cudaDeviceGetAttribute(&maxw[dev], cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess) maxw[dev] = 0;
        cudaGetLastError();
    }
    if (maxp[dev] <= 0 || maxw[dev] <= 0) return 0;
    bytes = std::min<size_t>(bytes, std::min<size_t>((size_t)maxp[dev], (size_t)maxw[dev]));
    if (set[dev] < bytes) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        set[dev] = bytes;
    }
    return bytes;
}

// default hot budget: the device's maximum persisting-L2 size
static size_t max_persisting_l2() {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, cur_device()) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return v > 0 ? (size_t)v : 0;
}

void spmm_launch(agcn_plan_s* p, const float* vals, const float* X, int32_t F, float* Y,
                 cudaStream_t s, const agcn_spmm_opts_t& o) {
    if (p->n == 0) return;
    const bool foreign = s != p->stream && !p->capturing;  // (capture: the plan is complete)
    if (foreign) {  // plan built on another stream: wait for it; remember this use for destroy
        AGCN_CUDA(cudaStreamWaitEvent(s, p->ready, 0));
        if (!p->last_use) AGCN_CUDA(cudaEventCreateWithFlags(&p->last_use, cudaEventDisableTiming));
    }
    struct Rec {  // record last_use after the launches below, on every exit path
        agcn_plan_s* p; cudaStream_t s; bool on;
        ~Rec() { if (on) cudaEventRecord(p->last_use, s); }
    } rec{p, s, foreign};
    // LOOPED (ablation 2, Fig. 4(a) / Table II): no combined warp -- one warp of 32 scalar lanes
    // walks the columns of a row in strides of 32
    Epi epi{o.self_scale != 0.f ? o.self : nullptr, o.bias, o.self_scale,
            o.aggregation == AGCN_AGG_MEAN, o.relu != 0, F, o.npeer, {}};
    for (int q = 0; q < o.npeer; ++q) epi.peer[q] = o.peer_out[q];
    const bool looped = o.kernel == AGCN_KERNEL_LOOPED;
    const bool v4 = !looped && (F % 4 == 0) && aligned16(X) && aligned16(Y);
    const int32_t FV = v4 ? F / 4 : F;
    const Shape sh = looped ? Shape{32, 1} : pick_shape(FV);
    if (p->partition == AGCN_PARTITION_WARP) {
        AGCN_CUDA(cudaMemsetAsync(Y, 0, sizeof(float) * (size_t)p->n * F, s));
        if (p->ntasks > 0) {
            WarpArgs a{p->tasks, p->ntasks, p->rowptr_copy, p->cols_copy, vals + p->rp_base, X, Y, FV};
            if (v4)
                AGCN_DISPATCH_LT(sh, warp_v4, a, s);
            else
                AGCN_DISPATCH_LT(sh, warp_v1, a, s);
        }
        if (epi.active()) launch_epilogue(Y, 0, p->n, F, nullptr, p->rowptr_copy, epi, s);
        return;
    }
    // kernel choice (agcn_spmm_opts_t): WIDE when applicable, else GENERAL
    const bool wide_ok = wide_supported(p, X, Y, F);
    int kernel = o.kernel;
    if (kernel == AGCN_KERNEL_AUTO) kernel = wide_ok ? AGCN_KERNEL_WIDE : AGCN_KERNEL_GENERAL;
    if (kernel == AGCN_KERNEL_LOOPED) kernel = AGCN_KERNEL_GENERAL;  // with the {32 lanes, scalar} shape
    AGCN_CHECK(kernel == AGCN_KERNEL_WIDE || kernel == AGCN_KERNEL_GENERAL, AGCN_ERR_INVALID_ARG,
               "unknown kernel");
    AGCN_CHECK(kernel != AGCN_KERNEL_WIDE || wide_ok, AGCN_ERR_UNSUPPORTED,
               "WIDE kernel needs F = 8 L <= 256, 32-byte aligned X/Y, max_block_warps <= 32");
    // oversized-row partial buffer of the paper's chunks (grows, stream-ordered)
    const size_t need = (size_t)p->ov_chunks * (size_t)F;
    // scratch captured by a graph (agcn_graph_create) must not move under it
    AGCN_CHECK(p->n_graphs.load() == 0 || (need <= p->ov_partial_floats &&
                                           (size_t)p->n_hot * (size_t)F <= p->xhot_floats),
               AGCN_ERR_UNSUPPORTED,
               "a CUDA graph of this plan holds its scratch: a larger F needs agcn_graph_destroy first "
               "(or create the graph with the largest F)");
    if (need > p->ov_partial_floats) {
        if (p->ov_partial) AGCN_CUDA(cudaFreeAsync(p->ov_partial, s));
        p->ov_partial = nullptr;
        p->ov_partial_floats = 0;
        AGCN_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p->ov_partial), need * sizeof(float), s));
        p->ov_partial_floats = need;
    }
    // hot X rows (agcn_opts_t.hot_rows): gathered into the plan's compact buffer every call
    // (X changes between calls), read by the kernels for columns encoded -1 - slot
    if (p->n_hot > 0) {
        const size_t hneed = (size_t)p->n_hot * (size_t)F;
        if (hneed > p->xhot_floats) {
            if (p->xhot) AGCN_CUDA(cudaFreeAsync(p->xhot, s));
            p->xhot = nullptr;
            p->xhot_floats = 0;
            AGCN_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p->xhot), hneed * sizeof(float), s));
            p->xhot_floats = hneed;
        }
        const int64_t vec = p->n_hot * (v4 ? F / 4 : F);
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((vec + 1023) / 1024, (int64_t)num_sms() * 8));
        if (v4)
            k_gather_hot<true><<<g, 256, 0, s>>>(X, p->hot_cols, p->n_hot, F, p->xhot);
        else
            k_gather_hot<false><<<g, 256, 0, s>>>(X, p->hot_cols, p->n_hot, F, p->xhot);
        post_launch();
    }
    // L2 residency of X (agcn_l2_hint_t)
    const double x_bytes = 4.0 * (double)p->x_rows * F;
    int l2 = o.l2_hint;
    // auto: evict_last on all of X when it fits in L2; plans with hot rows: the compact hot
    // buffer with evict_last hot / evict_first cold loads (C5 -1.8 % against plain loads, 3 x 3
    // runs, profiles/r02z_l2_modes.txt); otherwise plain loads.  The persisting window measured
    // slower in the bench flow (C5 3.57 vs 3.27 ms; it changes a device-wide limit) -- opt-in.
    if (l2 == AGCN_L2_AUTO)
        l2 = p->n_hot > 0 ? AGCN_L2_HOT_HINTS : (x_bytes <= kL2KeepBytes ? AGCN_L2_KEEP_ALL : AGCN_L2_NONE);
    AGCN_CHECK(l2 >= AGCN_L2_NONE && l2 <= AGCN_L2_HOT_HINTS, AGCN_ERR_INVALID_ARG, "unknown l2_hint");
    if ((l2 == AGCN_L2_HOT_WINDOW || l2 == AGCN_L2_HOT_HINTS) && p->n_hot == 0) l2 = AGCN_L2_NONE;
    size_t win = 0;
    if (l2 == AGCN_L2_HOT_WINDOW) {
        const size_t budget = o.hot_mb > 0 ? (size_t)o.hot_mb << 20 : max_persisting_l2();
        win = ensure_persisting_l2(std::min(budget, sizeof(float) * p->xhot_floats));
        if (win == 0) l2 = AGCN_L2_NONE;
    }
    BlockArgs a;
    a.desc = p->desc;
    a.nblocks = p->nblocks;
    a.first_ov = p->nb_small;
    a.db = p->deg_bound;
    a.stage = ((p->deg_bound + 3) & ~3) + 8;
    a.rso_stage = (p->mbw + 3) & ~3;
    a.cols = p->cols_copy;
    a.srp = p->sorted_rowptr;
    a.rso = p->row_src_off;
    a.perm = p->perm;
    a.vals = vals + p->rp_base;
    a.X = X;
    a.Xh = p->xhot;
    a.Y = Y;
    a.ovp = p->ov_partial;
    a.n_zero = p->n_zero;
    a.FV = FV;
    const size_t elt = v4 ? sizeof(float4) : sizeof(float);
    const size_t smem = (size_t)kWarpsPerCta * ((2 * a.stage + a.rso_stage) * 4 + 64 * sh.T * elt);
    a.keep = l2 == AGCN_L2_KEEP_ALL;
    // level 3 of the oversized rows of <= kHeavyChunks chunks fused into the WIDE kernel when
    // there are few chunks (saves the reduction launch on small graphs: C2 -4..7 %, C3 -7 %;
    // with C5's 201K chunks the per-chunk fence + counter costs more than the launch: +3 %;
    // profiles/r01bk_fused_level3.md)
    const bool fuse = kernel == AGCN_KERNEL_WIDE && p->n_ov > 0 && p->ov_chunks <= kFuseOvMaxChunks;
    if (fuse && !p->ov_cnt) {
        p->ov_cnt = dalloc<int32_t>(p->n_ov, s);
        AGCN_CUDA(cudaMemsetAsync(p->ov_cnt, 0, sizeof(int32_t) * p->n_ov, s));
    }
    if (kernel == AGCN_KERNEL_WIDE)
    {
        launch_wide(p, vals, X, p->xhot, F, Y, l2, win, fuse, o.chunk_shape, o.chunk_order == 0, epi, s);  // epilogue fused
        if (win > 0) {
            const int64_t lines = (int64_t)((win + 127) / 128);
            k_l2_discard<<<(unsigned)std::min<int64_t>((lines + 255) / 256, (int64_t)num_sms() * 8), 256, 0, s>>>(
                p->xhot, lines);
            post_launch();
        }
    }
    else if (v4)
        AGCN_DISPATCH_LT(sh, block_v4, a, s, smem);
    else
        AGCN_DISPATCH_LT(sh, block_v1, a, s, smem);
    if (kernel != AGCN_KERNEL_WIDE && epi.active())  // rows of degree <= deg_bound
        launch_epilogue(Y, 0, p->ov_start, F, p->perm, p->sorted_rowptr, epi, s);
    if (p->n_ov > 0 && !(fuse && p->n_ov_heavy == 0)) {  // level 3: fixed-order sums of partial rows
        const float* part = p->ov_partial;
        const int32_t* slots = p->ov_chunk_start;
        const int64_t nh = p->n_ov_heavy;
        // fused: only the heavy rows (CTAs [0, nh) of the kernel) are left
        const unsigned hgrid = fuse ? (unsigned)nh
                                    : (unsigned)(nh + (p->n_ov - nh + kReduceWarps - 1) / kReduceWarps);
        if (v4)
            k_ov_reduce_h<true><<<hgrid, kReduceWarps * 32, 0, s>>>(part, slots, p->perm, p->ov_start, p->n_ov,
                                                                   nh, Y, FV, p->sorted_rowptr, epi);
        else
            k_ov_reduce_h<false><<<hgrid, kReduceWarps * 32, 0, s>>>(part, slots, p->perm, p->ov_start,
                                                                    p->n_ov, nh, Y, FV, p->sorted_rowptr, epi);
        post_launch();
    }
}

}  // namespace agcn
