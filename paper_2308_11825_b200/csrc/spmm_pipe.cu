// spmm_pipe.cu -- SpMM kernel with an asynchronous shared-memory gather pipeline
// (AGCN_KERNEL_PIPE), F in {32, 64, 128, 256}.
//
// Same work decomposition, results contract and summation order as k_spmm_wide
// (spmm_wide.cu): one 128-bit descriptor {deg, loc, row, info} per warp at a
// time, a "combined warp" of L = F/8 lanes per X row moving 32 bytes per lane,
// G = 32/L combined warps per warp, rows of a descriptor round-robin over groups of K
// combined warps with a fixed xor-tree merge (level 2 of P:526-530), partial rows of the
// deg_bound chunks of oversized rows summed by k_ov_reduce (level 3).
//
// What changes is how the X rows travel (and which columns a lane owns: 2 x 16 bytes, one
// in each half of the row, so that each 16-byte cp.async of a combined warp is one
// contiguous half row).  k_spmm_wide holds U = 4 rows in flight per lane in
// registers (80 registers, 24 warps per SM: 96 KB of gathers in flight per SM), and is bound
// by that: the SpMM is a latency-bound gather (profiles/r01l_*).  Here every lane copies its
// 32-byte slice of an X row straight into a per-warp shared-memory ring with cp.async
// (LDGSTS, L2 only), NS - 1 entries ahead of the FMA that consumes it, so the rows in flight
// live in shared memory, not registers: NS = 8 stages x 1 KB per warp, 24 warps per SM ->
// 168 KB in flight per SM.  Rows past the end of a stream are zero-filled by cp.async itself
// (src-size 0), so the steady-state loop has no branches around the copies.
//
// Each combined warp walks ONE stream of entries: its rows (or its part of a row, K > 1),
// back to back; the accumulator is flushed every `seg` entries (warp-uniform).  The
// (colidx, val) pairs of the stream are read L at a time, one per lane, three batches deep
// (current, next, prefetch) and broadcast with shuffles.
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

struct PipeArgs {
    const int4* desc;
    int64_t nblocks;
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
};

__device__ __forceinline__ void cp16(uint32_t saddr, const void* g, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float4 lds4(uint32_t saddr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
    return v;
}

__device__ __forceinline__ void fma4(float4& a, float v, const float4& x) {
    a.x = fmaf(v, x.x, a.x);
    a.y = fmaf(v, x.y, a.y);
    a.z = fmaf(v, x.z, a.z);
    a.w = fmaf(v, x.w, a.w);
}

__device__ __forceinline__ float xadd(float v, int o) { return v + __shfl_xor_sync(0xffffffffu, v, o); }

// L lanes per X row (F = 8 L), NS pipeline stages (NS - 1 <= L), MINB CTAs per SM.
template <int L, int NS, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_pipe(const __grid_constant__ PipeArgs a) {
    constexpr int G = 32 / L;
    constexpr int F = 8 * L;
    static_assert(NS >= 2 && NS - 1 <= L, "the issue point must stay within the next pair batch");
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int s = lane / L, li = lane % L;
    const int warp = threadIdx.x >> 5;
    const int32_t gw = blockIdx.x * kWarps + warp;
    const int32_t W = gridDim.x * kWarps;
    // ring: [NS stages][2 halves][32 lanes][16 B]  (LDS.128 phases of 8 lanes: conflict-free)
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + warp * (NS * 1024) + lane * 16;
    // lane li owns columns [4 li, 4 li + 4) and [4 L + 4 li, 4 L + 4 li + 4) of a row: each
    // of the two 16-byte copies of a combined warp then covers one contiguous half row
    const float* __restrict__ Xl = a.X + li * 4;

    // degree-0 rows: Y row = 0 (reading Q16); 32 rows per warp step
    for (int64_t r0 = (int64_t)gw * 32; r0 < a.n_zero; r0 += (int64_t)W * 32) {
        const int32_t pr = r0 + lane < a.n_zero ? __ldg(a.perm + r0 + lane) : -1;
#pragma unroll 4
        for (int i = 0; i < 32; i += G) {
            const int32_t o = __shfl_sync(0xffffffffu, pr, i + s);
            if (o >= 0) {
                float* dst = a.Y + (int64_t)o * F + li * 4;
                __stcs(reinterpret_cast<float4*>(dst), make_float4(0.f, 0.f, 0.f, 0.f));
                __stcs(reinterpret_cast<float4*>(dst + 4 * L), make_float4(0.f, 0.f, 0.f, 0.f));
            }
        }
    }

    const int32_t nblocks = (int32_t)a.nblocks;
    for (int32_t b = gw; b < nblocks; b += W) {
        const int4 m = __ldg(a.desc + b);
        const bool ov = m.x > a.db;
        const int32_t R = ov ? 1 : (m.w & 0xffff);   // rows of the descriptor (<= 32)
        const int32_t d = ov ? m.w : m.x;            // nonzeros per row (chunk size if ov)
        int32_t rso_l = 0, dst_l = 0;                // per row (one per lane): entries, output
        if (lane < R) {
            rso_l = __ldg(a.rso + m.z + lane);
            if (ov)
                rso_l += m.y - __ldg(a.srp + m.z);   // chunk offset inside the row
            else
                dst_l = __ldg(a.perm + m.z + lane);
        }
        int K = 1;                                    // combined warps per row
        while (2 * K * R <= G) K *= 2;
        const int NG = G / K;                         // row groups per warp
        const int g = s / K, k = s - g * K;
        const int32_t seg = (d + K - 1) / K;          // entries per row part (warp-uniform)
        const int32_t p0 = k * seg;
        const int32_t len_k = max(0, min(d, p0 + seg) - p0);
        const int32_t T = ((R + NG - 1) / NG) * seg;  // stream length (warp-uniform)

        // pairs of stream entries [base, base + L), one per lane; c = -1 past the stream's end
        auto pairs = [&](int32_t base, int32_t& c, float& v) {
            const int32_t t = base + li;
            const int32_t ri = t / seg, j = t - ri * seg;
            const int32_t r = g + ri * NG;
            const int32_t rs = __shfl_sync(0xffffffffu, rso_l, min(r, 31));
            c = -1;
            v = 0.f;
            if (t < T && r < R && j < len_k) {
                c = __ldg(a.cols + rs + p0 + j);
                v = __ldg(a.vals + rs + p0 + j);
            }
        };
        // copy the X row slice of entry u (pair batch cb, lane u % L) into stage st
        auto issue = [&](int32_t u, int32_t cb, uint32_t st) {
            const int32_t cu = __shfl_sync(0xffffffffu, cb, s * L + (u & (L - 1)));
            const float* src = cu >= 0 ? Xl + (int64_t)cu * F : Xl;
            const uint32_t nbytes = cu >= 0 ? 16u : 0u;  // 0: zero-fill, nothing read
            cp16(st, src, nbytes);
            cp16(st + 512, src + 4 * L, nbytes);
            cp_commit();
        };
        int32_t c0, c1, c2;  // pair batches: current, next, prefetch
        float v0, v1, v2;
        pairs(0, c0, v0);
        pairs(L, c1, v1);
        pairs(2 * L, c2, v2);
#pragma unroll
        for (int u = 0; u < NS - 1; ++u) issue(u, c0, ring + u * 1024);  // prologue (batch 0)

        float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
        int32_t left = seg;                           // entries left in the current row part
        int32_t ri = 0;                               // current row part
        uint32_t st_c = ring, st_i = ring + (NS - 1) * 1024;  // consume / issue stages
        const uint32_t ring_end = ring + NS * 1024;
        for (int32_t t = 0; t < T; ++t) {
            const int32_t u = t + NS - 1;
            issue(u, (u ^ t) < L ? c0 : c1, st_i);    // u in the current or the next batch
            st_i = st_i + 1024 == ring_end ? ring : st_i + 1024;
            cp_wait<NS - 1>();                        // entry t has landed
            const float vt = __shfl_sync(0xffffffffu, v0, s * L + (t & (L - 1)));
            fma4(acc0, vt, lds4(st_c));
            fma4(acc1, vt, lds4(st_c + 512));
            st_c = st_c + 1024 == ring_end ? ring : st_c + 1024;
            if (--left == 0) {                        // end of a row part: merge, store
                for (int o = L; o < K * L; o <<= 1) {
                    acc0.x = xadd(acc0.x, o); acc0.y = xadd(acc0.y, o);
                    acc0.z = xadd(acc0.z, o); acc0.w = xadd(acc0.w, o);
                    acc1.x = xadd(acc1.x, o); acc1.y = xadd(acc1.y, o);
                    acc1.z = xadd(acc1.z, o); acc1.w = xadd(acc1.w, o);
                }
                const int32_t r = g + ri * NG;
                const int32_t rd = __shfl_sync(0xffffffffu, dst_l, min(r, 31));
                if (k == 0 && r < R) {
                    float* dst = (ov ? a.ovp + (int64_t)(b - a.first_ov) * F : a.Y + (int64_t)rd * F) + li * 4;
                    __stcs(reinterpret_cast<float4*>(dst), acc0);
                    __stcs(reinterpret_cast<float4*>(dst + 4 * L), acc1);
                }
                acc0 = acc1 = make_float4(0.f, 0.f, 0.f, 0.f);
                left = seg;
                ++ri;
            }
            if ((t & (L - 1)) == L - 1) {             // next pair batch
                c0 = c1; v0 = v1;
                c1 = c2; v1 = v2;
                pairs(t + 1 + 2 * L, c2, v2);
            }
        }
        cp_wait<0>();                                 // the trailing (zero-fill) copies
    }
}

template <int L, int NS, int MINB>
void launch_t(const PipeArgs& a, cudaStream_t s) {
    auto kern = k_spmm_pipe<L, NS, MINB>;
    constexpr size_t smem = (size_t)kWarps * NS * 1024;
    static int occ = -1;
    if (occ < 0) {
        AGCN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AGCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
        if (occ < 1) occ = 1;
    }
    constexpr int G = 32 / L;
    const int64_t work = std::max<int64_t>(a.nblocks, (a.n_zero + 32 * G - 1) / (32 * G));
    const int64_t want = (work + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * occ));
    kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
    post_launch();
}

int env_int(const char* name, int dflt) {  // experiment switch (A/B only)
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <int L>
void launch(const PipeArgs& a, cudaStream_t s) {
    // stages x CTAs per SM (AGCN_PIPE_VARIANT): 0: 8 stages, 3 CTAs; 1: 6 stages, 4 CTAs;
    // 2: 4 stages, 6 CTAs
    static const int variant = env_int("AGCN_PIPE_VARIANT", 0);
    constexpr int N8 = L >= 8 ? 8 : L + 1 > 4 ? 4 : L + 1;
    constexpr int N6 = L >= 6 ? 6 : N8;
    constexpr int N4 = L >= 4 ? 4 : N8;
    switch (variant) {
        case 1: launch_t<L, N6, 4>(a, s); break;
        case 2: launch_t<L, N4, 6>(a, s); break;
        default: launch_t<L, N8, 3>(a, s); break;
    }
}

}  // namespace

bool pipe_supported(const agcn_plan_s* p, const float* X, const float* Y, int32_t F) {
    const bool shape = F == 32 || F == 64 || F == 128 || F == 256;
    const bool al = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 31u) == 0;
    return shape && al && p->mbw <= 32;
}

void launch_pipe(agcn_plan_s* p, const float* vals, const float* X, int32_t F, float* Y, cudaStream_t s) {
    PipeArgs a{p->desc, p->nblocks, p->nb_small, p->n_zero, p->cols, p->sorted_rowptr, p->row_src_off,
               p->perm, vals + p->rp_base, X, Y, p->ov_partial, p->deg_bound};
    AGCN_CHECK(p->nblocks < (1ll << 31), AGCN_ERR_OVERFLOW, "too many descriptors");
    switch (F) {
        case 32: launch<4>(a, s); break;
        case 64: launch<8>(a, s); break;
        case 128: launch<16>(a, s); break;
        default: launch<32>(a, s); break;
    }
}

}  // namespace agcn
