// gemm_tc.cu -- Y = X . W on the 5th-generation tensor cores (tcgen05, kind::tf32), for the
// dense half of a GCN layer (X' = sigma(A' (X W))).
//
// The product is skinny -- M = rows of X (up to millions), K = F_in <= 256, N = F_out <= 256 --
// so it is HBM-bound (K*N*2/(4(K+N)) flop per byte), and one CTA per 128-row tile is the whole
// design: TMA (cp.async.bulk.tensor, SWIZZLE_128B) brings the 128 x K tile of X and, once per
// CTA, all of W^T (N x K, K-major) into shared memory; one elected thread issues the
// tcgen05.mma chain (M = 128, N, K in steps of 8) into a TMEM accumulator of N columns;
// tcgen05.commit signals an mbarrier; four warps read their 32 TMEM lanes (tcgen05.ld
// 32x32b) and write the rows, with an optional bias / ReLU.  Several CTAs per SM overlap one
// tile's loads with another's MMA and stores.
//
// Precision: kind::tf32 reads the fp32 operands with a 10-bit mantissa (products exact in the
// fp32 accumulator): |y - y_ref| <= 2^-9 sum_k |x_k w_k| + fp32 accumulation.  agcn_gemm_xw
// documents it; GCNLayer(precision="tf32") opts into it (default: fp32 cuBLAS).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace agcn {
namespace {

constexpr int kGemmThreads = 128;  // 4 warps: one per 32 TMEM lanes (rows) of the 128-row tile
constexpr int kBM = 128;           // rows per tile (UMMA M)
constexpr int kBK = 32;            // fp32 per 128-byte swizzle row (one TMA box / k stage)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row atoms of 1 KB
// stacked along M/N (stride byte offset 1 KB), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);         // start address [0,14)
    d |= (uint64_t)1 << 16;                          // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset [32,46)
    d |= (uint64_t)1 << 46;                          // version [46,48) = 1
    d |= (uint64_t)2 << 61;                          // layout type [61,64): SWIZZLE_128B
    return d;
}

// Instruction descriptor: D = F32, A = B = TF32, both K-major, N, M = 128.
template <int N>
__device__ __forceinline__ uint32_t idesc_tf32() {
    return (1u << 4)                 // c_format F32
           | (2u << 7)               // a_format TF32
           | (2u << 10)              // b_format TF32
           | ((uint32_t)(N >> 3) << 17)
           | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// N output columns (16..256, multiple of 16), KT = ceil(K / 32) k stages (runtime, <= kt_max).
template <int N>
__global__ void __launch_bounds__(kGemmThreads) k_gemm_tf32(const __grid_constant__ CUtensorMap tmX,
                                                           const __grid_constant__ CUtensorMap tmW,
                                                           float* __restrict__ Y, int64_t M, int32_t KT,
                                                           const float* __restrict__ bias, int32_t relu) {
    constexpr uint32_t kTmemCols = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB alignment for SWIZZLE_128B
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* sA = reinterpret_cast<float*>(smem);                                   // [KT][128][32]
    float* sB = reinterpret_cast<float*>(smem + (size_t)KT * kBM * kBK * 4);       // [KT][N][32]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)KT * (kBM + N) * kBK * 4);
    uint64_t* barA = bars;      // X tile landed
    uint64_t* barB = bars + 1;  // W landed (once)
    uint64_t* barM = bars + 2;  // MMA chain done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(barA, 1);
        mbar_init(barB, 1);
        mbar_init(barM, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (threadIdx.x == 0) {  // W^T, all k stages, once per CTA
        mbar_expect_tx(barB, (uint32_t)(KT * N * kBK * 4));
        for (int k = 0; k < KT; ++k) tma_load_2d(sB + (size_t)k * N * kBK, &tmW, barB, k * kBK, 0);
    }
    const int64_t ntiles = (M + kBM - 1) / kBM;
    const bool stage_out = N <= KT * kBK;            // the output tile fits in the X tile's space
    uint32_t phase = 0;
    bool w_ready = false;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, phase ^= 1) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(barA, (uint32_t)(KT * kBM * kBK * 4));
            for (int k = 0; k < KT; ++k)
                tma_load_2d(sA + (size_t)k * kBM * kBK, &tmX, barA, k * kBK, (int)(t * kBM));
            if (!w_ready) {
                mbar_wait(barB, 0);
                w_ready = true;
            }
            mbar_wait(barA, phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t idesc = idesc_tf32<N>();
            for (int k = 0; k < KT; ++k) {
                const uint32_t a0 = smem_u32(sA + (size_t)k * kBM * kBK);
                const uint32_t b0 = smem_u32(sB + (size_t)k * N * kBK);
#pragma unroll
                for (int kk = 0; kk < kBK / 8; ++kk)  // UMMA K = 8 tf32 = 32 bytes
                    umma_tf32(tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                              (k | kk) != 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(barM))
                         : "memory");
        }
        __syncwarp();
        mbar_wait(barM, phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // epilogue: warp w owns TMEM lanes (tile rows) [32 w, 32 w + 32)
        const int r = warp * 32 + lane;                 // row inside the tile
        const int64_t row = t * kBM + r;
        if (stage_out) {
            // the tile's rows are one contiguous block of Y: stage them in shared memory (the
            // consumed X tile; 16-byte chunks XOR-swizzled by row, conflict-free both ways)
            // and write the block out with fully coalesced 16-byte stores
            float4* st = reinterpret_cast<float4*>(sA);
            constexpr int NC = N / 4;                   // 16-byte chunks per row
            constexpr int SW = NC >= 8 ? 7 : NC - 1;
#pragma unroll 1
            for (int c0 = 0; c0 < N; c0 += 16) {
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    if (bias) {
                        o.x += __ldg(bias + c0 + i);
                        o.y += __ldg(bias + c0 + i + 1);
                        o.z += __ldg(bias + c0 + i + 2);
                        o.w += __ldg(bias + c0 + i + 3);
                    }
                    if (relu) {
                        o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                    }
                    const int c4 = (c0 + i) / 4;
                    st[r * NC + (c4 ^ (r & SW))] = o;
                }
            }
            __syncthreads();
            const int64_t rows = M - t * kBM < kBM ? M - t * kBM : (int64_t)kBM;
            float4* dst = reinterpret_cast<float4*>(Y + t * kBM * N);
            for (int q = threadIdx.x; q < rows * NC; q += kGemmThreads) {
                const int rr = q / NC, c4 = q - rr * NC;
                __stcs(dst + q, st[rr * NC + (c4 ^ (rr & SW))]);
            }
        } else {
#pragma unroll 1
            for (int c0 = 0; c0 < N; c0 += 16) {
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
                if (row < M) {
                    float* dst = Y + row * N + c0;
#pragma unroll
                    for (int i = 0; i < 16; i += 4) {
                        float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        if (bias) {
                            o.x += __ldg(bias + c0 + i);
                            o.y += __ldg(bias + c0 + i + 1);
                            o.z += __ldg(bias + c0 + i + 2);
                            o.w += __ldg(bias + c0 + i + 3);
                        }
                        if (relu) {
                            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                        }
                        __stcs(reinterpret_cast<float4*>(dst + i), o);
                    }
                }
            }
        }
        // TMEM and the X tile are reused by the next tile: everyone done reading first
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (threadIdx.x == 0 && !w_ready) mbar_wait(barB, 0);  // never leave a TMA in flight
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

// ---------------------------------------------------------------- pipelined (warp-specialized)
// One persistent CTA per SM streaming 128-row tiles: warp 0 (one lane) keeps NS X tiles in
// flight with TMA; warp 1 (one lane) issues the tcgen05.mma chain of a tile into one of two
// TMEM accumulators and commits it to "tile full" and "stage free" mbarriers; warps 2-5 drain
// the other accumulator (tcgen05.ld, bias / ReLU) and write the rows, so loads, MMAs and
// stores of consecutive tiles overlap inside the CTA.
constexpr int kWsThreads = 192;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int N, int NS, int CWT>
__global__ void __launch_bounds__(kWsThreads, 1) k_gemm_tf32_ws(const __grid_constant__ CUtensorMap tmX,
                                                               const __grid_constant__ CUtensorMap tmW,
                                                               float* __restrict__ Y, int64_t M, int32_t KT,
                                                               const float* __restrict__ bias, int32_t relu) {
    constexpr uint32_t kAcc = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;  // columns per accumulator
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const size_t a_bytes = (size_t)KT * kBM * kBK * 4;        // one X tile (all k stages)
    float* sA = reinterpret_cast<float*>(smem);                // [NS][KT][128][32]
    float* sB = reinterpret_cast<float*>(smem + NS * a_bytes); // [KT][N][32]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * a_bytes + (size_t)KT * N * kBK * 4);
    uint64_t* full = bars;            // [NS] X tile landed
    uint64_t* empty = bars + NS;      // [NS] X tile consumed by the MMAs
    uint64_t* acc_full = bars + 2 * NS;       // [2] accumulator ready
    uint64_t* acc_empty = bars + 2 * NS + 2;  // [2] accumulator drained (4 epilogue warps)
    uint64_t* barB = bars + 2 * NS + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 5);
    // epilogue staging: per epilogue warp 32 rows x CW columns, rows padded to CW + 4 floats
    constexpr int CW = N < CWT ? N : CWT, SP = CW + 4;
    float* staging = reinterpret_cast<float*>(smem + NS * a_bytes + (size_t)KT * N * kBK * 4 + 128);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, 4);
        }
        mbar_init(barB, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * kAcc));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (M + kBM - 1) / kBM;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            mbar_expect_tx(barB, (uint32_t)(KT * N * kBK * 4));
            for (int k = 0; k < KT; ++k) tma_load_2d(sB + (size_t)k * N * kBK, &tmW, barB, k * kBK, 0);
            int st = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(empty + st, ph ^ 1);            // first pass: free
                mbar_expect_tx(full + st, (uint32_t)a_bytes);
                float* dst = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(sA) + st * a_bytes);
                for (int k = 0; k < KT; ++k)
                    tma_load_2d(dst + (size_t)k * kBM * kBK, &tmX, full + st, k * kBK, (int)(t * kBM));
                if (++st == NS) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            mbar_wait(barB, 0);
            const uint32_t idesc = idesc_tf32<N>();
            int st = 0;
            uint32_t ph = 0, aph[2] = {0, 0};
            int acc = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(acc_empty + acc, aph[acc] ^ 1);  // accumulator drained (first use: free)
                mbar_wait(full + st, ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a_base = smem_u32(reinterpret_cast<unsigned char*>(sA) + st * a_bytes);
                for (int k = 0; k < KT; ++k) {
                    const uint32_t a0 = a_base + (uint32_t)(k * kBM * kBK * 4);
                    const uint32_t b0 = smem_u32(sB + (size_t)k * N * kBK);
#pragma unroll
                    for (int kk = 0; kk < kBK / 8; ++kk)
                        umma_tf32(tmem + acc * kAcc, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32),
                                  idesc, (k | kk) != 0);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(empty + st))
                             : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(acc_full + acc))
                             : "memory");
                aph[acc] ^= 1;
                acc ^= 1;
                if (++st == NS) { st = 0; ph ^= 1; }
            }
        }
    } else {  // ---- epilogue: warps 2..5 -> TMEM lane quadrant warp % 4
        const int quad = warp & 3;
        uint32_t aph[2] = {0, 0};
        int acc = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            mbar_wait(acc_full + acc, aph[acc]);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // TMEM row `lane` -> padded shared-memory rows -> coalesced row-segment stores (a
            // lane per TMEM row would store 16 B into 32 different rows per instruction)
            const int64_t row0 = t * kBM + quad * 32;
            float* stg = staging + quad * 32 * SP;
#pragma unroll 1
            for (int cb = 0; cb < N; cb += CW) {
#pragma unroll 1
                for (int c0 = 0; c0 < CW; c0 += 16) {
                    float v[16];
                    tmem_ld16(tmem + acc * kAcc + ((uint32_t)(quad * 32) << 16) + (uint32_t)(cb + c0), v);
#pragma unroll
                    for (int i = 0; i < 16; i += 4) {
                        float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        if (bias) {
                            o.x += __ldg(bias + cb + c0 + i);
                            o.y += __ldg(bias + cb + c0 + i + 1);
                            o.z += __ldg(bias + cb + c0 + i + 2);
                            o.w += __ldg(bias + cb + c0 + i + 3);
                        }
                        if (relu) {
                            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                        }
                        *reinterpret_cast<float4*>(stg + lane * SP + c0 + i) = o;
                    }
                }
                __syncwarp();
                constexpr int nv = CW / 4;
#pragma unroll 4
                for (int e = lane; e < 32 * nv; e += 32) {
                    const int r = e / nv, c = e - r * nv;
                    if (row0 + r < M)
                        __stcs(reinterpret_cast<float4*>(Y + (row0 + r) * N + cb) + c,
                               *reinterpret_cast<const float4*>(stg + r * SP + 4 * c));
                }
                __syncwarp();
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + acc);
            aph[acc] ^= 1;
            acc ^= 1;
        }
    }
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * kAcc));
}

// ---------------------------------------------------------------- fp32-accurate: 3xTF32
// X W in fp32 accuracy on the TF32 tensor cores by splitting both operands (the "3xTF32"
// scheme): x = x_hi + x_lo with x_hi = x with its low 13 mantissa bits cleared (a TF32 value,
// read exactly by kind::tf32 whether the hardware truncates or rounds) and x_lo = x - x_hi
// (exact in fp32, |x_lo| < 2^-10 |x|); likewise w.  Then
//     x w = x_hi w_hi + x_lo w_hi + x_hi w_lo + x_lo w_lo,
// the last term (< 2^-20 |x w|) dropped, x_lo / w_lo themselves read as TF32 (relative error
// 2^-10 of a term already 2^-10 small): |y - y_ref| <~ 2^-19 sum_k |x_k w_k| + fp32 accumulation,
// inside the layer tolerance 1e-5 sum|x w|.  Three tcgen05.mma per K step of 8, all into the
// same TMEM accumulator, in a fixed order (deterministic).
//
// Warp roles (persistent CTA per SM): warp 0 TMA producer (X k-stages of 128 rows x 32 columns
// into an NSK-slot ring; W^T once), warp 1 MMA issuer, warps 2-5 epilogue (TMEM -> bias/ReLU ->
// staged coalesced stores, two accumulators), warps 6-9 split each landed X stage in place
// (hi) plus into a lo ring slot of the same (swizzled) layout, then fence.proxy.async so the
// tensor core sees the generic-proxy writes.  W^T is split once per CTA the same way.
constexpr int kX3Threads = 320;

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
    hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    lo = x - hi;
}

template <int N, int NSK, int CWT>
__global__ void __launch_bounds__(kX3Threads, 1) k_gemm_3xtf32(const __grid_constant__ CUtensorMap tmX,
                                                              const __grid_constant__ CUtensorMap tmW,
                                                              float* __restrict__ Y, int64_t M, int32_t KT,
                                                              const float* __restrict__ bias, int32_t relu,
                                                              int64_t ldy) {
    constexpr uint32_t kAcc = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
    constexpr int kStage = kBM * kBK * 4;                      // one X k-stage (16 KB)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* sX = reinterpret_cast<float*>(smem);                                  // [NSK][128][32] (hi in place)
    float* sXl = reinterpret_cast<float*>(smem + NSK * kStage);                  // [NSK][128][32] lo
    float* sW = reinterpret_cast<float*>(smem + 2 * NSK * kStage);               // [KT][N][32] hi in place
    float* sWl = sW + (size_t)KT * N * kBK;                                      // [KT][N][32] lo
    uint64_t* bars = reinterpret_cast<uint64_t*>(sWl + (size_t)KT * N * kBK);
    uint64_t* full = bars;                 // [NSK] X stage landed (TMA)
    uint64_t* split = bars + NSK;          // [NSK] X stage split (4 converter warps)
    uint64_t* empty = bars + 2 * NSK;      // [NSK] X stage consumed (MMA commit)
    uint64_t* acc_full = bars + 3 * NSK;   // [2]
    uint64_t* acc_empty = bars + 3 * NSK + 2;  // [2] (4 epilogue warps)
    uint64_t* barW = bars + 3 * NSK + 4;   // W^T landed
    uint64_t* wsplit = bars + 3 * NSK + 5; // W^T split (4 converter warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NSK + 6);
    constexpr int CW = N < CWT ? N : CWT, SP = CW + 4;
    float* staging = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bars) + 256);  // after <= 19 barriers
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NSK; ++i) {
            mbar_init(full + i, 1);
            mbar_init(split + i, 4);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, 4);
        }
        mbar_init(barW, 1);
        mbar_init(wsplit, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * kAcc));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (M + kBM - 1) / kBM;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: W^T once, then every (tile, k-stage) in order
            mbar_expect_tx(barW, (uint32_t)(KT * N * kBK * 4));
            for (int k = 0; k < KT; ++k) tma_load_2d(sW + (size_t)k * N * kBK, &tmW, barW, k * kBK, 0);
            int st = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
                for (int k = 0; k < KT; ++k) {
                    mbar_wait(empty + st, ph ^ 1);
                    mbar_expect_tx(full + st, (uint32_t)kStage);
                    tma_load_2d(sX + (size_t)st * kBM * kBK, &tmX, full + st, k * kBK, (int)(t * kBM));
                    if (++st == NSK) { st = 0; ph ^= 1; }
                }
        }
    } else if (warp >= 6) {  // ---- converters: split W^T once, then every X stage
        const int ct = threadIdx.x - 6 * 32;   // 0..127
        mbar_wait(barW, 0);
        for (int64_t i = ct; i < (int64_t)KT * N * kBK; i += 128) {
            float h, l;
            split_tf32(sW[i], h, l);
            sW[i] = h;
            sWl[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(wsplit);
        int st = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
            for (int k = 0; k < KT; ++k) {
                mbar_wait(full + st, ph);
                float4* x4 = reinterpret_cast<float4*>(sX + (size_t)st * kBM * kBK);
                float4* l4 = reinterpret_cast<float4*>(sXl + (size_t)st * kBM * kBK);
#pragma unroll 4
                for (int i = ct; i < kBM * kBK / 4; i += 128) {
                    float4 v = x4[i], h, l;
                    split_tf32(v.x, h.x, l.x);
                    split_tf32(v.y, h.y, l.y);
                    split_tf32(v.z, h.z, l.z);
                    split_tf32(v.w, h.w, l.w);
                    x4[i] = h;
                    l4[i] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(split + st);
                if (++st == NSK) { st = 0; ph ^= 1; }
            }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer: x_hi w_hi + x_lo w_hi + x_hi w_lo per K step
            mbar_wait(wsplit, 0);
            const uint32_t idesc = idesc_tf32<N>();
            int st = 0;
            uint32_t ph = 0, aph[2] = {0, 0};
            int acc = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(acc_empty + acc, aph[acc] ^ 1);
                for (int k = 0; k < KT; ++k) {
                    mbar_wait(split + st, ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t xh = smem_u32(sX + (size_t)st * kBM * kBK), xl = smem_u32(sXl + (size_t)st * kBM * kBK);
                    const uint32_t wh = smem_u32(sW + (size_t)k * N * kBK), wl = smem_u32(sWl + (size_t)k * N * kBK);
#pragma unroll
                    for (int kk = 0; kk < kBK / 8; ++kk) {
                        const uint32_t d = tmem + acc * kAcc;
                        umma_tf32(d, umma_desc_sw128(xh + kk * 32), umma_desc_sw128(wh + kk * 32), idesc, (k | kk) != 0);
                        umma_tf32(d, umma_desc_sw128(xl + kk * 32), umma_desc_sw128(wh + kk * 32), idesc, 1);
                        umma_tf32(d, umma_desc_sw128(xh + kk * 32), umma_desc_sw128(wl + kk * 32), idesc, 1);
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(empty + st))
                                 : "memory");
                    if (++st == NSK) { st = 0; ph ^= 1; }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(acc_full + acc))
                             : "memory");
                aph[acc] ^= 1;
                acc ^= 1;
            }
        }
    } else {  // ---- epilogue: warps 2..5 -> TMEM lane quadrant warp % 4
        const int quad = warp & 3;
        uint32_t aph[2] = {0, 0};
        int acc = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            mbar_wait(acc_full + acc, aph[acc]);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t row0 = t * kBM + quad * 32;
            float* stg = staging + quad * 32 * SP;
#pragma unroll 1
            for (int cb = 0; cb < N; cb += CW) {
#pragma unroll 1
                for (int c0 = 0; c0 < CW; c0 += 16) {
                    float v[16];
                    tmem_ld16(tmem + acc * kAcc + ((uint32_t)(quad * 32) << 16) + (uint32_t)(cb + c0), v);
#pragma unroll
                    for (int i = 0; i < 16; i += 4) {
                        float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        if (bias) {
                            o.x += __ldg(bias + cb + c0 + i);
                            o.y += __ldg(bias + cb + c0 + i + 1);
                            o.z += __ldg(bias + cb + c0 + i + 2);
                            o.w += __ldg(bias + cb + c0 + i + 3);
                        }
                        if (relu) {
                            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                        }
                        *reinterpret_cast<float4*>(stg + lane * SP + c0 + i) = o;
                    }
                }
                __syncwarp();
                constexpr int nv = CW / 4;
#pragma unroll 4
                for (int e = lane; e < 32 * nv; e += 32) {
                    const int r = e / nv, c = e - r * nv;
                    if (row0 + r < M)
                        __stcs(reinterpret_cast<float4*>(Y + (row0 + r) * ldy + cb) + c,
                               *reinterpret_cast<const float4*>(stg + r * SP + 4 * c));
                }
                __syncwarp();
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + acc);
            aph[acc] ^= 1;
            acc ^= 1;
        }
    }
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * kAcc));
}

// ---------------------------------------------------------------- fp32 on the CUDA cores
// The fallback for output widths that are not a tcgen05 N (16, 32, 64, 128, 256): a plain fp32
// FFMA kernel, one thread per (row, 4 consecutive columns),
// K-loop in order with fmaf (the arithmetic of a textbook fp32 GEMM, deterministic).  W^T rows
// are read through the read-only cache; X rows are reused from L1 by the N / 4 threads of a row.
__global__ void k_gemm_fp32_cc(const float* __restrict__ X, int64_t M, int32_t K, const float* __restrict__ Wt,
                               int32_t N, float* __restrict__ Y, const float* __restrict__ bias, int32_t relu) {
    const int32_t nq = N / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * nq; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / nq;
        const int32_t c = (int32_t)(i - row * nq) * 4;
        const float* x = X + row * K;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        for (int32_t k = 0; k < K; ++k) {
            const float xv = __ldg(x + k);
            a0 = fmaf(xv, __ldg(Wt + (int64_t)c * K + k), a0);
            a1 = fmaf(xv, __ldg(Wt + (int64_t)(c + 1) * K + k), a1);
            a2 = fmaf(xv, __ldg(Wt + (int64_t)(c + 2) * K + k), a2);
            a3 = fmaf(xv, __ldg(Wt + (int64_t)(c + 3) * K + k), a3);
        }
        float4 o = make_float4(a0, a1, a2, a3);
        if (bias) {
            o.x += __ldg(bias + c); o.y += __ldg(bias + c + 1); o.z += __ldg(bias + c + 2); o.w += __ldg(bias + c + 3);
        }
        if (relu) {
            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
        }
        __stcs(reinterpret_cast<float4*>(Y + row * N + c), o);
    }
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    AGCN_CHECK(fn != nullptr, AGCN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D fp32 row-major [rows x cols] (ld = cols), box {32 cols, box_rows}, SWIZZLE_128B, OOB -> 0
CUtensorMap make_map(const float* base, int64_t rows, int64_t cols, uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AGCN_CHECK(r == CUDA_SUCCESS, AGCN_ERR_INVALID_ARG, "tensor map encode failed (alignment / sizes)");
    return m;
}

template <int N, int NS, int CWT = 64>
bool try_launch_ws(const CUtensorMap& mx, const CUtensorMap& mw, float* Y, int64_t M, int32_t KT, const float* bias,
                   int32_t relu, cudaStream_t s) {
    constexpr int CW = N < CWT ? N : CWT;
    const size_t smem = 1024 + (size_t)NS * KT * kBM * kBK * 4 + (size_t)KT * N * kBK * 4 + 128 +
                        (size_t)4 * 32 * (CW + 4) * 4;
    if (smem > 227 * 1024) return false;
    auto kern = k_gemm_tf32_ws<N, NS, CWT>;
    AGCN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = (M + kBM - 1) / kBM;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms()));
    kern<<<(unsigned)grid, kWsThreads, smem, s>>>(mx, mw, Y, M, KT, bias, relu);
    post_launch();
    return true;
}

template <int N>
void launch_gemm(const CUtensorMap& mx, const CUtensorMap& mw, float* Y, int64_t M, int32_t KT, const float* bias,
                 int32_t relu, cudaStream_t s) {
    // pipelined warp-specialized kernel when it fits, else one tile per CTA
    if (try_launch_ws<N, 4>(mx, mw, Y, M, KT, bias, relu, s) || try_launch_ws<N, 3>(mx, mw, Y, M, KT, bias, relu, s) ||
        try_launch_ws<N, 2>(mx, mw, Y, M, KT, bias, relu, s) || try_launch_ws<N, 1, 32>(mx, mw, Y, M, KT, bias, relu, s))
        return;
    const size_t smem = 1024 + (size_t)KT * (kBM + N) * kBK * 4 + 64;
    AGCN_CHECK(smem <= 227 * 1024, AGCN_ERR_UNSUPPORTED, "F_in x F_out too large for the tcgen05 GEMM");
    auto kern = k_gemm_tf32<N>;
    AGCN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    AGCN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGemmThreads, smem));
    constexpr int cols = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
    occ = std::max(1, std::min(occ, 512 / cols));  // resident CTAs share the SM's 512 TMEM columns
    const int64_t ntiles = (M + kBM - 1) / kBM;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms() * occ));
    kern<<<(unsigned)grid, kGemmThreads, smem, s>>>(mx, mw, Y, M, KT, bias, relu);
    post_launch();
}

template <int N, int NSK, int CWT>
bool try_launch_3x(const CUtensorMap& mx, const CUtensorMap& mw, float* Y, int64_t M, int32_t KT, const float* bias,
                   int32_t relu, int64_t ldy, cudaStream_t s) {
    constexpr int CW = N < CWT ? N : CWT;
    const size_t smem = 1024 + (size_t)2 * NSK * kBM * kBK * 4 + (size_t)2 * KT * N * kBK * 4 + 256 +
                        (size_t)4 * 32 * (CW + 4) * 4;
    if (smem > 227 * 1024) return false;
    auto kern = k_gemm_3xtf32<N, NSK, CWT>;
    AGCN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = (M + kBM - 1) / kBM;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms()));
    kern<<<(unsigned)grid, kX3Threads, smem, s>>>(mx, mw, Y, M, KT, bias, relu, ldy);
    post_launch();
    return true;
}

template <int N>
bool launch_3x(const CUtensorMap& mx, const CUtensorMap& mw, float* Y, int64_t M, int32_t KT, const float* bias,
               int32_t relu, int64_t ldy, cudaStream_t s) {
    return try_launch_3x<N, 4, 64>(mx, mw, Y, M, KT, bias, relu, ldy, s) ||
           try_launch_3x<N, 3, 32>(mx, mw, Y, M, KT, bias, relu, ldy, s) ||
           try_launch_3x<N, 2, 32>(mx, mw, Y, M, KT, bias, relu, ldy, s);
}

// Y[:, n0 : n0 + Ns] for one power-of-two slice width Ns (W^T rows n0 .. n0 + Ns: contiguous)
bool launch_3x_slice(const float* X, int64_t M, int32_t K, const float* Wt, int32_t Ns, int32_t n0, float* Y,
                     int32_t N, const float* bias, int32_t relu, cudaStream_t s) {
    const int32_t KT = (K + kBK - 1) / kBK;
    const CUtensorMap mx = make_map(X, M, K, kBM);
    const CUtensorMap mw = make_map(Wt + (int64_t)n0 * K, Ns, K, (uint32_t)Ns);
    float* y = Y + n0;
    const float* b = bias ? bias + n0 : nullptr;
    switch (Ns) {
        case 16: return launch_3x<16>(mx, mw, y, M, KT, b, relu, N, s);
        case 32: return launch_3x<32>(mx, mw, y, M, KT, b, relu, N, s);
        case 64: return launch_3x<64>(mx, mw, y, M, KT, b, relu, N, s);
        case 128: return launch_3x<128>(mx, mw, y, M, KT, b, relu, N, s);
        case 256: return launch_3x<256>(mx, mw, y, M, KT, b, relu, N, s);
        default: return false;
    }
}

}  // namespace

void gemm_xw_fp32(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y, const float* bias,
                  int32_t relu, cudaStream_t s) {
    AGCN_CHECK(M >= 0 && K >= 1 && K <= 256 && (K % 4) == 0, AGCN_ERR_UNSUPPORTED, "K must be in [4, 256], K % 4 == 0");
    AGCN_CHECK(N >= 4 && N <= 256 && N % 4 == 0, AGCN_ERR_UNSUPPORTED, "N must be in [4, 256], N % 4 == 0");
    AGCN_CHECK(X && Wt && Y, AGCN_ERR_INVALID_ARG, "NULL pointer");
    AGCN_CHECK(((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Wt) | reinterpret_cast<uintptr_t>(Y)) & 15u) == 0,
               AGCN_ERR_INVALID_ARG, "X, W^T and Y must be 16-byte aligned");
    if (M == 0) return;
    bool done = false;
    if (N == 16 || N == 32 || N == 64 || N == 128 || N == 256) {
        // one launch, or -- when the split W^T does not fit in shared memory next to the X ring --
        // column slices of W (each re-reads X; the products are column-separable)
        for (int32_t Ns = N; Ns >= 16 && !done; Ns /= 2) {
            // probe the slice width with the first slice (a launch only happens if it fits)
            if (!launch_3x_slice(X, M, K, Wt, Ns, 0, Y, N, bias, relu, s)) continue;
            for (int32_t n0 = Ns; n0 < N; n0 += Ns) {
                const bool ok = launch_3x_slice(X, M, K, Wt, Ns, n0, Y, N, bias, relu, s);
                AGCN_CHECK(ok, AGCN_ERR_CUDA, "internal: 3xTF32 slice launch");
            }
            done = true;
        }
    }
    if (!done) {
        const int64_t work = M * (N / 4);
        const unsigned grid = (unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 16);
        k_gemm_fp32_cc<<<grid, 256, 0, s>>>(X, M, K, Wt, N, Y, bias, relu);
        post_launch();
    }
}

void gemm_xw_tf32(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y, const float* bias,
                  int32_t relu, cudaStream_t s) {
    AGCN_CHECK(M >= 0 && K >= 1 && K <= 256 && (K % 4) == 0, AGCN_ERR_UNSUPPORTED, "K must be in [4, 256], K % 4 == 0");
    AGCN_CHECK(N == 16 || N == 32 || N == 64 || N == 128 || N == 256, AGCN_ERR_UNSUPPORTED,
               "N must be 16, 32, 64, 128 or 256");
    AGCN_CHECK(X && Wt && Y, AGCN_ERR_INVALID_ARG, "NULL pointer");
    AGCN_CHECK(((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Wt) | reinterpret_cast<uintptr_t>(Y)) & 15u) == 0,
               AGCN_ERR_INVALID_ARG, "X, W^T and Y must be 16-byte aligned");
    if (M == 0) return;
    const int32_t KT = (K + kBK - 1) / kBK;
    const CUtensorMap mx = make_map(X, M, K, kBM);
    const CUtensorMap mw = make_map(Wt, N, K, (uint32_t)N);
    switch (N) {
        case 16: launch_gemm<16>(mx, mw, Y, M, KT, bias, relu, s); break;
        case 32: launch_gemm<32>(mx, mw, Y, M, KT, bias, relu, s); break;
        case 64: launch_gemm<64>(mx, mw, Y, M, KT, bias, relu, s); break;
        case 128: launch_gemm<128>(mx, mw, Y, M, KT, bias, relu, s); break;
        default: launch_gemm<256>(mx, mw, Y, M, KT, bias, relu, s); break;
    }
}

}  // namespace agcn
