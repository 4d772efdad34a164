// tma_gather_probe.cu -- can TMA tile::gather4 with a decoupled producer warp beat register
// (LDG.E.256) gathers on B200?  The SpMM's inner operation: gather F = 64 float rows of X by a
// list of row indices and sum them (tools/gather_probe.cu is the LDG side).
//
// k_tma_pc<S, C, P>: one producer warp + C consumer warps per CTA, a ring of S stages of 32 rows
// (8 KB) in shared memory.  The producer keeps the row indices of its next P chunks in
// registers (loaded P chunks ahead, so index latency is off the critical path) and issues
// eight gather4 per stage (lanes 0..7, 4 rows = 1 KB each) completing on the stage's full
// mbarrier; consumer warp w takes stages w, w + C, ... and frees them through the empty
// mbarrier.  Bytes in flight per SM = S * 8 KB * CTAs, independent of registers.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_gather_probe.cu -o tma_gather_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int F = 64;
constexpr int ROWB = F * 4;
constexpr int STAGE_B = 32 * ROWB;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}

template <int S, int C, int P>
__global__ void __launch_bounds__(32 * (C + 1)) k_tma_pc(const __grid_constant__ CUtensorMap tmap,
                                                        const int* __restrict__ idx, long n_idx,
                                                        float* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char ring[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&full[k])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&empty[k])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long nch = (n_idx + 31) / 32;
    const long G = gridDim.x;
    if (warp == 0) {
        int pre[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const long q = (blockIdx.x + (long)p * G) * 32 + lane;
            pre[p] = q < n_idx ? __ldg(idx + q) : 0;
        }
        for (long jb = 0;; jb += P) {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const long jj = jb + p;
                const long ch = blockIdx.x + jj * G;
                if (ch >= nch) return;
                const int k = (int)(jj % S);
                if (jj >= S) mbar_wait(su32(&empty[k]), (uint32_t)(((jj / S) - 1) & 1));
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                                 :: "r"(su32(&full[k])), "r"(STAGE_B) : "memory");
                __syncwarp();
                const int b = (lane & 7) * 4;
                const int r0 = __shfl_sync(0xffffffffu, pre[p], b), r1 = __shfl_sync(0xffffffffu, pre[p], b + 1);
                const int r2 = __shfl_sync(0xffffffffu, pre[p], b + 2), r3 = __shfl_sync(0xffffffffu, pre[p], b + 3);
                if (lane < 8)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                        :: "r"(su32(ring + (size_t)k * STAGE_B + lane * 4 * ROWB)), "l"(&tmap), "r"(0),
                           "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&full[k]))
                        : "memory");
                const long qn = (blockIdx.x + (jj + P) * G) * 32 + lane;
                pre[p] = qn < n_idx ? __ldg(idx + qn) : 0;
            }
        }
    }
    // consumers
    const int c = warp - 1;
    const int s = lane >> 4, li = lane & 15;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (long jj = c;; jj += C) {
        const long ch = blockIdx.x + jj * G;
        if (ch >= nch) break;
        const int k = (int)(jj % S);
        mbar_wait(su32(&full[k]), (uint32_t)((jj / S) & 1));
        const float4* rows = reinterpret_cast<const float4*>(ring + (size_t)k * STAGE_B);
#pragma unroll 8
        for (int r = s; r < 32; r += 2) {
            const float4 v = rows[r * 16 + li];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[k])) : "memory");
    }
    out[blockIdx.x * 32 * (C + 1) + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// register baseline: LDG.E.256 (8 lanes x 32 B per row), U rows in flight per lane
template <int U>
__global__ void __launch_bounds__(256) k_ldg256(const float* __restrict__ X, const int* __restrict__ idx, long n_idx,
                                                float* __restrict__ out) {
    const int lane = threadIdx.x & 31, s = lane >> 3, li = lane & 7;
    const long gw = (long)blockIdx.x * 8 + (threadIdx.x >> 5), W = (long)gridDim.x * 8;
    float acc = 0.f;
    for (long base = gw * 4 * U; base < n_idx; base += W * 4 * U) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long q = base + s * U + u;
            int r = q < n_idx ? __ldg(idx + q) : 0;
            asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]),
                           "=f"(v[u][5]), "=f"(v[u][6]), "=f"(v[u][7])
                         : "l"(X + (long)r * F + li * 8));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[u][j];
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    long n_rows = argc > 1 ? atol(argv[1]) : (1 << 18);
    long n_idx = argc > 2 ? atol(argv[2]) : (1l << 26);
    int skew = argc > 3 ? atoi(argv[3]) : 0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<int> h(n_idx);
    std::mt19937_64 g(7);
    if (!skew) {
        std::uniform_int_distribution<long> d(0, n_rows - 1);
        for (auto& x : h) x = (int)d(g);
    } else {  // R-MAT-like column popularity: 23 independent bits, P(bit = 1) = 0.24, scrambled
        std::uniform_real_distribution<double> d(0, 1);
        int bits = 0;
        while ((1l << bits) < n_rows) ++bits;
        for (auto& x : h) {
            long v = 0;
            for (int b = 0; b < bits; ++b) v |= (long)(d(g) < 0.24) << b;
            x = (int)((((unsigned long)v * 2654435761ul) ^ 0x5bd1e995ul) % (unsigned long)n_rows);
        }
    }
    float *X, *out;
    int* idx;
    CK(cudaMalloc(&X, (size_t)n_rows * ROWB));
    CK(cudaMalloc(&idx, sizeof(int) * n_idx));
    CK(cudaMalloc(&out, sizeof(float) * sms * 8 * 1024));
    CK(cudaMemset(X, 0, (size_t)n_rows * ROWB));
    CK(cudaMemcpy(idx, h.data(), sizeof(int) * n_idx, cudaMemcpyHostToDevice));
    char* flush;
    CK(cudaMalloc(&flush, 512 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double gbytes = (double)n_idx * ROWB / 1e9;
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            CK(cudaMemset(flush, it, 512 << 20));
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        printf("%-34s n_rows=%ld (%.0f MB) skew=%d  %.3f ms  %.2f TB/s gathered\n", name, n_rows,
               n_rows * ROWB / 1e6, skew, best, gbytes / best);
    };
    timeit("ldg256 U=4 grid=148x3 (24 warps)", [&] { k_ldg256<4><<<sms * 3, 256>>>(X, idx, n_idx, out); });
    timeit("ldg256 U=4 grid=148x8 (64 warps)", [&] { k_ldg256<4><<<sms * 8, 256>>>(X, idx, n_idx, out); });

    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)n_rows};
    cuuint64_t strides[1] = {(cuuint64_t)ROWB};
    cuuint32_t box[2] = {(cuuint32_t)F, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tensor map encode failed %d\n", (int)r); return 1; }
    auto run = [&](auto kern, int S, int C, int ctas, const char* tag) {
        size_t smem = (size_t)S * STAGE_B;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        char name[80];
        snprintf(name, sizeof(name), "tma-pc S=%d C=%d ctas/SM=%d %s", S, C, ctas, tag);
        timeit(name, [&] { kern<<<sms * ctas, 32 * (C + 1), smem>>>(tm, idx, n_idx, out); });
    };
    run(k_tma_pc<8, 4, 8>, 8, 4, 2, "");
    run(k_tma_pc<12, 4, 8>, 12, 4, 1, "");
    run(k_tma_pc<12, 4, 8>, 12, 4, 2, "");
    run(k_tma_pc<16, 8, 8>, 16, 8, 1, "");
    run(k_tma_pc<24, 8, 8>, 24, 8, 1, "");
    run(k_tma_pc<26, 13, 8>, 26, 13, 1, "");
    run(k_tma_pc<13, 6, 8>, 13, 6, 2, "");
    return 0;
}
