// gather_probe.cu -- microbenchmark of the SpMM's inner operation on B200: gather of
// F-float rows of X by a list of row indices, summed per warp (the "L2->SM gather roof").
//   (a) LDG.128 by combined warps (16 lanes x float4 per row for F = 64), U loads in flight
//   (b) TMA tile::gather4 (cp.async.bulk.tensor.2d ... gather4) into a shared-memory ring
// Index streams: uniform random, or skewed (R-MAT-like power law) over n rows.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 gather_probe.cu -o gather_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int F = 64;          // floats per row
constexpr int FV = F / 4;      // float4 per row
constexpr int ROWB = F * 4;    // bytes per row

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float4* __restrict__ X, const int* __restrict__ idx, long n_idx,
                                             float* __restrict__ out) {
    const int lane = threadIdx.x & 31, s = lane / FV, li = lane % FV;
    const long gw = (long)blockIdx.x * 8 + (threadIdx.x >> 5), W = (long)gridDim.x * 8;
    float4 acc = make_float4(0, 0, 0, 0);
    // each warp takes chunks of 2U indices: sub-warp s takes U of them
    for (long base = gw * 2 * U; base < n_idx; base += W * 2 * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long q = base + s * U + u;
            int r = q < n_idx ? __ldg(idx + q) : 0;
            v[u] = q < n_idx ? __ldg(X + (long)r * FV + li) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// 256-bit gathers (LDG.E.256): 8 lanes x 32 B per row at F = 64.  HINT: 0 normal; 1 evict_last
// for rows flagged hot (bit 31 of the index), evict_first otherwise; 2 all evict_first.
struct f8 { float v[8]; };
template <int HINT>
__device__ __forceinline__ f8 ld256(const float* p, bool hot) {
    f8 r;
    if (HINT == 1 && hot)
        asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    else if (HINT >= 1)
        asm volatile("ld.global.nc.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    else
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                       "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    return r;
}
template <int U, int HINT>
__global__ void __launch_bounds__(256) k_ldg256(const float* __restrict__ X, const int* __restrict__ idx, long n_idx,
                                                float* __restrict__ out) {
    constexpr int LP = F / 8;  // lanes per row
    const int lane = threadIdx.x & 31, s = lane / LP, li = lane % LP;
    constexpr int G = 32 / LP;
    const long gw = (long)blockIdx.x * 8 + (threadIdx.x >> 5), W = (long)gridDim.x * 8;
    float acc = 0.f;
    for (long base = gw * G * U; base < n_idx; base += W * G * U) {
        f8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long q = base + s * U + u;
            int r = q < n_idx ? __ldg(idx + q) : 0;
            v[u] = ld256<HINT>(X + (long)(r & 0x7fffffff) * F + li * 8, r < 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[u].v[j];
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA gather: each warp owns a ring of S stages; a stage = 32 rows (8 gather4) = 8 KB.
template <int S>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx,
                                             long n_idx, float* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = sm + (size_t)warp * S * 32 * ROWB;
    __shared__ __align__(8) uint64_t bar[4][S];
    const long gw = (long)blockIdx.x * 4 + warp, W = (long)gridDim.x * 4;
    if (lane == 0)
        for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&bar[warp][k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const long nchunks = (n_idx + 31) / 32;
    // chunk sequence of this warp: gw, gw+W, ...
    auto issue = [&](long chunk, int k) {
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[warp][k])), "r"(32 * ROWB));
        }
        __syncwarp();
        // lanes 0..7 each issue one gather4 (rows 4l..4l+3 of the chunk)
        if (lane < 8) {
            long q = chunk * 32 + lane * 4;
            int r0 = q + 0 < n_idx ? idx[q + 0] : 0, r1 = q + 1 < n_idx ? idx[q + 1] : 0;
            int r2 = q + 2 < n_idx ? idx[q + 2] : 0, r3 = q + 3 < n_idx ? idx[q + 3] : 0;
            uint32_t dst = smem_u32(ring + ((size_t)k * 32 + lane * 4) * ROWB);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(dst), "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[warp][k]))
                : "memory");
        }
    };
    float4 acc = make_float4(0, 0, 0, 0);
    long c = gw;
    int nfly = 0;
    for (int k = 0; k < S && c + (long)k * W < nchunks; ++k) { issue(c + (long)k * W, k); ++nfly; }
    uint32_t phase = 0;
    int k = 0;
    for (; c < nchunks; c += W) {
        // wait stage k
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(smem_u32(&bar[warp][k])), "r"((phase >> k) & 1));
        }
        phase ^= (1u << k);
        const float4* rows = reinterpret_cast<const float4*>(ring + (size_t)k * 32 * ROWB);
        const int s = lane / FV, li = lane % FV;
#pragma unroll 4
        for (int r = s; r < 32; r += 2) {
            float4 v = rows[r * FV + li];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        __syncwarp();
        long nc = c + (long)S * W;
        if (nc < nchunks) issue(nc, k);
        k = (k + 1) % S;
    }
    out[blockIdx.x * 128 + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    long n_rows = argc > 1 ? atol(argv[1]) : (1 << 18);     // 64 MB at F=64
    long n_idx = argc > 2 ? atol(argv[2]) : (1l << 26);
    int skew = argc > 3 ? atoi(argv[3]) : 0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<int> h(n_idx);
    std::mt19937_64 g(7);
    if (!skew) {
        std::uniform_int_distribution<long> d(0, n_rows - 1);
        for (auto& x : h) x = (int)d(g);
    } else {  // power-law-ish: row = n * u^3 (hot low rows), then a fixed scramble
        std::uniform_real_distribution<double> d(0, 1);
        for (auto& x : h) { double u = d(g); x = (int)std::min<double>(n_rows - 1, n_rows * u * u * u * u); }
        for (auto& x : h) x = (int)(((unsigned long)x * 2654435761ul) % (unsigned long)n_rows);
    }
    float *X, *out;
    int* idx;
    CK(cudaMalloc(&X, (size_t)n_rows * ROWB));
    CK(cudaMalloc(&idx, sizeof(int) * n_idx));
    CK(cudaMalloc(&out, sizeof(float) * sms * 64 * 256));
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
        printf("%-28s n_rows=%ld (%.0f MB) skew=%d  %.3f ms  %.2f TB/s gathered\n", name, n_rows,
               n_rows * ROWB / 1e6, skew, best, gbytes / best);
    };
    for (int occ : {4, 8}) {
        timeit(occ == 4 ? "ldg U=4 grid=148x4" : "ldg U=4 grid=148x8",
               [&] { k_ldg<4><<<sms * occ, 256>>>(reinterpret_cast<float4*>(X), idx, n_idx, out); });
        timeit(occ == 4 ? "ldg U=8 grid=148x4" : "ldg U=8 grid=148x8",
               [&] { k_ldg<8><<<sms * occ, 256>>>(reinterpret_cast<float4*>(X), idx, n_idx, out); });
    }
    // 256-bit loads, and the hot/cold eviction policy: flag the most frequent rows (hot set of
    // ~100 MB = 390K rows at F = 64) in bit 31 of the index.
    {
        std::vector<int> cnt(n_rows, 0);
        for (auto x : h) cnt[x]++;
        std::vector<int> order(n_rows);
        for (long i = 0; i < n_rows; ++i) order[i] = (int)i;
        long K = std::min<long>(n_rows, 390000);
        std::nth_element(order.begin(), order.begin() + K, order.end(),
                         [&](int a, int b) { return cnt[a] > cnt[b]; });
        std::vector<char> hot(n_rows, 0);
        for (long i = 0; i < K; ++i) hot[order[i]] = 1;
        long hot_refs = 0;
        std::vector<int> hf(n_idx);
        for (long i = 0; i < n_idx; ++i) { hf[i] = hot[h[i]] ? (int)(h[i] | 0x80000000u) : h[i]; hot_refs += hot[h[i]]; }
        printf("hot set %ld rows (%.0f MB) receives %.1f%% of refs\n", K, K * ROWB / 1e6, 100.0 * hot_refs / n_idx);
        int* idxf;
        CK(cudaMalloc(&idxf, sizeof(int) * n_idx));
        CK(cudaMemcpy(idxf, hf.data(), sizeof(int) * n_idx, cudaMemcpyHostToDevice));
        for (int occ : {4, 8}) {
            char name[64];
            snprintf(name, sizeof(name), "ldg256 U=4 normal x%d", occ);
            timeit(name, [&] { k_ldg256<4, 0><<<sms * occ, 256>>>(X, idxf, n_idx, out); });
            snprintf(name, sizeof(name), "ldg256 U=4 hot/cold x%d", occ);
            timeit(name, [&] { k_ldg256<4, 1><<<sms * occ, 256>>>(X, idxf, n_idx, out); });
            snprintf(name, sizeof(name), "ldg256 U=2 hot/cold x%d", occ);
            timeit(name, [&] { k_ldg256<2, 1><<<sms * occ, 256>>>(X, idxf, n_idx, out); });
            snprintf(name, sizeof(name), "ldg256 U=4 all-first x%d", occ);
            timeit(name, [&] { k_ldg256<4, 2><<<sms * occ, 256>>>(X, idxf, n_idx, out); });
        }
        cudaFree(idxf);
    }
    if (getenv("PROBE_NO_TMA")) return 0;
    // TMA tensor map: 2D {F, n_rows} fp32, box {F, 1}
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
    printf("tensor map encode: %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
        for (int S : {2, 4}) {
            size_t smem = (size_t)4 * S * 32 * ROWB;
            for (int ctas : {1, 2}) {
                char name[64];
                snprintf(name, sizeof(name), "tma S=%d ctas/SM=%d", S, ctas);
                if (S == 2) {
                    CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    timeit(name, [&] { k_tma<2><<<sms * ctas, 128, smem>>>(tm, idx, n_idx, out); });
                } else {
                    CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    timeit(name, [&] { k_tma<4><<<sms * ctas, 128, smem>>>(tm, idx, n_idx, out); });
                }
            }
        }
    }
    return 0;
}
