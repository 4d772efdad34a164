// l2_probe.cu -- does an L2 set-aside (cudaLimitPersistingL2CacheSize) make L2::evict_last
// X-row loads stick on B200?  Random 256-byte row gathers (F = 64 fp32) from a table of
// n_rows rows while a streaming buffer of the CSR's size is read alongside (evict-first), as
// in the SpMM.  Rows are drawn from a skewed distribution; the hottest K rows are "hot".
// Variants: plain loads; evict_last on hot rows; evict_last on hot rows + set-aside;
// access-policy window over the whole table + set-aside.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 l2_probe.cu -o l2_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int F = 64;

struct f8 { float4 a, b; };

template <int MODE>  // 0 plain, 1 evict_last on hot (bit 31), evict_first on cold
__device__ __forceinline__ f8 ld(const float* p, bool hot) {
    f8 r;
    if (MODE == 1 && hot)
        asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w) : "l"(p));
    else if (MODE == 1)
        asm volatile("ld.global.nc.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w) : "l"(p));
    else
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w) : "l"(p));
    return r;
}

// 8 lanes per row, 4 rows per warp-step, U = 4 in flight; every index also streams 8 bytes
// of a "CSR" buffer (evict-first), like the SpMM.
template <int MODE>
__global__ void __launch_bounds__(256, 4) k_gather(const float* __restrict__ X, const int* __restrict__ idx,
                                                   long n_idx, const int2* __restrict__ csr, float* out) {
    const int lane = threadIdx.x & 31, s = lane / 8, li = lane % 8;
    const long gw = (long)blockIdx.x * 8 + (threadIdx.x >> 5), W = (long)gridDim.x * 8;
    float acc = 0.f;
    for (long base = gw * 32; base < n_idx; base += W * 32) {
        const long q = base + lane;
        int c = q < n_idx ? __ldcs(idx + q) : 0;
        int2 e = q < n_idx ? __ldcs(csr + q) : make_int2(0, 0);
        acc += (float)e.x;
#pragma unroll
        for (int k = 0; k < 8; k += 4) {
            f8 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cu = __shfl_sync(0xffffffffu, c, s * 8 + k + u);
                v[u] = ld<MODE>(X + (long)(cu & 0x7fffffff) * F + li * 8, cu < 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += v[u].a.x + v[u].b.w;
        }
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
    long n_rows = argc > 1 ? atol(argv[1]) : 8388608;
    long n_idx = argc > 2 ? atol(argv[2]) : (1l << 26);
    long K = argc > 3 ? atol(argv[3]) : 390000;  // hot rows
    double alpha = argc > 4 ? atof(argv[4]) : 1.0; // Zipf exponent of the row popularity
    int dev = 0, sms = 0, maxp = 0, l2 = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    printf("L2 %d B, max persisting L2 %d B\n", l2, maxp);
    // Zipf-like popularity over a scrambled row order
    std::vector<double> w(n_rows);
    double tot = 0;
    for (long i = 0; i < n_rows; ++i) tot += (w[i] = 1.0 / pow((double)(i + 1), alpha));
    std::vector<double> cdf(n_rows);
    double acc = 0;
    for (long i = 0; i < n_rows; ++i) cdf[i] = (acc += w[i] / tot);
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> u(0, 1);
    std::vector<int> h(n_idx);
    long hot_refs = 0;
    for (auto& x : h) {
        long r = std::lower_bound(cdf.begin(), cdf.end(), u(g)) - cdf.begin();
        if (r >= n_rows) r = n_rows - 1;
        bool hot = r < K;
        hot_refs += hot;
        long row = (long)(((unsigned long)r * 2654435761ul) % (unsigned long)n_rows);
        x = (int)row | (hot ? (int)0x80000000 : 0);
    }
    printf("n_rows %ld (%.0f MB), hot %ld rows (%.0f MB) get %.1f%% of refs\n", n_rows, n_rows * 256 / 1e6, K,
           K * 256 / 1e6, 100.0 * hot_refs / n_idx);
    float *X, *out;
    int* idx;
    int2* csr;
    CK(cudaMalloc(&X, (size_t)n_rows * F * 4));
    CK(cudaMemset(X, 0, (size_t)n_rows * F * 4));
    CK(cudaMalloc(&idx, sizeof(int) * n_idx));
    CK(cudaMalloc(&csr, sizeof(int2) * n_idx));
    CK(cudaMemset(csr, 0, sizeof(int2) * n_idx));
    CK(cudaMalloc(&out, sizeof(float) * sms * 8 * 256));
    CK(cudaMemcpy(idx, h.data(), sizeof(int) * n_idx, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, int mode) {
        for (int it = 0; it < 3; ++it) {
            if (mode == 0) k_gather<0><<<sms * 4, 256, 0, st>>>(X, idx, n_idx, csr, out);
            else k_gather<1><<<sms * 4, 256, 0, st>>>(X, idx, n_idx, csr, out);
        }
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(e0, st);
            if (mode == 0) k_gather<0><<<sms * 4, 256, 0, st>>>(X, idx, n_idx, csr, out);
            else k_gather<1><<<sms * 4, 256, 0, st>>>(X, idx, n_idx, csr, out);
            cudaEventRecord(e1, st);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        printf("%-44s %.3f ms  %.2f TB/s gathered\n", name, best, n_idx * 256.0 / best / 1e9);
    };
    run("plain", 0);
    run("hot evict_last / cold evict_first, no set-aside", 1);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
    run("hot evict_last / cold evict_first, set-aside max", 1);
    run("plain, set-aside max", 0);
    // access policy window over the first min(table, maxp) bytes
    cudaStreamAttrValue a{};
    size_t win = std::min<size_t>((size_t)n_rows * F * 4, (size_t)maxp);
    a.accessPolicyWindow.base_ptr = X;
    a.accessPolicyWindow.num_bytes = win;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));
    run("plain + policy window (first max bytes)", 0);
    return 0;
}
