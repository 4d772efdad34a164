// scan.cu -- device exclusive prefix sum (int32), used by the counting sort and the
// row-pointer update of the degree-sorted CSR.  Three phases: per-tile reduce, a single-CTA
// scan of the tile sums, per-tile scan + carry.  Tiles of 4096 elements (1024 threads x 4).
#include "internal.h"

namespace agcn {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int32_t warp_incl_scan(int32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive block scan of one value per thread; returns the prefix, *total = block sum.
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* total) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t wtot;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t inc = warp_incl_scan(v);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        int32_t s = lane < nw ? wsum[lane] : 0;
        int32_t si = warp_incl_scan(s);
        if (lane < nw) wsum[lane] = si - s;
        if (lane == nw - 1) wtot = si;
    }
    __syncthreads();
    int32_t r = inc - v + wsum[w];
    *total = wtot;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_tile_reduce(const int32_t* __restrict__ in,
                                                             int64_t n, int32_t* __restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    int32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of the tile sums in place (any count, sequential carry).
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(int32_t* __restrict__ sums, int64_t m) {
    int32_t carry = 0;
    for (int64_t base = 0; base < m; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        int32_t v = i < m ? sums[i] : 0;
        int32_t tot;
        int32_t ex = block_excl_scan(v, &tot);
        if (i < m) sums[i] = ex + carry;
        carry += tot;
    }
    if (threadIdx.x == 0) sums[m] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const int32_t* __restrict__ in,
                                                           int32_t* __restrict__ out, int64_t n,
                                                           const int32_t* __restrict__ sums,
                                                           int64_t ntiles) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    int32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int32_t tot;
    int32_t ex = block_excl_scan(s, &tot) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = sums[ntiles];
}

// One CTA for short arrays (one launch instead of three): tiles in order with a carry.
// In place is fine: every tile is read before it is written, by the same threads.
__global__ void __launch_bounds__(kScanThreads) k_scan_small(const int32_t* __restrict__ in,
                                                            int32_t* __restrict__ out, int64_t n) {
    int32_t carry = 0;
    for (int64_t t0 = 0; t0 < n; t0 += kScanTile) {
        const int64_t base = t0 + (int64_t)threadIdx.x * kScanItems;
        int32_t v[kScanItems];
        int32_t sum = 0;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            v[i] = base + i < n ? in[base + i] : 0;
            sum += v[i];
        }
        int32_t tot;
        int32_t ex = block_excl_scan(sum, &tot) + carry;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            if (base + i < n) out[base + i] = ex;
            ex += v[i];
        }
        carry += tot;
    }
    if (threadIdx.x == 0) out[n] = carry;
}

constexpr int64_t kSmallScan = 16 * kScanTile;  // up to 64K elements: single CTA

}  // namespace

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        AGCN_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), s));
        return;
    }
    if (n <= kSmallScan) {
        k_scan_small<<<1, kScanThreads, 0, s>>>(in, out, n);
        post_launch();
        return;
    }
    const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    Scratch tmp(s);
    int32_t* sums = tmp.alloc<int32_t>(ntiles + 1);
    k_tile_reduce<<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, sums);
    post_launch();
    k_scan_sums<<<1, kScanThreads, 0, s>>>(sums, ntiles);
    post_launch();
    k_tile_scan<<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, out, n, sums, ntiles);
    post_launch();
}

}  // namespace agcn
