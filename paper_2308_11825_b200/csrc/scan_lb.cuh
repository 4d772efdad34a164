// scan_lb.cuh -- single-pass exclusive prefix sum (int32) with decoupled look-back: one
// launch for any length (plus a memset of the tile status words), used by the counting sort
// and the row-pointer update of the degree-sorted CSR.
//
// Tiles of kLbTile = 4096 elements, claimed in order through an atomic counter (so a tile only
// ever waits on tiles whose CTAs are already running).  Each of the 8 warps of a CTA owns 512
// consecutive elements and reads them warp-striped (lane l: elements 32 j + l, coalesced),
// scanning them with 16 warp scans and a running carry; warp 0 scans the 8 warp totals,
// publishes the tile aggregate, looks back over its predecessors 32 at a time (nearest
// inclusive prefix first), and publishes the tile's inclusive prefix.  Status word per tile:
// (flag << 32) | value, flag 1 = aggregate, 2 = inclusive prefix, written and read as one
// volatile 64-bit access.
//
// Src::get(i) returns element i (called once per element, in any order, possibly with side
// effects on other arrays); out[i] = sum_{j<i} get(j) for i < n and out[n] = total.  In place
// (out aliasing Src's input) is fine: a tile reads all of its elements before writing them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace agcn {

constexpr int kLbThreads = 256;
constexpr int kLbWarps = kLbThreads / 32;
constexpr int kLbItems = 16;                          // per lane
constexpr int64_t kLbTile = (int64_t)kLbThreads * kLbItems;  // 4096

__device__ __forceinline__ int32_t lb_warp_incl(int32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// status: [ntiles] zeroed words; counter: zeroed (NULL when there is one tile)
template <class Src>
__global__ void __launch_bounds__(kLbThreads) k_scan_lb(Src src, int32_t* out, int64_t n,
                                                        unsigned long long* __restrict__ status,
                                                        int32_t* __restrict__ counter) {
    __shared__ int32_t s_tile;
    __shared__ int32_t s_off[kLbWarps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tile = counter ? atomicAdd(counter, 1) : 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t seg = tile * kLbTile + (int64_t)w * (32 * kLbItems);
    int32_t v[kLbItems];
    int32_t run = 0;
#pragma unroll
    for (int j = 0; j < kLbItems; ++j) {  // all loads first (independent: in flight together)
        const int64_t i = seg + 32 * j + lane;
        v[j] = i < n ? src.get(i) : 0;
    }
#pragma unroll
    for (int j = 0; j < kLbItems; ++j) {
        const int32_t x = v[j];
        const int32_t inc = lb_warp_incl(x, lane);
        v[j] = run + inc - x;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_off[w] = run;
    __syncthreads();
    if (w == 0) {
        const int32_t ws = lane < kLbWarps ? s_off[lane] : 0;
        const int32_t wi = lb_warp_incl(ws, lane);
        const int32_t agg = __shfl_sync(0xffffffffu, wi, kLbWarps - 1);
        int32_t prefix = 0;
        if (tile > 0) {
            if (lane == 0) lb_store(status + tile, (1ull << 32) | (uint32_t)agg);
            int64_t t = tile - 1;
            while (true) {
                const int64_t k = t - lane;
                unsigned long long st = 2ull << 32;  // before tile 0: an inclusive prefix of 0
                if (k >= 0) {
                    do {
                        st = lb_load(status + k);
                    } while ((st >> 32) == 0);
                }
                const unsigned incl = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                const int f = incl ? __ffs(incl) - 1 : 31;   // nearest inclusive prefix
                int32_t val = lane <= f ? (int32_t)(uint32_t)st : 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                prefix += val;
                if (incl) break;
                t -= 32;
            }
        }
        if (lane == 0 && status) lb_store(status + tile, (2ull << 32) | (uint32_t)(prefix + agg));
        if (lane < kLbWarps) s_off[lane] = prefix + wi - ws;
        if (lane == 0 && (tile + 1) * kLbTile >= n) out[n] = prefix + agg;  // last tile: the total
    }
    __syncthreads();
    const int32_t off = s_off[w];
#pragma unroll
    for (int j = 0; j < kLbItems; ++j) {
        const int64_t i = seg + 32 * j + lane;
        if (i < n) out[i] = v[j] + off;
    }
}

// elements of an int32 array
struct ArraySrc {
    const int32_t* in;
    __device__ __forceinline__ int32_t get(int64_t i) const { return in[i]; }
};

// Launch k_scan_lb over n >= 1 elements on stream s; status_counter: (ntiles + 1) 64-bit words
// of device scratch (zeroed here), or NULL when n <= kLbTile.
template <class Src>
void launch_scan_lb(const Src& src, int32_t* out, int64_t n, unsigned long long* status_counter, cudaStream_t s) {
    const int64_t ntiles = (n + kLbTile - 1) / kLbTile;
    unsigned long long* status = nullptr;
    int32_t* counter = nullptr;
    if (ntiles > 1) {
        AGCN_CUDA(cudaMemsetAsync(status_counter, 0, sizeof(unsigned long long) * (size_t)(ntiles + 1), s));
        status = status_counter;
        counter = reinterpret_cast<int32_t*>(status_counter + ntiles);
    }
    k_scan_lb<Src><<<(unsigned)ntiles, kLbThreads, 0, s>>>(src, out, n, status, counter);
    post_launch();
}

}  // namespace agcn
