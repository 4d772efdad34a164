// colmap.cuh -- optional column relabel into the padded multi-GPU layout:
// column j owned by shard p (bounds[p] <= j < bounds[p+1]) is read from row
// p * slot_rows + (j - bounds[p]) of the all-gathered X buffer.
#pragma once
#include <stdint.h>

namespace agcn {

constexpr int kMaxColParts = 64;

struct ColMap {
    int32_t nparts;     // 0: identity
    int32_t slot_rows;
    int64_t n_cols;
    int64_t bounds[kMaxColParts + 1];
};

__device__ __forceinline__ int32_t map_col(int32_t j, const ColMap& cm) {
    if (cm.nparts <= 0) return j;
    int p = 0;
    while (p + 1 < cm.nparts && (int64_t)j >= cm.bounds[p + 1]) ++p;
    return (int32_t)(p * (int64_t)cm.slot_rows + (j - cm.bounds[p]));
}

}  // namespace agcn
