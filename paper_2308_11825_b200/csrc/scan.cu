// scan.cu -- device exclusive prefix sum (int32), used by the counting sort, the
// row-pointer update of the degree-sorted CSR and the transpose: the single-pass decoupled
// look-back scan of scan_lb.cuh (one memset + one launch for any length).
#include "internal.h"
#include "scan_lb.cuh"

namespace agcn {

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        AGCN_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t), s));
        return;
    }
    const int64_t ntiles = (n + kLbTile - 1) / kLbTile;
    Scratch tmp(s);
    unsigned long long* st = ntiles > 1 ? tmp.alloc<unsigned long long>(ntiles + 1) : nullptr;
    launch_scan_lb(ArraySrc{in}, out, n, st, s);
}

}  // namespace agcn
