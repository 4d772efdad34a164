// stream_probe.cu -- the gather roof for C5's ACTUAL column stream.
//
// Replays a column-index stream (C5's degree-sorted colidx, in the order the SpMM executes its
// descriptors) as 256-byte X-row gathers (F = 64: 8 lanes x 32 B per row, 4 combined warps per
// warp, U rows in flight per lane), the same access shape as k_spmm_wide.  Each warp takes CH
// consecutive entries per step (CH / 4 per combined warp), grid-strided like the descriptors.
// Options: an encoded stream where c < 0 means row ~c of a compact hot buffer Xh; L2 hints
// (hot evict_last / cold evict_first); reading a vals stream; storing one output row per
// combined warp and step (the Y stores).  Driven by tools/stream_probe.py (ctypes).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC stream_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct f8 {
    float4 a, b;
};

// PROBE_NA (-DPROBE_NA): the loads skip L1 allocation (.L1::no_allocate), as k_spmm_wide's do
#ifdef PROBE_NA
#define NA ".L1::no_allocate"
#else
#define NA ""
#endif
template <int HINT>  // 0 plain, 1 evict_last, 2 evict_first
__device__ __forceinline__ void ld8(f8& r, const float* p) {
    if (HINT == 1)
        asm volatile("ld.global.nc" NA ".L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else if (HINT == 2)
        asm volatile("ld.global.nc" NA ".L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
    else
        asm volatile("ld.global.nc" NA ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                       "=f"(r.b.z), "=f"(r.b.w)
                     : "l"(p));
}

__device__ __forceinline__ void fma8(f8& acc, float v, const f8& x) {
    acc.a.x = fmaf(v, x.a.x, acc.a.x); acc.a.y = fmaf(v, x.a.y, acc.a.y);
    acc.a.z = fmaf(v, x.a.z, acc.a.z); acc.a.w = fmaf(v, x.a.w, acc.a.w);
    acc.b.x = fmaf(v, x.b.x, acc.b.x); acc.b.y = fmaf(v, x.b.y, acc.b.y);
    acc.b.z = fmaf(v, x.b.z, acc.b.z); acc.b.w = fmaf(v, x.b.w, acc.b.w);
}

// ENC: decode c < 0 -> Xh row ~c; HINTS: hot evict_last / cold evict_first; VALS: read a vals
// stream; STORE: one output row per combined warp and step.
template <int U, int MINB, bool ENC, bool HINTS, bool VALS, bool STORE>
__global__ void __launch_bounds__(256, MINB)
    k_stream(const float* __restrict__ X, const float* __restrict__ Xh, const int* __restrict__ idx,
             const float* __restrict__ vals, int64_t n, int CH, float* __restrict__ out, int64_t out_rows,
             int64_t zero_rows) {
    const int lane = threadIdx.x & 31, s = lane >> 3, li = lane & 7;
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), W = (int64_t)gridDim.x * 8;
    const int part = CH / 4;
    f8 acc;
    acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t step = gw; step * CH < n; step += W) {
        const int64_t b0 = step * CH + (int64_t)s * part;
        const int64_t myend = b0 + part < n ? b0 + part : n;
        int c = 0, cn = 0;
        float v = 1.f, vn = 1.f;
        if (b0 + li < myend) {
            c = __ldcs(idx + b0 + li);
            if (VALS) v = __ldcs(vals + b0 + li);
        }
        for (int base = 0; base < part; base += 8) {
            const int64_t jn = b0 + base + 8 + li;
            if (base + 8 < part && jn < myend) {
                cn = __ldcs(idx + jn);
                if (VALS) vn = __ldcs(vals + jn);
            }
            const int64_t nb = myend - (b0 + base);
#pragma unroll
            for (int q = 0; q < 8; q += U) {
                f8 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int cu = __shfl_sync(0xffffffffu, c, s * 8 + q + u);
                    if (q + u < nb) {
                        if (ENC && cu < 0) {
                            if (HINTS) ld8<1>(x[u], Xh + (int64_t)(~cu) * 64 + li * 8);
                            else ld8<0>(x[u], Xh + (int64_t)(~cu) * 64 + li * 8);
                        } else {
                            if (HINTS) ld8<2>(x[u], X + (int64_t)cu * 64 + li * 8);
                            else ld8<0>(x[u], X + (int64_t)cu * 64 + li * 8);
                        }
                    } else {
                        x[u].a = x[u].b = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float vu = VALS ? __shfl_sync(0xffffffffu, v, s * 8 + q + u) : 1.f;
                    fma8(acc, vu, x[u]);
                }
            }
            c = cn;
            v = vn;
        }
        if (STORE) {
            float* o = out + ((step * 4 + s) % out_rows) * 64 + li * 8;
            __stcs(reinterpret_cast<float4*>(o), acc.a);
            __stcs(reinterpret_cast<float4*>(o) + 1, acc.b);
            acc.a = acc.b = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    if (STORE) {  // the rest of the output rows (the SpMM's zero rows), after the stream
        const int64_t done = ((n + CH - 1) / CH) * 4;
        for (int64_t r = done + gw * 4 + s; r < done + zero_rows; r += W * 4) {
            float* o = out + (r % out_rows) * 64 + li * 8;
            __stcs(reinterpret_cast<float4*>(o), make_float4(0.f, 0.f, 0.f, 0.f));
            __stcs(reinterpret_cast<float4*>(o) + 1, make_float4(0.f, 0.f, 0.f, 0.f));
        }
    }
    if (!STORE) {  // keep the loads alive
        float t = acc.a.x + acc.a.y + acc.a.z + acc.a.w + acc.b.x + acc.b.y + acc.b.z + acc.b.w;
        if (t == 123.456f) out[0] = t;
    }
}

template <int U, int MINB, bool ENC, bool HINTS, bool VALS, bool STORE>
int run_t(const float* X, const float* Xh, const int* idx, const float* vals, int64_t n, int CH, float* out,
          int64_t out_rows, cudaStream_t st, int64_t zero_rows = 0) {
    auto k = k_stream<U, MINB, ENC, HINTS, VALS, STORE>;
    int occ = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
    k<<<sms * occ, 256, 0, st>>>(X, Xh, idx, vals, n, CH, out, out_rows, zero_rows);
    return cudaGetLastError() == cudaSuccess ? occ : -1;
}

template <int U, int MINB, bool ENC, bool HINTS>
int run_v(int vs, const float* X, const float* Xh, const int* idx, const float* vals, int64_t n, int CH,
          float* out, int64_t out_rows, cudaStream_t st) {
    return vs ? run_t<U, MINB, ENC, HINTS, true, true>(X, Xh, idx, vals, n, CH, out, out_rows, st)
              : run_t<U, MINB, ENC, HINTS, false, false>(X, Xh, idx, vals, n, CH, out, out_rows, st);
}

template <int U, int MINB>
int run_u(int enc, int hints, int vs, const float* X, const float* Xh, const int* idx, const float* vals,
          int64_t n, int CH, float* out, int64_t out_rows, cudaStream_t st) {
    if (!enc) return run_v<U, MINB, false, false>(vs, X, Xh, idx, vals, n, CH, out, out_rows, st);
    return hints ? run_v<U, MINB, true, true>(vs, X, Xh, idx, vals, n, CH, out, out_rows, st)
                 : run_v<U, MINB, true, false>(vs, X, Xh, idx, vals, n, CH, out, out_rows, st);
}

}  // namespace

// shape: 0 = U 4 at 3 CTAs/SM (the SpMM's default), 1 = U 2 at 4 CTAs/SM, 2 = U 4 at 4, 3 = U 8 at 2,
// 4 = U 2 at 8 CTAs/SM.  Returns the CTAs per SM launched, -1 on a launch error.
extern "C" int probe_stream(int shape, int enc, int hints, int vals_store, const float* X, const float* Xh,
                            const int* idx, const float* vals, int64_t n, int CH, float* out,
                            int64_t out_rows, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (shape) {
        case 1: return run_u<2, 4>(enc, hints, vals_store, X, Xh, idx, vals, n, CH, out, out_rows, st);
        case 2: return run_u<4, 4>(enc, hints, vals_store, X, Xh, idx, vals, n, CH, out, out_rows, st);
        case 3: return run_u<8, 2>(enc, hints, vals_store, X, Xh, idx, vals, n, CH, out, out_rows, st);
        case 4: return run_u<2, 8>(enc, hints, vals_store, X, Xh, idx, vals, n, CH, out, out_rows, st);
        default: return run_u<4, 3>(enc, hints, vals_store, X, Xh, idx, vals, n, CH, out, out_rows, st);
    }
}

// the kernel-matched variant: U 4 at 3 CTAs/SM, hot/cold hints, vals stream, output-row stores
// plus `zero_rows` more zero rows after the stream (the SpMM's degree-0 rows)
extern "C" int probe_stream_full(const float* X, const float* Xh, const int* idx, const float* vals, int64_t n,
                                 int CH, float* out, int64_t out_rows, int64_t zero_rows, int hints, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    return hints ? run_t<4, 3, true, true, true, true>(X, Xh, idx, vals, n, CH, out, out_rows, st, zero_rows)
                 : run_t<4, 3, true, false, true, true>(X, Xh, idx, vals, n, CH, out, out_rows, st, zero_rows);
}

// persisting-L2 window over [base, base + bytes) on `stream` (hitRatio 1), after setting the
// set-aside to `setaside` bytes; bytes = 0 clears the window.
extern "C" int probe_window(void* stream, const void* base, size_t bytes, size_t setaside) {
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside) != cudaSuccess) return -1;
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = bytes ? 1.0f : 0.f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) return -2;
    if (!bytes) cudaCtxResetPersistingL2Cache();
    return 0;
}
