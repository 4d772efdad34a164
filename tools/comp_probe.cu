// comp_probe.cu -- does generic compressible memory (cuMemCreate, CU_MEM_ALLOCATION_COMP_GENERIC)
// cut the DRAM cost of the SpMM's zero-row stores?  C5-shaped: Y = 8.4M rows x 256 B, 54 % of
// the rows (random) written as zeros, the rest with data; times (CUDA events, median of 9) the
// zero-row stores alone, the data-row stores alone, both, and a random 256-B row gather over
// the result, each on plain cudaMalloc memory and on compressible memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o comp_probe tools/comp_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
    printf("%s failed: %s\n", #x, s); exit(1); } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); exit(1); } } while (0)

__global__ void k_store_rows(float* Y, const int* rows, int64_t nrows, int F, float val) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lanes = F / 4;
    const int64_t r = t / lanes;
    if (r >= nrows) return;
    const int l = (int)(t % lanes);
    const float v = val == 0.f ? 0.f : val * (float)(r % 977);
    __stcs(reinterpret_cast<float4*>(Y + (int64_t)rows[r] * F) + l, make_float4(v, v + 1, v + 2, v + 3));
}

__global__ void k_gather_rows(const float* X, const int* cols, int64_t m, int F, float* out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lanes = F / 4;
    const int64_t e = t / lanes;
    if (e >= m) return;
    const int l = (int)(t % lanes);
    float4 x = __ldg(reinterpret_cast<const float4*>(X + (int64_t)cols[e] * F) + l);
    if (x.x == 12345.f) out[0] = x.y;  // keep the load
}

static float* alloc_comp(size_t bytes, bool comp, CUmemGenericAllocationHandle* h, size_t* sz) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    prop.allocFlags.compressionType = comp ? CU_MEM_ALLOCATION_COMP_GENERIC : 0;
    size_t gran = 0;
    CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    bytes = (bytes + gran - 1) / gran * gran;
    CK(cuMemCreate(h, bytes, &prop, 0));
    CUmemAllocationProp got = {};
    CK(cuMemGetAllocationPropertiesFromHandle(&got, *h));
    printf("  alloc %zu MB comp requested %d granted %d (granularity %zu)\n", bytes >> 20, (int)comp,
           (int)got.allocFlags.compressionType, gran);
    CUdeviceptr p;
    CK(cuMemAddressReserve(&p, bytes, 0, 0, 0));
    CK(cuMemMap(p, bytes, 0, *h, 0));
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(p, bytes, &acc, 1));
    *sz = bytes;
    return reinterpret_cast<float*>(p);
}

template <class F>
static float time_ms(F f, cudaStream_t s) {
    std::vector<float> v;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) {
        cudaEventRecord(a, s);
        f();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i) v.push_back(ms);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

int main() {
    CK(cuInit(0));
    RK(cudaFree(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int sup = 0;
    CK(cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev));
    printf("generic compression supported: %d\n", sup);
    const int64_t n = 1 << 23;
    const int F = 64;
    const size_t bytes = (size_t)n * F * 4;
    std::mt19937_64 rng(5);
    std::vector<int> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = (int)i;
    std::shuffle(perm.begin(), perm.end(), rng);
    const int64_t nz = (int64_t)(0.541 * n);  // C5: 54.1 % degree-0 rows
    std::sort(perm.begin(), perm.begin() + nz);
    std::sort(perm.begin() + nz, perm.end());
    int *d_rows, *d_cols;
    RK(cudaMalloc(&d_rows, sizeof(int) * n));
    RK(cudaMemcpy(d_rows, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    const int64_t m = 1 << 26;
    std::vector<int> cols(m);
    for (auto& c : cols) c = (int)(rng() % n);
    RK(cudaMalloc(&d_cols, sizeof(int) * m));
    RK(cudaMemcpy(d_cols, cols.data(), sizeof(int) * m, cudaMemcpyHostToDevice));
    float* d_out;
    RK(cudaMalloc(&d_out, 64));
    void* scratch;
    RK(cudaMalloc(&scratch, 512 << 20));
    cudaStream_t s = 0;
    for (int comp = 0; comp < 2; ++comp) {
        if (comp && !sup) break;
        CUmemGenericAllocationHandle h;
        size_t sz;
        float* Y = alloc_comp(bytes, comp, &h, &sz);
        const int64_t tz = nz * (F / 4), td = (n - nz) * (F / 4), tg = m * (F / 4);
        auto zero = [&] { k_store_rows<<<(unsigned)((tz + 255) / 256), 256, 0, s>>>(Y, d_rows, nz, F, 0.f); };
        auto data = [&] { k_store_rows<<<(unsigned)((td + 255) / 256), 256, 0, s>>>(Y, d_rows + nz, n - nz, F, 1.f); };
        auto gath = [&] { k_gather_rows<<<(unsigned)((tg + 255) / 256), 256, 0, s>>>(Y, d_cols, m, F, d_out); };
        auto flush = [&] { cudaMemsetAsync(scratch, comp, 512 << 20, s); };
        float tzr = time_ms([&] { zero(); }, s);
        float tdt = time_ms([&] { data(); }, s);
        float tbo = time_ms([&] { zero(); data(); }, s);
        data();
        zero();
        float tgt = time_ms([&] { gath(); }, s);
        flush();
        RK(cudaStreamSynchronize(s));
        float tzc = time_ms([&] { flush(); zero(); }, s) - time_ms([&] { flush(); }, s);
        printf("%s: zero rows %.3f ms (%.2f TB/s of rows)  data rows %.3f ms  both %.3f ms  "
               "zero after flush %.3f ms  gather 2^26 rows %.3f ms (%.2f TB/s)\n",
               comp ? "compressible" : "plain       ", tzr, nz * F * 4.0 / tzr / 1e9, tdt, tbo, tzc, tgt,
               m * F * 4.0 / tgt / 1e9);
        RK(cudaGetLastError());
        CK(cuMemUnmap((CUdeviceptr)Y, sz));
        CK(cuMemRelease(h));
        CK(cuMemAddressFree((CUdeviceptr)Y, sz));
    }
    return 0;
}
