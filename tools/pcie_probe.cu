// pcie_probe.cu -- host<->device copy bandwidth from pinned memory: one copy vs the same bytes
// split into k chunks on k streams (copy engines), H2D alone, D2H alone, and both directions at
// once (the e2e executor's overlap).  1 GiB per direction, median of 5.
//   nvcc -O3 -o pcie_probe tools/pcie_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
    const size_t B = 1ull << 30;
    void *h_in, *h_out, *d_in, *d_out;
    RK(cudaMallocHost(&h_in, B));
    RK(cudaMallocHost(&h_out, B));
    RK(cudaMalloc(&d_in, B));
    RK(cudaMalloc(&d_out, B));
    cudaStream_t st[8];
    for (auto& s : st) RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {          // 0 H2D, 1 D2H, 2 both
        for (int k : {1, 2, 4, 8}) {
            std::vector<float> v;
            for (int rep = 0; rep < 6; ++rep) {
                RK(cudaDeviceSynchronize());
                cudaEventRecord(a, 0);
                for (int i = 0; i < k; ++i) cudaStreamWaitEvent(st[i], a, 0);
                const size_t c = B / k;
                for (int i = 0; i < k; ++i) {
                    if (mode != 1)
                        cudaMemcpyAsync((char*)d_in + i * c, (char*)h_in + i * c, c, cudaMemcpyHostToDevice, st[i]);
                    if (mode != 0)
                        cudaMemcpyAsync((char*)h_out + i * c, (char*)d_out + i * c, c, cudaMemcpyDeviceToHost,
                                        st[(i + (mode == 2 ? k / 2 : 0)) % k]);
                }
                for (int i = 0; i < k; ++i) {
                    cudaEvent_t e;
                    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
                    cudaEventRecord(e, st[i]);
                    cudaStreamWaitEvent(0, e, 0);
                    cudaEventDestroy(e);
                }
                cudaEventRecord(b, 0);
                RK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) v.push_back(ms);
            }
            std::sort(v.begin(), v.end());
            const float ms = v[v.size() / 2];
            printf("%s streams %d: %.2f ms  %.1f GB/s per direction\n", mode == 0 ? "H2D " : mode == 1 ? "D2H " : "both",
                   k, ms, B / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
