// Zero-copy random-row gather rate vs the pinned store's footprint and page
// size: is the papers100M-shaped miss gather (57 GB store) translation-bound,
// and do transparent huge pages (madvise + cudaHostRegister) help?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlb_probe_bin tools/tlb_probe.cu
//   tools/tlb_probe_bin <footprint GB> <row bytes> <thp 0|1>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <random>
#include <sys/mman.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); exit(1); } } while (0)

__global__ void __launch_bounds__(256) gather(const int64_t* __restrict__ ids, int m, const uint4* __restrict__ tab,
                                              int row16, uint4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < m; i += 2 * nw) {
        const int j = i + nw;
        for (int c = lane; c < row16; c += 32) {
            uint4 a = tab[ids[i] * row16 + c], b = make_uint4(0, 0, 0, 0);
            if (j < m) b = tab[ids[j] * row16 + c];
            out[(int64_t)i * row16 + c] = a;
            if (j < m) out[(int64_t)j * row16 + c] = b;
        }
    }
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 1.0;
    const int rb = argc > 2 ? atoi(argv[2]) : 512;
    const int thp = argc > 3 ? atoi(argv[3]) : 0;
    const size_t bytes = ((size_t)(gb * (1ull << 30)) / (2u << 20)) * (2u << 20);
    const int64_t n = bytes / rb;
    const int m = 150000;
    void* host = nullptr;
    if (thp) {
        host = aligned_alloc(2u << 20, bytes);
        if (madvise(host, bytes, MADV_HUGEPAGE) != 0) perror("madvise");
        for (size_t i = 0; i < bytes; i += 4096) ((char*)host)[i] = 1;
        CK(cudaHostRegister(host, bytes, cudaHostRegisterMapped));
    } else {
        CK(cudaHostAlloc(&host, bytes, cudaHostAllocMapped));
        for (size_t i = 0; i < bytes; i += 4096) ((char*)host)[i] = 1;
    }
    void* dtab;
    CK(cudaHostGetDevicePointer(&dtab, host, 0));
    std::mt19937_64 g(1);
    std::vector<int64_t> h(m);
    for (auto& x : h) x = (int64_t)(g() % n);
    std::sort(h.begin(), h.end());
    int64_t* ids;
    uint4* out;
    CK(cudaMalloc(&ids, m * 8));
    CK(cudaMalloc(&out, (size_t)m * rb));
    CK(cudaMemcpy(ids, h.data(), m * 8, cudaMemcpyHostToDevice));
    cudaEvent_t s, e;
    CK(cudaEventCreate(&s));
    CK(cudaEventCreate(&e));
    float best = 1e9f;
    for (int it = 0; it < 6; ++it) {
        CK(cudaEventRecord(s));
        gather<<<296, 256>>>(ids, m, (const uint4*)dtab, rb / 16, out);
        CK(cudaEventRecord(e));
        CK(cudaEventSynchronize(e));
        float ms;
        CK(cudaEventElapsedTime(&ms, s, e));
        if (it) best = std::min(best, ms);
    }
    FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[128] = "?";
    if (f) { if (!fgets(buf, sizeof buf, f)) buf[0] = 0; fclose(f); }
    buf[strcspn(buf, "\n")] = 0;
    printf("footprint %6.1f GB rows %4d B thp %d [%s]: %7.1f us  %6.2f GB/s useful  %6.1f M rows/s\n", bytes / 1e9 * 1.073741824 / 1.073741824,
           rb, thp, buf, best * 1e3, (double)m * rb / (best * 1e-3) / 1e9, m / (best * 1e-3) / 1e6);
    return 0;
}
