// Zero-copy random-row read probe: does the PTX cache operator of the 16-B
// host loads change how many bytes cross the host link (ncu pcie__read_bytes)
// and the useful rate? 400-B rows, sorted random IDs, warp per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc tools/zc_probe.cu && /tmp/zc
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); exit(1); } } while (0)

template <int V>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    uint4 r;
    if (V == 0) asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 2) asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 3) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 4) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 5) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 6) asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    if (V == 7) asm volatile("ld.global.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int V>
__global__ void __launch_bounds__(256) gather(const int32_t* __restrict__ ids, int m, const uint4* __restrict__ tab,
                                              int row16, uint4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < m; i += 2 * nw) {
        const int j = i + nw;
        uint4 a = make_uint4(0, 0, 0, 0), b = a;
        if (lane < row16) a = ld16<V>(tab + (int64_t)ids[i] * row16 + lane);
        if (j < m && lane < row16) b = ld16<V>(tab + (int64_t)ids[j] * row16 + lane);
        if (lane < row16) out[(int64_t)i * row16 + lane] = a;
        if (j < m && lane < row16) out[(int64_t)j * row16 + lane] = b;
    }
}

template <int V>
float run(const int32_t* ids, int m, const uint4* tab, int row16, uint4* out, int ctas) {
    cudaEvent_t s, e;
    CK(cudaEventCreate(&s));
    CK(cudaEventCreate(&e));
    float best = 1e9f;
    for (int it = 0; it < 5; ++it) {
        CK(cudaEventRecord(s));
        gather<V><<<ctas, 256>>>(ids, m, tab, row16, out);
        CK(cudaEventRecord(e));
        CK(cudaEventSynchronize(e));
        float ms;
        CK(cudaEventElapsedTime(&ms, s, e));
        if (it) best = std::min(best, ms);
    }
    return best;
}

int main(int argc, char** argv) {
    const int64_t n = 2400000;
    const int rb = 400, row16 = rb / 16;
    const int m = argc > 1 ? atoi(argv[1]) : 87000;
    void* host;
    CK(cudaHostAlloc(&host, n * rb, cudaHostAllocMapped));
    memset(host, 1, n * rb);
    void* dtab;
    CK(cudaHostGetDevicePointer(&dtab, host, 0));
    std::mt19937_64 g(1);
    std::vector<int32_t> h(m);
    for (auto& x : h) x = (int32_t)(g() % n);
    std::sort(h.begin(), h.end());
    int32_t* ids;
    uint4* out;
    CK(cudaMalloc(&ids, m * 4));
    CK(cudaMalloc(&out, (size_t)m * rb));
    CK(cudaMemcpy(ids, h.data(), m * 4, cudaMemcpyHostToDevice));
    const int ctas = 296;
    float t[8] = {run<0>(ids, m, (const uint4*)dtab, row16, out, ctas), run<1>(ids, m, (const uint4*)dtab, row16, out, ctas),
                  run<2>(ids, m, (const uint4*)dtab, row16, out, ctas), run<3>(ids, m, (const uint4*)dtab, row16, out, ctas),
                  run<4>(ids, m, (const uint4*)dtab, row16, out, ctas), run<5>(ids, m, (const uint4*)dtab, row16, out, ctas),
                  run<6>(ids, m, (const uint4*)dtab, row16, out, ctas), run<7>(ids, m, (const uint4*)dtab, row16, out, ctas)};
    const char* names[8] = {"ld.global", "ld.global.cg", "ld.global.cs", "ld.global.cv", "ld.global.nc.L1::no_allocate",
                            "ld.volatile.global", "ld.global.L2::64B", "ld.global.L2::256B"};
    for (int v = 0; v < 8; ++v)
        printf("%-45s %8.1f us  %6.2f GB/s useful  %6.1f M rows/s\n", names[v], t[v] * 1e3, (double)m * rb / (t[v] * 1e-3) / 1e9,
               m / (t[v] * 1e-3) / 1e6);
    return 0;
}
