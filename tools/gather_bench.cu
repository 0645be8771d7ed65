// Microbenchmark of miss-row fetch strategies from pinned host memory
// (zero-copy over PCIe) on the B200. Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint4 ld_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// A: flattened 16B chunks, unroll U
template <int U>
__global__ void gather_flat(const int* ids, int n, const char* table, int rb, char* out) {
    int64_t cpr = rb / 16, total = (int64_t)n * cpr, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < total; c0 += stride * U) {
        uint4 v[U]; int64_t dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t c = c0 + u * stride; dst[u] = -1;
            if (c < total) { int64_t r = c / cpr, p = c - r * cpr; v[u] = ld_nc(table + (int64_t)ids[r] * rb + p * 16); dst[u] = r * rb + p * 16; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) if (dst[u] >= 0) *(uint4*)(out + dst[u]) = v[u];
    }
}

// B: warp per row, lanes < cpr load one 16B chunk; R rows per warp in flight
template <int R>
__global__ void gather_warp(const int* ids, int n, const char* table, int rb, char* out) {
    int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int cpr = rb / 16;
    for (int64_t r0 = w * R; r0 < n; r0 += nw * R) {
        uint4 v[R];
#pragma unroll
        for (int u = 0; u < R; ++u) if (r0 + u < n && lane < cpr) v[u] = ld_nc(table + (int64_t)ids[r0 + u] * rb + lane * 16);
#pragma unroll
        for (int u = 0; u < R; ++u) if (r0 + u < n && lane < cpr) *(uint4*)(out + (r0 + u) * rb + lane * 16) = v[u];
    }
}

// C: TMA bulk copies (cp.async.bulk) host row -> smem, then smem -> out
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes) : "memory");
}

template <int ROWS, int STAGES>
__global__ void gather_tma(const int* ids, int n, const char* table, int rb, char* out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bars[STAGES];
    const int stage_bytes = ROWS * rb;
    if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    int64_t ngroups = (n + ROWS - 1) / ROWS;
    int it = 0;
    // single producer thread issues; all threads then copy out via bulk store by thread 0
    for (int64_t g0 = blockIdx.x; g0 < ngroups; g0 += (int64_t)gridDim.x * STAGES) {
        int issued = 0;
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                int64_t g = g0 + (int64_t)s * gridDim.x;
                if (g >= ngroups) break;
                int64_t r0 = g * ROWS; int nr = (int)((n - r0) < ROWS ? (n - r0) : ROWS);
                mbar_expect(&bars[s], nr * rb);
                for (int r = 0; r < nr; ++r) bulk_g2s(sm + s * stage_bytes + r * rb, table + (int64_t)ids[r0 + r] * rb, rb, &bars[s]);
                issued++;
            }
            for (int s = 0; s < issued; ++s) {
                mbar_wait(&bars[s], it & 1);
                int64_t g = g0 + (int64_t)s * gridDim.x; int64_t r0 = g * ROWS; int nr = (int)((n - r0) < ROWS ? (n - r0) : ROWS);
                bulk_s2g(out + r0 * rb, sm + s * stage_bytes, nr * rb);
            }
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;");
        }
        it++;
        __syncthreads();
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;");
}

int small_grid_sweep(const int* dids, int n, const char* dtab, int rb, char* out);
int main(int argc, char** argv) {
    const int64_t nn = 2400000; const int rb = argc > 1 ? atoi(argv[1]) : 400; const int n = argc > 2 ? atoi(argv[2]) : 84000;
    char* table; CK(cudaHostAlloc(&table, nn * rb, cudaHostAllocMapped));
    for (int64_t i = 0; i < nn * rb; i += 4096) table[i] = (char)i;
    std::mt19937_64 g(1); std::vector<int> ids(n);
    for (auto& x : ids) x = (int)(g() % nn);
    std::sort(ids.begin(), ids.end());
    int* dids; CK(cudaMalloc(&dids, n * 4)); CK(cudaMemcpy(dids, ids.data(), n * 4, cudaMemcpyHostToDevice));
    char* out; CK(cudaMalloc(&out, (int64_t)n * rb));
    char* dtab; CK(cudaHostGetDevicePointer((void**)&dtab, table, 0));
    char* hbuf; CK(cudaMalloc(&hbuf, (size_t)n * rb));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a); for (int i = 0; i < 20; ++i) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        printf("%-28s %8.3f ms  %7.2f GB/s\n", name, ms, (double)n * rb / (ms * 1e-3) / 1e9);
    };
    // reference: one big memcpy of the same byte count
    timeit("memcpy H2D contiguous", [&] { cudaMemcpyAsync(hbuf, table, (size_t)n * rb, cudaMemcpyHostToDevice); });
    if (argc > 3) return small_grid_sweep(dids, n, dtab, rb, out);
    for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
        char nm[64];
        snprintf(nm, 64, "flat U4 grid %d", grid); timeit(nm, [&] { gather_flat<4><<<grid, 256>>>(dids, n, dtab, rb, out); });
        snprintf(nm, 64, "flat U8 grid %d", grid); timeit(nm, [&] { gather_flat<8><<<grid, 256>>>(dids, n, dtab, rb, out); });
        snprintf(nm, 64, "warp R4 grid %d", grid); timeit(nm, [&] { gather_warp<4><<<grid, 256>>>(dids, n, dtab, rb, out); });
        snprintf(nm, 64, "warp R8 grid %d", grid); timeit(nm, [&] { gather_warp<8><<<grid, 256>>>(dids, n, dtab, rb, out); });
    }
    {   // HBM-resident table: 250K random rows
        char* dt; CK(cudaMalloc(&dt, nn * rb));
        CK(cudaMemset(dt, 1, nn * rb));
        int n2 = 250000; std::vector<int> ids2(n2); for (auto& x : ids2) x = (int)(g() % nn); std::sort(ids2.begin(), ids2.end());
        int* d2; CK(cudaMalloc(&d2, n2 * 4)); CK(cudaMemcpy(d2, ids2.data(), n2 * 4, cudaMemcpyHostToDevice));
        char* o2; CK(cudaMalloc(&o2, (int64_t)n2 * rb));
        auto t2 = [&](const char* name, auto fn) {
            for (int i = 0; i < 3; ++i) fn();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a); for (int i = 0; i < 20; ++i) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
            printf("HBM %-24s %8.3f ms  %7.1f GB/s (r+w)\n", name, ms, 2.0 * n2 * rb / (ms * 1e-3) / 1e9);
        };
        for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
            char nm[64];
            snprintf(nm, 64, "flat U4 grid %d", grid); t2(nm, [&] { gather_flat<4><<<grid, 256>>>(d2, n2, dt, rb, o2); });
            snprintf(nm, 64, "warp R4 grid %d", grid); t2(nm, [&] { gather_warp<4><<<grid, 256>>>(d2, n2, dt, rb, o2); });
            snprintf(nm, 64, "warp R8 grid %d", grid); t2(nm, [&] { gather_warp<8><<<grid, 256>>>(d2, n2, dt, rb, o2); });
        }
    }
    for (int grid : {148, 148 * 2, 148 * 4}) {
        char nm[64];
        {
            const int ROWS = 16, ST = 4; size_t sm = ROWS * rb * ST;
            CK(cudaFuncSetAttribute(gather_tma<ROWS, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            snprintf(nm, 64, "tma 16x4 grid %d", grid); timeit(nm, [&] { gather_tma<ROWS, ST><<<grid, 32, sm>>>(dids, n, dtab, rb, out); });
        }
        {
            const int ROWS = 32, ST = 8; size_t sm = ROWS * rb * ST;
            CK(cudaFuncSetAttribute(gather_tma<ROWS, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            snprintf(nm, 64, "tma 32x8 grid %d", grid); timeit(nm, [&] { gather_tma<ROWS, ST><<<grid, 32, sm>>>(dids, n, dtab, rb, out); });
        }
    }
    CK(cudaGetLastError());
    return 0;
}
// (appended) small-grid sweep for the host-link gather: how few warps saturate PCIe
int small_grid_sweep(const int* dids, int n, const char* dtab, int rb, char* out) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int threads : {64, 128, 256}) for (int grid : {37, 74, 148, 296}) {
        for (int i = 0; i < 3; ++i) gather_warp<4><<<grid, threads>>>(dids, n, dtab, rb, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a); for (int i = 0; i < 20; ++i) gather_warp<4><<<grid, threads>>>(dids, n, dtab, rb, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        printf("warp R4 grid %4d x %3d thr  %8.3f ms  %7.2f GB/s\n", grid, threads, ms, (double)n * rb / (ms * 1e-3) / 1e9);
    }
    return 0;
}
