// Host-link read rate of spans of S contiguous bytes at random 16-B-aligned
// offsets of pinned (mapped) host memory: SM 16-B loads (warp per span) vs
// TMA bulk copies (cp.async.bulk global->shared, one elected thread, then a
// bulk store to the output) vs one big cudaMemcpy. Question: do large TMA
// bulk reads issue bigger PCIe requests than SM loads (payload efficiency)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void sm_spans(const char* __restrict__ host, const int64_t* __restrict__ offs, int n, int S, char* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
        const uint4* s = (const uint4*)(host + offs[i]);
        uint4* d = (uint4*)(out + i * S);
        for (int c = lane; c < S / 16; c += 32) d[c] = __ldg(s + c);
    }
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// one warp per CTA; lane 0 issues; 2 stages of S bytes in smem
__global__ void tma_spans(const char* __restrict__ host, const int64_t* __restrict__ offs, int n, int S, char* out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned phase[2] = {0, 0};
    int it = 0;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x, ++it) {
        const int s = it & 1;
        char* buf = sm + s * S;
        // the store that last used this stage must have read the smem
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&bar[s])), "r"(S));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_addr(buf)), "l"(host + offs[i]), "r"(S), "r"(smem_addr(&bar[s])) : "memory");
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                     :: "r"(smem_addr(&bar[s])), "r"(phase[s]));
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(out + i * S), "r"(smem_addr(buf)), "r"(S) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
    }
    asm volatile("cp.async.bulk.wait_group 0;");
}

// TMA with D loads in flight per CTA (D stages), lane 0 issues all
template <int D>
__global__ void tma_spans_deep(const char* __restrict__ host, const int64_t* __restrict__ offs, int n, int S, char* out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[D];
    if (threadIdx.x == 0) {
        for (int s = 0; s < D; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned ph = 0;
    for (int64_t i0 = blockIdx.x * (int64_t)D; i0 < n; i0 += (int64_t)gridDim.x * D) {
        const int cnt = (int)((n - i0) < D ? (n - i0) : D);
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        for (int s = 0; s < cnt; ++s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&bar[s])), "r"(S));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(smem_addr(sm + s * S)), "l"(host + offs[i0 + s]), "r"(S), "r"(smem_addr(&bar[s])) : "memory");
        }
        for (int s = 0; s < cnt; ++s) {
            asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                         :: "r"(smem_addr(&bar[s])), "r"(ph));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(out + (i0 + s) * S), "r"(smem_addr(sm + s * S)), "r"(S) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;");
        ph ^= 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;");
}

int main() {
    const size_t HB = (size_t)2 << 30;
    char* h;
    CK(cudaHostAlloc(&h, HB, cudaHostAllocMapped));
    for (size_t i = 0; i < HB; i += 4096) h[i] = (char)i;
    char* hd;
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    const size_t total = (size_t)256 << 20;
    char* out;
    CK(cudaMalloc(&out, total + (1 << 20)));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    {
        char* d;
        CK(cudaMalloc(&d, total));
        for (int r = 0; r < 2; ++r) cudaMemcpy(d, h, total, cudaMemcpyHostToDevice);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 256MB: %.2f GB/s\n", 5.0 * total / (ms * 1e-3) / 1e9);
        cudaFree(d);
    }
    const int Ss[] = {400, 800, 1600, 3200, 6400, 12800};
    for (int S : Ss) {
        const int n = (int)(total / S);
        int64_t* ho = (int64_t*)malloc(n * 8);
        srand(7);
        for (int i = 0; i < n; ++i) ho[i] = ((int64_t)(((uint64_t)rand() << 16) ^ rand()) % (int64_t)((HB - S) / 16)) * 16;
        int64_t* dof;
        CK(cudaMalloc(&dof, n * 8));
        CK(cudaMemcpy(dof, ho, n * 8, cudaMemcpyHostToDevice));
        auto run = [&](const char* nm, auto fn) {
            fn();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) fn();
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("S=%5d %-22s %.2f GB/s\n", S, nm, 3.0 * n * S / (ms * 1e-3) / 1e9);
        };
        run("sm warp/span g592", [&] { sm_spans<<<592, 256>>>(hd, dof, n, S, out); });
        run("sm warp/span g1184", [&] { sm_spans<<<1184, 256>>>(hd, dof, n, S, out); });
        CK(cudaFuncSetAttribute(tma_spans, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 12800));
        run("tma 2-stage g1184", [&] { tma_spans<<<1184, 32, 2 * S>>>(hd, dof, n, S, out); });
        run("tma 2-stage g2368", [&] { tma_spans<<<2368, 32, 2 * S>>>(hd, dof, n, S, out); });
        CK(cudaFuncSetAttribute(tma_spans_deep<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 12800));
        run("tma 8-deep g592", [&] { tma_spans_deep<8><<<592, 32, 8 * S>>>(hd, dof, n, S, out); });
        run("tma 8-deep g1184", [&] { tma_spans_deep<8><<<1184, 32, 8 * S>>>(hd, dof, n, S, out); });
        CK(cudaGetLastError());
        cudaFree(dof);
        free(ho);
    }
    return 0;
}
