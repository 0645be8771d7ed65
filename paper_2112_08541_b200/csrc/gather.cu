// K5/K6: feature-row gather for a mini-batch (net-new: the reference only
// counts bytes, cachesim.py:261-272; contract rows[i] = F[batch[i]]).
//
// out[i] = src_row[i] >= 0 ? ring_rows[src_row[i]]   (cache hit, HBM)
//                          : table[ids[i]]            (miss: zero-copy read of
//                                                      pinned host memory over
//                                                      the host link, or HBM)
// Warp per row: every load instruction of a warp touches exactly one row
// (400 B = 25 lanes x 16 B), which keeps the host-link read requests whole
// (measured on the box: 45.6 GB/s of zero-copy reads of random 400-byte rows
// vs 42.8 GB/s for a flat chunk mapping; HBM: 5.1 vs 4.3 TB/s r+w), and
// kRows rows per warp are in flight at once. `mode` selects all rows, only
// cache hits (src_row >= 0) or only misses (src_row < 0), so hits (HBM) and
// misses (host link) can run as separate kernels.
#include "common.cuh"

namespace bgl {

constexpr int kGThreads = 256;

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_na_v4(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ const unsigned char* row_src(int64_t row, const int32_t* ids, const int64_t* src_row,
                                                        const unsigned char* ring, const unsigned char* table,
                                                        int64_t rb) {
    int64_t s = src_row ? __ldg(src_row + row) : -1;
    return s >= 0 ? ring + s * rb : table + (int64_t)__ldg(ids + row) * rb;
}

constexpr int kRows = 4;

__global__ void __launch_bounds__(kGThreads)
gather_v4_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ src_row,
                 const int64_t* __restrict__ n_dev, const unsigned char* __restrict__ ring,
                 const unsigned char* __restrict__ table, int64_t rb, unsigned char* __restrict__ out, int mode,
                 unsigned char* __restrict__ push_out, const int32_t* __restrict__ push_pos) {
    const int64_t n = *n_dev;
    const int cpr = (int)(rb >> 4);
    const int lane = lane_id();
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = w * kRows; r0 < n; r0 += nw * kRows) {
        const unsigned char* src[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            src[u] = nullptr;
            const int64_t r = r0 + u;
            if (r < n) {
                const int64_t s = src_row ? __ldg(src_row + r) : -1;
                const bool take = mode == 0 || (mode == 1 ? s >= 0 : s < 0);
                if (take) src[u] = s >= 0 ? ring + s * rb : table + (int64_t)__ldg(ids + r) * rb;
            }
        }
        for (int c = lane; c < cpr; c += 32) {
            uint4 v[kRows];
#pragma unroll
            for (int u = 0; u < kRows; ++u)
                if (src[u]) v[u] = ld_nc_v4(src[u] + c * 16);
            if (out) {
#pragma unroll
                for (int u = 0; u < kRows; ++u)
                    if (src[u]) st_na_v4(out + (r0 + u) * rb + c * 16, v[u]);
            }
            if (push_out) {   // home-push: the same row straight into the worker GPU's output (peer memory)
#pragma unroll
                for (int u = 0; u < kRows; ++u)
                    if (src[u])
                        st_na_v4(push_out + (int64_t)__ldg(push_pos + r0 + u) * rb + c * 16, v[u]);
            }
        }
    }
    if (push_out) __threadfence_system();   // peer stores visible system-wide before the caller's barrier
}

// Compacted miss list (bgl_cache_lookup_misses): row j of the list is batch
// position pos[j]; out[pos[j]] = table[ids[pos[j]]]. Every warp keeps R real
// rows in flight (the mode-2 pass above skips the ~2/3 hits of each group of
// kRows and so has ~1.3 rows in flight per warp on the host link).
template <int R>
__global__ void __launch_bounds__(kGThreads)
gather_list_kernel(const int32_t* __restrict__ pos, const int64_t* __restrict__ count_dev,
                   const int32_t* __restrict__ ids, const unsigned char* __restrict__ table, int64_t rb,
                   unsigned char* __restrict__ out, unsigned char* __restrict__ push_out,
                   const int32_t* __restrict__ push_pos) {
    const int64_t n = *count_dev;
    const int cpr = (int)(rb >> 4);
    const int lane = lane_id();
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j0 = w * R; j0 < n; j0 += nw * R) {
        const unsigned char* src[R];
        int64_t dst[R];
        // one lane per row fetches (pos, id); broadcast by shuffle
        int32_t my_p = -1, my_id = 0;
        if (lane < R && j0 + lane < n) {
            my_p = __ldg(pos + j0 + lane);
            my_id = __ldg(ids + my_p);
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int32_t p = __shfl_sync(0xffffffffu, my_p, u);
            const int32_t v = __shfl_sync(0xffffffffu, my_id, u);
            src[u] = p >= 0 ? table + (int64_t)v * rb : nullptr;
            dst[u] = p;
        }
        for (int c = lane; c < cpr; c += 32) {
            uint4 v[R];
#pragma unroll
            for (int u = 0; u < R; ++u)
                if (src[u]) v[u] = ld_nc_v4(src[u] + c * 16);
            if (out) {
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (src[u]) st_na_v4(out + dst[u] * rb + c * 16, v[u]);
            }
            if (push_out) {
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (src[u]) st_na_v4(push_out + (int64_t)__ldg(push_pos + dst[u]) * rb + c * 16, v[u]);
            }
        }
    }
    if (push_out) __threadfence_system();   // peer stores visible system-wide before the caller's barrier
}

// Span-aware miss gather. Proximity ordering puts most misses of a batch in
// runs of consecutive node IDs (C2: ~75% of miss rows in runs >= 2), and in a
// sorted distinct batch consecutive IDs sit at consecutive positions, so a run
// is a contiguous span of the feature store AND of the output. Each warp takes
// kSpanChunk entries of the compacted miss list: single rows go through 16-B
// SM loads (as gather_list_kernel); every run of >= 2 rows is one TMA bulk copy
// host -> shared memory (cp.async.bulk, completion on a per-warp mbarrier) and
// one bulk store shared -> output. Measured on the box (tools/tma_probe.cu):
// bulk reads of 800 / 1600 / 3200-B spans reach 47.4 / 49.4 / 50.4 GB/s of
// the link vs 45.4 for 16-B loads of 400-B rows (the link's completions carry
// more payload per request); single 400-B bulk reads are slower (39.5), hence
// the split.
constexpr int kSpanChunk = 16;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kGThreads)
gather_span_kernel(const int32_t* __restrict__ pos, const int64_t* __restrict__ count_dev,
                   const int32_t* __restrict__ ids, const unsigned char* __restrict__ table, int64_t rb,
                   unsigned char* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kGThreads / 32];
    const int lane = lane_id(), wid = warp_id();
    unsigned char* stage = smem + (int64_t)wid * kSpanChunk * rb;
    const unsigned bar = smem_u32(&bars[wid]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t n = *count_dev;
    const int cpr = (int)(rb >> 4);
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lt = (1u << lane) - 1u;
    unsigned phase = 0;
    for (int64_t j0 = w * kSpanChunk; j0 < n; j0 += nw * kSpanChunk) {
        const int m = (int)((n - j0) < kSpanChunk ? (n - j0) : kSpanChunk);
        int32_t p = -1, v = 0;
        if (lane < m) {
            p = __ldg(pos + j0 + lane);
            v = __ldg(ids + p);
        }
        const int32_t pv = __shfl_up_sync(0xffffffffu, v, 1);
        const bool inrow = lane < m;
        const bool start = inrow && (lane == 0 || pv + 1 != v);
        const unsigned sm = __ballot_sync(0xffffffffu, start);
        // span length of a start lane: distance to the next start (or m)
        const unsigned after = sm & ~((lt << 1) | 1u);
        const int next = after ? __ffs(after) - 1 : m;
        const int len = start ? next - lane : 0;
        const bool bulk = len >= 2;
        const unsigned bm = __ballot_sync(0xffffffffu, bulk);
        // wait until the previous chunk's bulk stores (each lane's own group) have read the stage
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        int tx = bulk ? len * (int)rb : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
        if (bm) {
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(tx) : "memory");
            __syncwarp();
            if (bulk)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                    :: "r"(smem_u32(stage + (int64_t)lane * rb)), "l"(table + (int64_t)v * rb),
                       "r"((unsigned)(len * rb)), "r"(bar) : "memory");
        }
        // single rows: 16-B loads, 2 rows in flight
        unsigned singles = sm & ~bm;
        while (singles) {
            const int a = __ffs(singles) - 1;
            singles &= singles - 1;
            int b = -1;
            if (singles) {
                b = __ffs(singles) - 1;
                singles &= singles - 1;
            }
            const int32_t pa = __shfl_sync(0xffffffffu, p, a), va = __shfl_sync(0xffffffffu, v, a);
            const int32_t pb = __shfl_sync(0xffffffffu, p, b < 0 ? a : b), vb = __shfl_sync(0xffffffffu, v, b < 0 ? a : b);
            const unsigned char* sa = table + (int64_t)va * rb;
            const unsigned char* sb = table + (int64_t)vb * rb;
            for (int c = lane; c < cpr; c += 32) {
                const uint4 x = ld_nc_v4(sa + c * 16);
                uint4 y;
                if (b >= 0) y = ld_nc_v4(sb + c * 16);
                st_na_v4(out + (int64_t)pa * rb + c * 16, x);
                if (b >= 0) st_na_v4(out + (int64_t)pb * rb + c * 16, y);
            }
        }
        if (bm) {
            asm volatile("{\n.reg .pred P;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}"
                         :: "r"(bar), "r"(phase) : "memory");
            phase ^= 1u;
            if (bulk)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             :: "l"(out + (int64_t)p * rb), "r"(smem_u32(stage + (int64_t)lane * rb)),
                                "r"((unsigned)(len * rb)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(kGThreads)
gather_v1_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ src_row,
                 const int64_t* __restrict__ n_dev, const unsigned char* __restrict__ ring,
                 const unsigned char* __restrict__ table, int64_t rb, unsigned char* __restrict__ out, int mode) {
    const int64_t n = *n_dev;
    const int64_t cpr = rb >> 2;
    const int64_t total = n * cpr;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t row = c / cpr;
        int64_t part = c - row * cpr;
        const int64_t sr = src_row ? __ldg(src_row + row) : -1;
        if (mode != 0 && (mode == 1) != (sr >= 0)) continue;
        const unsigned char* s = row_src(row, ids, src_row, ring, table, rb) + part * 4;
        *reinterpret_cast<uint32_t*>(out + row * rb + part * 4) = *reinterpret_cast<const uint32_t*>(s);
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void synth_kernel(int64_t first, int64_t nrows, int32_t dim, uint64_t seed, float* __restrict__ out) {
    const int64_t total = nrows * dim;
    const uint64_t salt = seed * 0xD1B54A32D192ED03ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / dim;
        int64_t j = i - r * dim;
        uint64_t key = ((uint64_t)(first + r) << 20) | (uint64_t)j;
        uint64_t z = splitmix64(key + salt);
        out[i] = (float)((double)((z >> 40) & 0xFFFFFFull) * (1.0 / 16777216.0) - 0.5);
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

int bgl_gather_rows(const int32_t* ids, const int64_t* src_row, const int64_t* n_dev, int64_t max_n,
                    const void* ring_rows, const void* table, int64_t row_bytes, void* out, int32_t mode,
                    int32_t ctas, void* stream) {
    BGL_CHECK_ARG(mode >= 0 && mode <= 2, "gather mode must be 0 (all), 1 (hits) or 2 (misses)");
    BGL_CHECK_ARG(row_bytes > 0 && row_bytes % 4 == 0, "row_bytes must be a positive multiple of 4");
    BGL_CHECK_ARG(ids && n_dev && table && out, "bgl_gather_rows: null pointer");
    BGL_CHECK_ARG(src_row == nullptr || ring_rows != nullptr, "bgl_gather_rows: src_row without ring rows");
    if (max_n <= 0) return BGL_OK;
    cudaStream_t st = as_stream(stream);
    const bool v4 = (row_bytes % 16 == 0) && ((uintptr_t)table % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                    (ring_rows == nullptr || (uintptr_t)ring_rows % 16 == 0);
    if (v4) {
        unsigned grid = grid_for(ceil_div(max_n, kRows) * 32, kGThreads, 4);
        int threads = kGThreads;
        if (ctas > 0) {   // latency-bound host-link reads: ~150 warps saturate it (tools/gather_bench.cu)
            grid = (unsigned)ctas;
            threads = 256;
        }
        gather_v4_kernel<<<grid, threads, 0, st>>>(ids, src_row, n_dev, (const unsigned char*)ring_rows,
                                                     (const unsigned char*)table, row_bytes, (unsigned char*)out,
                                                     mode, nullptr, nullptr);
        return launch_status("gather_v4_kernel");
    }
    int64_t chunks = max_n * (row_bytes / 4);
    gather_v1_kernel<<<grid_for(chunks, kGThreads, 8), kGThreads, 0, st>>>(
        ids, src_row, n_dev, (const unsigned char*)ring_rows, (const unsigned char*)table, row_bytes,
        (unsigned char*)out, mode);
    return launch_status("gather_v1_kernel");
}

int bgl_gather_rows_push(const int32_t* ids, const int64_t* src_row, const int64_t* n_dev, int64_t max_n,
                         const void* ring_rows, const void* table, int64_t row_bytes, void* out, void* push_out,
                         const int32_t* push_pos, int32_t mode, int32_t ctas, void* stream) {
    BGL_CHECK_ARG(mode >= 0 && mode <= 2, "gather mode must be 0 (all), 1 (hits) or 2 (misses)");
    BGL_CHECK_ARG(ids && n_dev && table && push_out && push_pos, "bgl_gather_rows_push: null pointer");
    BGL_CHECK_ARG(src_row == nullptr || ring_rows != nullptr, "bgl_gather_rows_push: src_row without ring rows");
    BGL_CHECK_ARG(row_bytes % 16 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)out % 16 == 0 &&
                      (uintptr_t)push_out % 16 == 0,
                  "bgl_gather_rows_push: 16-byte aligned rows required");
    if (max_n <= 0) return BGL_OK;
    unsigned grid = grid_for(ceil_div(max_n, kRows) * 32, kGThreads, 4);
    int threads = kGThreads;
    if (ctas > 0) {
        grid = (unsigned)ctas;
        threads = 256;
    }
    gather_v4_kernel<<<grid, threads, 0, as_stream(stream)>>>(
        ids, src_row, n_dev, (const unsigned char*)ring_rows, (const unsigned char*)table, row_bytes,
        (unsigned char*)out, mode, (unsigned char*)push_out, push_pos);
    return launch_status("gather_v4_kernel(push)");
}

int bgl_gather_list(const int32_t* pos, const int64_t* count_dev, int64_t max_n, const int32_t* ids,
                    const void* table, int64_t row_bytes, void* out, void* push_out, const int32_t* push_pos,
                    int32_t rows_in_flight, int32_t ctas, void* stream) {
    BGL_CHECK_ARG(pos && count_dev && ids && table && (out || push_out), "bgl_gather_list: null pointer");
    BGL_CHECK_ARG((push_out == nullptr) == (push_pos == nullptr), "bgl_gather_list: push_out and push_pos go together");
    BGL_CHECK_ARG(row_bytes % 16 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)out % 16 == 0 &&
                      (uintptr_t)push_out % 16 == 0,
                  "bgl_gather_list: 16-byte aligned rows required");
    BGL_CHECK_ARG(rows_in_flight == 0 || rows_in_flight == 2 || rows_in_flight == 4 || rows_in_flight == 8,
                  "rows_in_flight must be 0 (default), 2, 4 or 8");
    if (max_n <= 0) return BGL_OK;
    const int R = rows_in_flight ? rows_in_flight : 4;
    unsigned grid = ctas > 0 ? (unsigned)ctas : grid_for(ceil_div(max_n, R) * 32, kGThreads, 4);
    cudaStream_t st = as_stream(stream);
    auto T = (const unsigned char*)table;
    auto O = (unsigned char*)out;
    auto P = (unsigned char*)push_out;
    if (R == 2) gather_list_kernel<2><<<grid, kGThreads, 0, st>>>(pos, count_dev, ids, T, row_bytes, O, P, push_pos);
    else if (R == 8) gather_list_kernel<8><<<grid, kGThreads, 0, st>>>(pos, count_dev, ids, T, row_bytes, O, P, push_pos);
    else gather_list_kernel<4><<<grid, kGThreads, 0, st>>>(pos, count_dev, ids, T, row_bytes, O, P, push_pos);
    return launch_status("gather_list_kernel");
}

int bgl_gather_spans(const int32_t* pos, const int64_t* count_dev, int64_t max_n, const int32_t* ids,
                     const void* table, int64_t row_bytes, void* out, int32_t ctas, void* stream) {
    BGL_CHECK_ARG(pos && count_dev && ids && table && out, "bgl_gather_spans: null pointer");
    BGL_CHECK_ARG(row_bytes % 16 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)out % 16 == 0,
                  "bgl_gather_spans: 16-byte aligned rows required");
    BGL_CHECK_ARG(row_bytes * kSpanChunk * (kGThreads / 32) <= 200 * 1024, "bgl_gather_spans: rows too wide");
    if (max_n <= 0) return BGL_OK;
    const size_t smem = (size_t)row_bytes * kSpanChunk * (kGThreads / 32);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        BGL_TRY(cuda_status(cudaFuncSetAttribute(gather_span_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem), "cudaFuncSetAttribute(gather_span)"));
        configured = smem;
    }
    unsigned grid = ctas > 0 ? (unsigned)ctas : grid_for(ceil_div(max_n, kSpanChunk) * 32, kGThreads, 2);
    gather_span_kernel<<<grid, kGThreads, smem, as_stream(stream)>>>(pos, count_dev, ids, (const unsigned char*)table,
                                                                      row_bytes, (unsigned char*)out);
    return launch_status("gather_span_kernel");
}

int bgl_synthetic_features(int64_t first_node, int64_t num_nodes, int32_t dim, uint64_t seed, float* out,
                           void* stream) {
    BGL_CHECK_ARG(dim >= 1 && dim < (1 << 20), "dim must be in [1, 2^20)");
    BGL_CHECK_ARG(first_node >= 0 && num_nodes >= 0, "negative range");
    if (num_nodes == 0) return BGL_OK;
    synth_kernel<<<grid_for(num_nodes * dim, 256, 16), 256, 0, as_stream(stream)>>>(first_node, num_nodes, dim, seed,
                                                                                    out);
    return launch_status("synth_kernel");
}

}  // extern "C"
