// Multi-GPU exchange helpers for the node-ID-sharded cache (home of node v is
// GPU v % H, gnnio/cachesim.py:319-320):
//   partition  stable split of a sorted batch by home -> H ascending buckets
//              (the insert order each home needs, cachesim.py:341-342) and the
//              position of every bucketed ID in the batch;
//   scatter    rows returned by the homes back into batch order;
//   compact    positions of a batch whose outcome code is >= a threshold
//              (the worker's own device-missed rows, fetched by the worker).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "scan.cuh"

namespace bgl {

constexpr int kXThreads = 256;
constexpr int kXRounds = 4;
constexpr int kXTile = kXThreads * kXRounds;
constexpr int kXMaxHomes = 64;

__global__ void __launch_bounds__(kXThreads)
home_count_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int32_t H,
                  int64_t* __restrict__ tile_counts) {
    __shared__ int32_t s_cnt[kXMaxHomes];
    const int64_t n = *n_dev;
    for (int h = threadIdx.x; h < H; h += blockDim.x) s_cnt[h] = 0;
    __syncthreads();
    for (int r = 0; r < kXRounds; ++r) {
        const int64_t e = blockIdx.x * (int64_t)kXTile + r * kXThreads + threadIdx.x;
        const int h = e < n ? ids[e] % H : -1;
        for (int y = 0; y < H; ++y) {
            const unsigned m = __ballot_sync(0xffffffffu, h == y);
            if (lane_id() == 0 && m) atomicAdd(&s_cnt[y], __popc(m));
        }
    }
    __syncthreads();
    for (int h = threadIdx.x; h < H; h += blockDim.x) tile_counts[blockIdx.x * (int64_t)H + h] = s_cnt[h];
}

// one block: per-home exclusive offsets over (home, tile) in home-major order
__global__ void home_scan_kernel(int64_t* __restrict__ tile_counts, int64_t ntiles, int32_t H,
                                 int64_t* __restrict__ counts_out) {
    __shared__ int64_t s_red[kXThreads / 32 + 1];
    int64_t carry = 0;
    for (int h = 0; h < H; ++h) {
        int64_t home_total = 0;
        for (int64_t b = 0; b < ntiles; b += blockDim.x) {
            const int64_t t = b + threadIdx.x;
            const int64_t v = t < ntiles ? tile_counts[t * H + h] : 0;
            int64_t tot;
            const int64_t ex = block_excl_scan(v, s_red, &tot);
            if (t < ntiles) tile_counts[t * H + h] = carry + home_total + ex;
            home_total += tot;
        }
        if (threadIdx.x == 0) counts_out[h] = home_total;
        carry += home_total;
    }
}

__global__ void __launch_bounds__(kXThreads)
home_scatter_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int32_t H,
                    const int64_t* __restrict__ tile_off, int32_t* __restrict__ out_ids,
                    int32_t* __restrict__ out_pos) {
    constexpr int NW = kXThreads / 32;
    __shared__ int32_t s_w[NW][kXMaxHomes];
    __shared__ int64_t s_run[kXMaxHomes];
    const int64_t n = *n_dev;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    for (int h = threadIdx.x; h < H; h += blockDim.x) s_run[h] = tile_off[blockIdx.x * (int64_t)H + h];
    __syncthreads();
    for (int r = 0; r < kXRounds; ++r) {
        const int64_t e = blockIdx.x * (int64_t)kXTile + r * kXThreads + threadIdx.x;
        const int32_t v = e < n ? ids[e] : 0;
        const int h = e < n ? v % H : -1;
        int rank = 0;
        for (int y = 0; y < H; ++y) {
            const unsigned m = __ballot_sync(0xffffffffu, h == y);
            if (h == y) rank = __popc(m & lt);
            if (lane == 0) s_w[wid][y] = __popc(m);
        }
        __syncthreads();
        if (h >= 0) {
            int64_t p = s_run[h] + rank;
            for (int w = 0; w < wid; ++w) p += s_w[w][h];
            out_ids[p] = v;
            out_pos[p] = (int32_t)e;
        }
        __syncthreads();
        for (int y = threadIdx.x; y < H; y += blockDim.x) {
            int64_t add = 0;
            for (int w = 0; w < NW; ++w) add += s_w[w][y];
            s_run[y] += add;
        }
        __syncthreads();
    }
}

// home_scatter with the exchange fused in: every bucketed ID (and its batch
// position) is stored straight into its HOME GPU's receive area over peer
// memory (CUDA IPC mappings, NVLink), at its offset inside the bucket; the
// first block also stores the bucket sizes. Ends with a system-scope fence so
// the stores are visible to the homes once the kernel has completed (the
// caller then crosses a barrier).
__global__ void __launch_bounds__(kXThreads)
home_push_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int32_t H,
                 const int64_t* __restrict__ tile_off, const int64_t* __restrict__ counts,
                 int32_t* const* __restrict__ peer_ids, int32_t* const* __restrict__ peer_pos,
                 int64_t* const* __restrict__ peer_cnt) {
    constexpr int NW = kXThreads / 32;
    __shared__ int32_t s_w[NW][kXMaxHomes];
    __shared__ int64_t s_run[kXMaxHomes];
    __shared__ int64_t s_start[kXMaxHomes];
    const int64_t n = *n_dev;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x == 0) {
        int64_t c = 0;
        for (int h = 0; h < H; ++h) {
            s_start[h] = c;
            c += counts[h];
        }
    }
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        s_run[h] = tile_off[blockIdx.x * (int64_t)H + h];
        if (blockIdx.x == 0) *peer_cnt[h] = counts[h];
    }
    __syncthreads();
    for (int r = 0; r < kXRounds; ++r) {
        const int64_t e = blockIdx.x * (int64_t)kXTile + r * kXThreads + threadIdx.x;
        const int32_t v = e < n ? ids[e] : 0;
        const int h = e < n ? v % H : -1;
        int rank = 0;
        for (int y = 0; y < H; ++y) {
            const unsigned m = __ballot_sync(0xffffffffu, h == y);
            if (h == y) rank = __popc(m & lt);
            if (lane == 0) s_w[wid][y] = __popc(m);
        }
        __syncthreads();
        if (h >= 0) {
            int64_t p = s_run[h] + rank;
            for (int w = 0; w < wid; ++w) p += s_w[w][h];
            p -= s_start[h];
            peer_ids[h][p] = v;
            peer_pos[h][p] = (int32_t)e;
        }
        __syncthreads();
        for (int y = threadIdx.x; y < H; y += blockDim.x) {
            int64_t add = 0;
            for (int w = 0; w < NW; ++w) add += s_w[w][y];
            s_run[y] += add;
        }
        __syncthreads();
    }
    __threadfence_system();
}

__global__ void scatter_rows_kernel(const int32_t* __restrict__ pos, const int64_t* __restrict__ n_dev,
                                    const unsigned char* __restrict__ rows, int64_t rb,
                                    unsigned char* __restrict__ out) {
    const int64_t n = *n_dev;
    const int lane = lane_id();
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
        const unsigned char* s = rows + i * rb;
        unsigned char* d = out + (int64_t)pos[i] * rb;
        if ((rb & 15) == 0) {
            for (int64_t b = (int64_t)lane * 16; b < rb; b += 32 * 16)
                *reinterpret_cast<uint4*>(d + b) = *reinterpret_cast<const uint4*>(s + b);
        } else if ((rb & 3) != 0) {
            for (int64_t b = lane; b < rb; b += 32) d[b] = s[b];
        } else {
            for (int64_t b = (int64_t)lane * 4; b < rb; b += 32 * 4)
                *reinterpret_cast<uint32_t*>(d + b) = *reinterpret_cast<const uint32_t*>(s + b);
        }
    }
    __threadfence_system();   // `out` may be a peer GPU's buffer (codes pushed to the worker)
}


// Ordered stream compaction of code >= min_code (4 consecutive codes per
// thread, block scan + decoupled look-back over tiles of kXTile).
__global__ void __launch_bounds__(kXThreads)
compact_codes_kernel(const uint8_t* __restrict__ codes, const int64_t* __restrict__ n_dev, int32_t min_code,
                     ScanState ss, int32_t* __restrict__ pos_out, int64_t* __restrict__ count_out) {
    __shared__ int64_t s_red[kXThreads / 32 + 1];
    __shared__ int64_t s_agg[1], s_pre[1], s_tile;
    const int64_t n = *n_dev;
    const int64_t ntiles = n > 0 ? ceil_div(n, kXTile) : 1;
    const int64_t tile = claim_tile(ss, &s_tile);
    if (tile >= ntiles) return;
    const int64_t base = tile * kXTile + (int64_t)threadIdx.x * kXRounds;
    bool f[kXRounds];
    int64_t cnt = 0;
#pragma unroll
    for (int u = 0; u < kXRounds; ++u) {
        f[u] = base + u < n && (int32_t)codes[base + u] >= min_code;
        cnt += f[u];
    }
    int64_t total;
    const int64_t ex = block_excl_scan(cnt, s_red, &total);
    if (threadIdx.x == 0) s_agg[0] = total;
    __syncthreads();
    lookback<1>(ss, tile, s_agg, s_pre);
    int64_t r = s_pre[0] + ex;
#pragma unroll
    for (int u = 0; u < kXRounds; ++u)
        if (f[u]) pos_out[r++] = (int32_t)(base + u);
    if (tile == ntiles - 1 && threadIdx.x == 0) *count_out = s_pre[0] + total;
}

// Host-level hand-off (the reference's one shared host level, cachesim.py:
// 202, 330-344, owned by one GPU): the worker's device-missed IDs (ascending)
// and their batch positions stored into the owner's receive area (peer memory).
__global__ void push_pairs_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ pos,
                                  const int64_t* __restrict__ n_dev, int32_t* __restrict__ dst_ids,
                                  int32_t* __restrict__ dst_pos, int64_t* __restrict__ dst_cnt) {
    const int64_t n = *n_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = pos[i];
        dst_ids[i] = ids[p];
        dst_pos[i] = p;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *dst_cnt = n;
    __threadfence_system();   // peer stores visible system-wide before the caller's barrier
}

// Owner side: the host level's lookup codes of a worker's device-missed IDs
// (a single-level FIFO whose hits are the host hits) become H / M at their
// batch positions in the worker's outcome codes (peer stores).
__global__ void host_level_codes_kernel(const uint8_t* __restrict__ hl_codes, const int32_t* __restrict__ pos,
                                        const int64_t* __restrict__ n_dev, uint8_t* __restrict__ dst_codes) {
    const int64_t n = *n_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst_codes[pos[i]] = hl_codes[i] == 0 ? (uint8_t)2 : (uint8_t)3;
    __threadfence_system();
}

// Fold the host level's counters into the cache counters: its hits turn
// device misses (counted M by the homes) into H; its inserts / evictions are
// the host level's (CacheSimReport.batch_host_hits / _misses / _insertions /
// _evictions, cachesim.py:346-356).
__global__ void host_level_account_kernel(int64_t* __restrict__ hl_counters, int64_t* __restrict__ counters) {
    if (threadIdx.x != 0) return;
    counters[3] += hl_counters[1];
    counters[4] -= hl_counters[1];
    counters[5] += hl_counters[5];
    counters[6] += hl_counters[6];
    for (int k = 0; k < 8; ++k) hl_counters[k] = 0;
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_partition_workspace(int64_t max_n, int32_t num_homes) {
    return (size_t)std::max<int64_t>(1, ceil_div(max_n, kXTile)) * num_homes * 8 + 256;
}

int bgl_partition_by_home(const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t num_homes,
                          int32_t* out_ids, int32_t* out_pos, int64_t* counts_dev, void* workspace, void* stream) {
    BGL_CHECK_ARG(num_homes >= 1 && num_homes <= kXMaxHomes, "num_homes must be in [1, 64]");
    BGL_CHECK_ARG(ids && n_dev && out_ids && out_pos && counts_dev && workspace, "bgl_partition_by_home: null");
    cudaStream_t st = as_stream(stream);
    const int64_t ntiles = std::max<int64_t>(1, ceil_div(max_n, kXTile));
    int64_t* tc = reinterpret_cast<int64_t*>(workspace);
    home_count_kernel<<<(unsigned)ntiles, kXThreads, 0, st>>>(ids, n_dev, num_homes, tc);
    BGL_TRY(launch_status("home_count_kernel"));
    home_scan_kernel<<<1, kXThreads, 0, st>>>(tc, ntiles, num_homes, counts_dev);
    BGL_TRY(launch_status("home_scan_kernel"));
    home_scatter_kernel<<<(unsigned)ntiles, kXThreads, 0, st>>>(ids, n_dev, num_homes, tc, out_ids, out_pos);
    return launch_status("home_scatter_kernel");
}

int bgl_partition_push(const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t num_homes,
                       int32_t* const* peer_ids, int32_t* const* peer_pos, int64_t* const* peer_cnt,
                       int64_t* counts_dev, void* workspace, void* stream) {
    BGL_CHECK_ARG(num_homes >= 1 && num_homes <= kXMaxHomes, "num_homes must be in [1, 64]");
    BGL_CHECK_ARG(ids && n_dev && peer_ids && peer_pos && peer_cnt && counts_dev && workspace,
                  "bgl_partition_push: null pointer");
    cudaStream_t st = as_stream(stream);
    const int64_t ntiles = std::max<int64_t>(1, ceil_div(max_n, kXTile));
    int64_t* tc = reinterpret_cast<int64_t*>(workspace);
    home_count_kernel<<<(unsigned)ntiles, kXThreads, 0, st>>>(ids, n_dev, num_homes, tc);
    BGL_TRY(launch_status("home_count_kernel"));
    home_scan_kernel<<<1, kXThreads, 0, st>>>(tc, ntiles, num_homes, counts_dev);
    BGL_TRY(launch_status("home_scan_kernel"));
    home_push_kernel<<<(unsigned)ntiles, kXThreads, 0, st>>>(ids, n_dev, num_homes, tc, counts_dev, peer_ids,
                                                              peer_pos, peer_cnt);
    return launch_status("home_push_kernel");
}

size_t bgl_compact_codes_workspace(int64_t max_n) {
    return scan_state_bytes(1, std::max<int64_t>(1, ceil_div(std::max<int64_t>(max_n, 1), kXTile)));
}

int bgl_compact_codes(const uint8_t* codes, const int64_t* n_dev, int64_t max_n, int32_t min_code, int32_t* pos_out,
                      int64_t* count_out, void* workspace, void* stream) {
    BGL_CHECK_ARG(codes && n_dev && pos_out && count_out && workspace, "bgl_compact_codes: null pointer");
    BGL_CHECK_ARG(max_n >= 0, "bgl_compact_codes: max_n < 0");
    cudaStream_t st = as_stream(stream);
    const int64_t tiles = std::max<int64_t>(1, ceil_div(std::max<int64_t>(max_n, 1), kXTile));
    BGL_TRY(reset_scan_state(workspace, 1, tiles, st));
    compact_codes_kernel<<<(unsigned)tiles, kXThreads, 0, st>>>(codes, n_dev, min_code,
                                                                 make_scan_state(workspace, 1, tiles), pos_out,
                                                                 count_out);
    return launch_status("compact_codes_kernel");
}

int bgl_scatter_rows(const int32_t* pos, const int64_t* n_dev, int64_t max_n, const void* rows, int64_t row_bytes,
                     void* out, void* stream) {
    BGL_CHECK_ARG(pos && n_dev && rows && out, "bgl_scatter_rows: null pointer");
    BGL_CHECK_ARG(row_bytes > 0, "row_bytes must be positive");
    if (max_n <= 0) return BGL_OK;
    scatter_rows_kernel<<<grid_for(max_n * 32, 256, 8), 256, 0, as_stream(stream)>>>(
        pos, n_dev, (const unsigned char*)rows, row_bytes, (unsigned char*)out);
    return launch_status("scatter_rows_kernel");
}

int bgl_push_pairs(const int32_t* ids, const int32_t* pos, const int64_t* n_dev, int64_t max_n, int32_t* dst_ids,
                   int32_t* dst_pos, int64_t* dst_cnt, void* stream) {
    BGL_CHECK_ARG(ids && pos && n_dev && dst_ids && dst_pos && dst_cnt, "bgl_push_pairs: null pointer");
    push_pairs_kernel<<<grid_for(std::max<int64_t>(max_n, 1), 256, 4), 256, 0, as_stream(stream)>>>(
        ids, pos, n_dev, dst_ids, dst_pos, dst_cnt);
    return launch_status("push_pairs_kernel");
}

int bgl_host_level_codes(const uint8_t* hl_codes, const int32_t* pos, const int64_t* n_dev, int64_t max_n,
                         uint8_t* dst_codes, void* stream) {
    BGL_CHECK_ARG(hl_codes && pos && n_dev && dst_codes, "bgl_host_level_codes: null pointer");
    host_level_codes_kernel<<<grid_for(std::max<int64_t>(max_n, 1), 256, 4), 256, 0, as_stream(stream)>>>(
        hl_codes, pos, n_dev, dst_codes);
    return launch_status("host_level_codes_kernel");
}

int bgl_host_level_account(int64_t* hl_counters, int64_t* counters, void* stream) {
    BGL_CHECK_ARG(hl_counters && counters, "bgl_host_level_account: null pointer");
    host_level_account_kernel<<<1, 32, 0, as_stream(stream)>>>(hl_counters, counters);
    return launch_status("host_level_account_kernel");
}

int bgl_ipc_get_handle(void* dev_ptr, void* handle_out, int64_t* offset_out) {
    BGL_CHECK_ARG(dev_ptr && handle_out && offset_out, "bgl_ipc_get_handle: null pointer");
    // The handle names the whole allocation (a caching allocator hands out
    // sub-ranges): report the offset of dev_ptr inside it. Driver API via
    // dlsym so the library has no link-time dependency on libcuda.
    using range_fn = int (*)(unsigned long long*, size_t*, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
        void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
        if (h) fn = reinterpret_cast<range_fn>(dlsym(h, "cuMemGetAddressRange_v2"));
        BGL_CHECK_ARG(fn != nullptr, "bgl_ipc_get_handle: cuMemGetAddressRange unavailable");
    }
    unsigned long long base = 0;
    size_t size = 0;
    BGL_CHECK_ARG(fn(&base, &size, (unsigned long long)dev_ptr) == 0, "cuMemGetAddressRange failed");
    *offset_out = (int64_t)((unsigned long long)dev_ptr - base);
    return cuda_status(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out), dev_ptr),
                       "cudaIpcGetMemHandle");
}

int bgl_ipc_open_handle(const void* handle, void** dev_ptr_out) {
    BGL_CHECK_ARG(handle && dev_ptr_out, "bgl_ipc_open_handle: null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return cuda_status(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int bgl_ipc_close(void* dev_ptr) {
    return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

}  // extern "C"
