// Static-degree cache warm-up on the device (gnnio.cachesim.warm_static,
// cachesim.py:206-224): per shard h (nodes v % d == h) the `capacity`
// highest-degree nodes, ties to the lower ID; then the host level takes the
// highest-degree nodes among the rest. Sort-free: a per-shard degree
// histogram gives each shard's threshold degree t_h and how many nodes of
// degree exactly t_h it still needs (host arithmetic on the histogram); the
// ties are ranked by ID with an ascending stable compaction.
#include <algorithm>

#include "common.cuh"
#include "scan.cuh"

namespace bgl {

constexpr int kSThreads = 256;
constexpr int kSItems = 8;
constexpr int kSTile = kSThreads * kSItems;

__device__ __forceinline__ int64_t degree_of(const int64_t* indptr, int64_t v) { return indptr[v + 1] - indptr[v]; }

// hist[h][min(deg, maxdeg)] += 1 for every node not excluded
__global__ void degree_hist_kernel(const int64_t* __restrict__ indptr, int64_t n, int32_t d, int64_t maxdeg,
                                   const uint8_t* __restrict__ exclude, unsigned long long* __restrict__ hist) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (exclude && exclude[v]) continue;
        int64_t deg = degree_of(indptr, v);
        if (deg > maxdeg) deg = maxdeg;
        atomicAdd(hist + (v % d) * (maxdeg + 1) + deg, 1ull);
    }
}

// flags[v] = mode 0: deg == t[h] (tie candidates); mode 1: deg > t[h] or tie_sel[v]
__global__ void select_flags_kernel(const int64_t* __restrict__ indptr, int64_t n, int32_t d,
                                    const int64_t* __restrict__ thresh, const uint8_t* __restrict__ exclude,
                                    const uint8_t* __restrict__ tie_sel, int mode, uint8_t* __restrict__ flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        uint8_t f = 0;
        if (!(exclude && exclude[v])) {
            const int64_t deg = degree_of(indptr, v);
            const int64_t t = thresh[v % d];
            f = mode == 0 ? (deg == t) : (deg > t || (tie_sel && tie_sel[v]));
        }
        flags[v] = f;
    }
}

// stable compaction of the flagged node IDs (ascending), decoupled look-back
__global__ void __launch_bounds__(kSThreads)
compact_flags_kernel(const uint8_t* __restrict__ flags, int64_t n, ScanState ss, int32_t* __restrict__ out,
                     int64_t* __restrict__ count) {
    __shared__ int64_t s_red[kSThreads / 32 + 1];
    __shared__ int64_t s_agg[1], s_pre[1], s_slot;
    const int64_t ntiles = n > 0 ? ceil_div(n, kSTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int64_t v0 = tile * kSTile + (int64_t)threadIdx.x * kSItems;
    int64_t c = 0;
    for (int j = 0; j < kSItems; ++j) c += (v0 + j < n && flags[v0 + j]);
    int64_t tot;
    int64_t ex = block_excl_scan(c, s_red, &tot);
    if (threadIdx.x == 0) s_agg[0] = tot;
    __syncthreads();
    lookback<1>(ss, tile, s_agg, s_pre);
    int64_t p = s_pre[0] + ex;
    for (int j = 0; j < kSItems; ++j)
        if (v0 + j < n && flags[v0 + j]) out[p++] = (int32_t)(v0 + j);
    if (tile == ntiles - 1 && threadIdx.x == 0) *count = s_pre[0] + tot;
}

}  // namespace bgl

using namespace bgl;

extern "C" {

int bgl_degree_histogram(const int64_t* indptr, int64_t num_nodes, int32_t num_shards, int64_t max_degree,
                         const uint8_t* exclude, int64_t* hist, void* stream) {
    BGL_CHECK_ARG(indptr && hist && num_nodes >= 0 && num_shards >= 1 && max_degree >= 0,
                  "bgl_degree_histogram: bad arguments");
    cudaStream_t st = as_stream(stream);
    BGL_TRY(cuda_status(cudaMemsetAsync(hist, 0, (size_t)num_shards * (max_degree + 1) * 8, st), "hist memset"));
    if (num_nodes == 0) return BGL_OK;
    degree_hist_kernel<<<grid_for(num_nodes, 256), 256, 0, st>>>(indptr, num_nodes, num_shards, max_degree, exclude,
                                                                 (unsigned long long*)hist);
    return launch_status("degree_hist_kernel");
}

int bgl_select_flags(const int64_t* indptr, int64_t num_nodes, int32_t num_shards, const int64_t* thresh,
                     const uint8_t* exclude, const uint8_t* tie_sel, int32_t mode, uint8_t* flags, void* stream) {
    BGL_CHECK_ARG(indptr && thresh && flags && (mode == 0 || mode == 1), "bgl_select_flags: bad arguments");
    if (num_nodes == 0) return BGL_OK;
    select_flags_kernel<<<grid_for(num_nodes, 256), 256, 0, as_stream(stream)>>>(indptr, num_nodes, num_shards,
                                                                                 thresh, exclude, tie_sel, mode, flags);
    return launch_status("select_flags_kernel");
}

size_t bgl_compact_workspace(int64_t num_nodes) {
    return scan_state_bytes(1, std::max<int64_t>(1, ceil_div(num_nodes, kSTile)));
}

int bgl_compact_flags(const uint8_t* flags, int64_t num_nodes, int32_t* out_ids, int64_t* count_dev, void* workspace,
                      void* stream) {
    BGL_CHECK_ARG(flags && out_ids && count_dev && workspace, "bgl_compact_flags: null pointer");
    cudaStream_t st = as_stream(stream);
    const int64_t tiles = std::max<int64_t>(1, ceil_div(num_nodes, kSTile));
    BGL_TRY(reset_scan_state(workspace, 1, tiles, st));
    compact_flags_kernel<<<(unsigned)tiles, kSThreads, 0, st>>>(flags, num_nodes, make_scan_state(workspace, 1, tiles),
                                                                 out_ids, count_dev);
    return launch_status("compact_flags_kernel");
}

}  // extern "C"
