// Partition accounting of simulate_epoch (gnnio/sampler.py:139-153): seed
// load, per-hop request load and local/remote lookup counts, and the
// origin propagation through parent_idx.
#include "common.cuh"

namespace bgl {

constexpr int kAThreads = 256;
constexpr int kMaxParts = 1024;

__global__ void __launch_bounds__(kAThreads)
account_kernel(const int32_t* __restrict__ parents, const int64_t* __restrict__ n_dev,
               const int32_t* __restrict__ origins, const int32_t* __restrict__ part_of, int32_t k,
               int64_t* __restrict__ load, int64_t* __restrict__ local_remote) {
    __shared__ int64_t s_load[kMaxParts];
    for (int i = threadIdx.x; i < k; i += blockDim.x) s_load[i] = 0;
    __syncthreads();
    const int64_t n = *n_dev;
    int64_t loc = 0, cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t pp = part_of[parents[i]];
        atomicAdd((unsigned long long*)&s_load[pp], 1ull);
        if (origins) {
            loc += (pp == origins[i]);
            cnt += 1;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        if (s_load[i]) atomicAdd((unsigned long long*)&load[i], (unsigned long long)s_load[i]);
    if (origins) {
        loc = warp_sum_i64(loc);
        cnt = warp_sum_i64(cnt);
        if (lane_id() == 0 && cnt) {
            atomicAdd((unsigned long long*)&local_remote[0], (unsigned long long)loc);
            atomicAdd((unsigned long long*)&local_remote[1], (unsigned long long)(cnt - loc));
        }
    }
}

__global__ void take_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ idx,
                            const int64_t* __restrict__ n_dev, int32_t* __restrict__ out) {
    const int64_t n = *n_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

}  // namespace bgl

using namespace bgl;

extern "C" {

int bgl_comm_account(const int32_t* parents, const int64_t* num_dev, int64_t max_n, const int32_t* origins,
                     const int32_t* part_of, int32_t k, int64_t* load, int64_t* local_remote, void* stream) {
    BGL_CHECK_ARG(k >= 1 && k <= kMaxParts, "number of partitions must be in [1, 1024]");
    BGL_CHECK_ARG(parents && num_dev && part_of && load, "bgl_comm_account: null pointer");
    BGL_CHECK_ARG(origins == nullptr || local_remote != nullptr, "bgl_comm_account: local_remote required");
    if (max_n <= 0) return BGL_OK;
    account_kernel<<<grid_for(max_n, kAThreads, 2), kAThreads, 0, as_stream(stream)>>>(parents, num_dev, origins,
                                                                                        part_of, k, load, local_remote);
    return launch_status("account_kernel");
}

int bgl_take_i32(const int32_t* src, const int32_t* idx, const int64_t* num_dev, int64_t max_n, int32_t* out,
                 void* stream) {
    BGL_CHECK_ARG(src && idx && num_dev && out, "bgl_take_i32: null pointer");
    if (max_n <= 0) return BGL_OK;
    take_kernel<<<grid_for(max_n, 256), 256, 0, as_stream(stream)>>>(src, idx, num_dev, out);
    return launch_status("take_kernel");
}

}  // extern "C"
