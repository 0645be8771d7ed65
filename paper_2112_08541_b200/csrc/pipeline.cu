// Per-step staging for the CUDA-graph-captured mini-batch pipeline: the
// batch index lives on the device, so one captured graph replays every step
// of an epoch without host-side arguments.
#include <algorithm>

#include "common.cuh"
#include "pcg64.cuh"

namespace bgl {

__global__ void stage_batch_kernel(const int32_t* __restrict__ order, int64_t total, int64_t b, int64_t nb,
                                   const uint64_t* __restrict__ tables, int64_t* __restrict__ batch_counter,
                                   int32_t* __restrict__ seeds_out, int64_t* __restrict__ seed_count,
                                   uint64_t* __restrict__ table_out, int64_t* __restrict__ batch_index_out,
                                   const int64_t* __restrict__ fed_count, int64_t stride, int64_t offset) {
    const int64_t i = (*batch_counter * stride + offset) % nb;
    // host-fed mode: `order` holds just this batch (fed_count entries)
    const int64_t lo = fed_count ? 0 : i * b;
    const int64_t hi = fed_count ? *fed_count : (lo + b < total ? lo + b : total);
    for (int64_t k = threadIdx.x; k < hi - lo; k += blockDim.x) seeds_out[k] = order[lo + k];
    for (int k = threadIdx.x; k < kPcgTableRows * 4; k += blockDim.x) table_out[k] = tables[i * kPcgTableRows * 4 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
        *seed_count = hi - lo;
        if (batch_index_out) *batch_index_out = i;
        *batch_counter += 1;
    }
}

// Result hand-off to the host without a host sync: the distinct IDs of the
// batch (count known only on the device) and an 8-word counter block are
// stored straight into mapped pinned host memory (posted PCIe writes).
__global__ void d2h_result_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                  const int64_t* __restrict__ counters, int32_t* __restrict__ host_ids,
                                  int64_t* __restrict__ host_meta) {
    const int64_t n = *n_dev;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nv = n >> 2;
    const int4* src4 = reinterpret_cast<const int4*>(ids);
    int4* dst4 = reinterpret_cast<int4*>(host_ids);
    for (int64_t i = t0; i < nv; i += stride) dst4[i] = src4[i];
    for (int64_t i = (nv << 2) + t0; i < n; i += stride) host_ids[i] = ids[i];
    if (t0 == 0) {
        host_meta[0] = n;
        for (int k = 0; k < 8; ++k) host_meta[1 + k] = counters ? counters[k] : 0;
    }
}

}  // namespace bgl

using namespace bgl;

namespace bgl {
// off[batch] is only read here; one thread writes off[batch + 1]
__global__ void trace_append_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ n_dev,
                                    int32_t* __restrict__ dst, int64_t* __restrict__ off, int64_t batch) {
    const int64_t n = *n_dev;
    const int64_t o = off[batch];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[o + i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) off[batch + 1] = o + n;
}
}  // namespace bgl

extern "C" {

int bgl_stage_batch(const int32_t* order, int64_t total, int64_t batch_size, int64_t num_batches,
                    const uint64_t* tables, int64_t* batch_counter, int32_t* seeds_out, int64_t* seed_count_out,
                    uint64_t* table_out, int64_t* batch_index_out, const int64_t* fed_count_dev,
                    int64_t batch_stride, int64_t batch_offset, void* stream) {
    BGL_CHECK_ARG(order && tables && batch_counter && seeds_out && seed_count_out && table_out,
                  "bgl_stage_batch: null pointer");
    BGL_CHECK_ARG(batch_size >= 1 && num_batches >= 1 && total >= 1, "bgl_stage_batch: empty schedule");
    BGL_CHECK_ARG(batch_stride >= 1 && batch_offset >= 0, "bgl_stage_batch: bad stride/offset");
    stage_batch_kernel<<<1, 1024, 0, as_stream(stream)>>>(order, total, batch_size, num_batches, tables,
                                                          batch_counter, seeds_out, seed_count_out, table_out,
                                                          batch_index_out, fed_count_dev, batch_stride,
                                                          batch_offset);
    return launch_status("stage_batch_kernel");
}

int bgl_trace_append(const int32_t* src, const int64_t* n_dev, int64_t max_n, int32_t* dst, int64_t* off,
                     int64_t batch, void* stream) {
    BGL_CHECK_ARG(src && n_dev && dst && off && batch >= 0, "bgl_trace_append: bad argument");
    if (max_n <= 0) max_n = 1;
    trace_append_kernel<<<grid_for(max_n, 256, 4), 256, 0, as_stream(stream)>>>(src, n_dev, dst, off, batch);
    return launch_status("trace_append_kernel");
}

int bgl_d2h_result(const int32_t* ids, const int64_t* n_dev, int64_t max_n, const int64_t* counters,
                   int32_t* host_ids, int64_t* host_meta, void* stream) {
    BGL_CHECK_ARG(ids && n_dev && host_ids && host_meta, "bgl_d2h_result: null pointer");
    BGL_CHECK_ARG(((uintptr_t)ids & 15) == 0 && ((uintptr_t)host_ids & 15) == 0, "buffers must be 16-byte aligned");
    d2h_result_kernel<<<grid_for(std::max<int64_t>(max_n / 4, 1), 256, 2), 256, 0, as_stream(stream)>>>(
        ids, n_dev, counters, host_ids, host_meta);
    return launch_status("d2h_result_kernel");
}

}  // extern "C"
