// Per-step staging for the CUDA-graph-captured mini-batch pipeline: the
// batch index lives on the device, so one captured graph replays every step
// of an epoch without host-side arguments.
#include "common.cuh"

namespace bgl {

__global__ void stage_batch_kernel(const int32_t* __restrict__ order, int64_t total, int64_t b, int64_t nb,
                                   const uint64_t* __restrict__ tables, int64_t* __restrict__ batch_counter,
                                   int32_t* __restrict__ seeds_out, int64_t* __restrict__ seed_count,
                                   uint64_t* __restrict__ table_out, int64_t* __restrict__ batch_index_out,
                                   const int64_t* __restrict__ fed_count) {
    const int64_t i = *batch_counter % nb;
    // host-fed mode: `order` holds just this batch (fed_count entries)
    const int64_t lo = fed_count ? 0 : i * b;
    const int64_t hi = fed_count ? *fed_count : (lo + b < total ? lo + b : total);
    for (int64_t k = threadIdx.x; k < hi - lo; k += blockDim.x) seeds_out[k] = order[lo + k];
    for (int k = threadIdx.x; k < 65 * 4; k += blockDim.x) table_out[k] = tables[i * 65 * 4 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
        *seed_count = hi - lo;
        if (batch_index_out) *batch_index_out = i;
        *batch_counter += 1;
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

int bgl_stage_batch(const int32_t* order, int64_t total, int64_t batch_size, int64_t num_batches,
                    const uint64_t* tables, int64_t* batch_counter, int32_t* seeds_out, int64_t* seed_count_out,
                    uint64_t* table_out, int64_t* batch_index_out, const int64_t* fed_count_dev,
                    void* stream) {
    BGL_CHECK_ARG(order && tables && batch_counter && seeds_out && seed_count_out && table_out,
                  "bgl_stage_batch: null pointer");
    BGL_CHECK_ARG(batch_size >= 1 && num_batches >= 1 && total >= 1, "bgl_stage_batch: empty schedule");
    stage_batch_kernel<<<1, 1024, 0, as_stream(stream)>>>(order, total, batch_size, num_batches, tables,
                                                          batch_counter, seeds_out, seed_count_out, table_out,
                                                          batch_index_out, fed_count_dev);
    return launch_status("stage_batch_kernel");
}

}  // extern "C"
