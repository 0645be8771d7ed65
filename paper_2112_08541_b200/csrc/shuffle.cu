// Shuffling error of a mini-batch schedule on the device
// (gnnio.ordering.shuffling_error, ordering.py:157-186): per batch, the total
// variation distance between the batch's label frequencies and the label
// frequencies of the whole schedule,
//     tv_i = 0.5 * sum_c | cnt_i[c] / len_i - cnt[c] / total |   (fp64)
// One pass builds the global histogram, one CTA per batch builds the batch
// histogram in shared memory and reduces the TV distance.
#include <algorithm>

#include "common.cuh"

namespace bgl {

constexpr int kTThreads = 256;

__global__ void label_hist_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ order,
                                  int64_t total, int32_t num_classes, unsigned long long* __restrict__ hist,
                                  int32_t* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = labels[order[i]];
        if (l < 0 || l >= num_classes) {
            atomicExch(bad, 1);
            continue;
        }
        atomicAdd(hist + l, 1ull);
    }
}

__global__ void __launch_bounds__(kTThreads)
batch_tv_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ order, int64_t total,
                const int64_t* __restrict__ batch_off, int32_t num_classes, const unsigned long long* __restrict__ hist,
                double* __restrict__ tv) {
    extern __shared__ unsigned int s_cnt[];
    __shared__ double s_red[kTThreads / 32];
    const int64_t batch = blockIdx.x;
    const int64_t lo = batch_off[batch];
    const int64_t hi = batch_off[batch + 1];
    for (int c = threadIdx.x; c < num_classes; c += blockDim.x) s_cnt[c] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const int32_t l = labels[order[i]];
        if (l >= 0 && l < num_classes) atomicAdd(&s_cnt[l], 1u);
    }
    __syncthreads();
    const double len = (double)(hi - lo > 0 ? hi - lo : 1), all = (double)total;
    double acc = 0.0;
    for (int c = threadIdx.x; c < num_classes; c += blockDim.x)
        acc += fabs((double)s_cnt[c] / len - (double)hist[c] / all);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane_id() == 0) s_red[warp_id()] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kTThreads / 32; ++w) s += s_red[w];
        tv[batch] = 0.5 * s;
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_shuffling_workspace(int32_t num_classes) { return (size_t)std::max(num_classes, 1) * 8 + 256; }

int bgl_shuffling_tv(const int32_t* labels, const int32_t* order, int64_t total, const int64_t* batch_off,
                     int64_t num_batches, int32_t num_classes, void* workspace, double* tv_out,
                     int32_t* bad_label_dev, void* stream) {
    BGL_CHECK_ARG(labels && order && batch_off && workspace && tv_out && bad_label_dev,
                  "bgl_shuffling_tv: null pointer");
    BGL_CHECK_ARG(num_batches >= 1 && total >= 1, "empty schedule");
    BGL_CHECK_ARG(num_classes >= 1 && num_classes <= 16384, "num_classes must be in [1, 16384]");
    cudaStream_t st = as_stream(stream);
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(workspace);
    BGL_TRY(cuda_status(cudaMemsetAsync(hist, 0, (size_t)num_classes * 8, st), "hist memset"));
    BGL_TRY(cuda_status(cudaMemsetAsync(bad_label_dev, 0, 4, st), "flag memset"));
    label_hist_kernel<<<grid_for(total, 256), 256, 0, st>>>(labels, order, total, num_classes, hist, bad_label_dev);
    BGL_TRY(launch_status("label_hist_kernel"));
    const int64_t nb = num_batches;
    const size_t smem = (size_t)num_classes * 4;
    if (smem > 48 * 1024)
        BGL_TRY(cuda_status(cudaFuncSetAttribute(batch_tv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem), "cudaFuncSetAttribute(batch_tv)"));
    batch_tv_kernel<<<(unsigned)nb, kTThreads, smem, st>>>(labels, order, total, batch_off, num_classes, hist,
                                                            tv_out);
    return launch_status("batch_tv_kernel");
}

}  // extern "C"
