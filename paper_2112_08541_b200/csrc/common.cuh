// Shared helpers for the bgl_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>
#include <string>

#include "../../include/bgl_b200.h"

namespace bgl {

constexpr int kNumSMs = 148;   // B200: 2 dies x 74 SMs

void set_error(const char* fmt, ...);

inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return BGL_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? BGL_ENOMEM : BGL_ECUDA;
}

inline int launch_status(const char* what) { return cuda_status(cudaGetLastError(), what); }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid for a grid-stride loop: enough CTAs to fill every SM `per_sm` times,
// never more than the work needs.
inline unsigned grid_for(int64_t items, int threads, int per_sm = 8) {
    int64_t need = ceil_div(items > 0 ? items : 1, threads);
    int64_t cap = (int64_t)kNumSMs * per_sm;
    return (unsigned)(need < cap ? need : cap);
}

#define BGL_CHECK_ARG(cond, ...)              \
    do {                                      \
        if (!(cond)) {                        \
            ::bgl::set_error(__VA_ARGS__);    \
            return BGL_EINVAL;                \
        }                                     \
    } while (0)

#define BGL_TRY(expr)                         \
    do {                                      \
        int _st = (expr);                     \
        if (_st != BGL_OK) return _st;        \
    } while (0)

// ---------------------------------------------------------------- device utils
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T ld_volatile(const T* p) { return *(const volatile T*)p; }

// Poll of a look-back status word (flag and value packed in one 64-bit word,
// published by device-scope atomics): a relaxed load at GPU scope. A volatile
// load compiles to LDG.E.STRONG.SYS (system scope) on sm_100a, which costs
// more than an L2 round trip on every window of a look-back chain.
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Inclusive warp scan (Kogge-Stone).
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, writes the block total to *total. `smem` needs blockDim/32 slots.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T* total) {
    const int lane = lane_id(), wid = warp_id(), nw = blockDim.x >> 5;
    T incl = warp_incl_scan(v);
    if (lane == 31) smem[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        T w = lane < nw ? smem[lane] : T(0);
        T wi = warp_incl_scan(w);
        if (lane < nw) smem[lane] = wi - w;
        if (lane == nw - 1) smem[nw] = wi;
    }
    __syncthreads();
    T res = smem[wid] + incl - v;
    *total = smem[nw];
    __syncthreads();
    return res;
}

}  // namespace bgl
