// Single-pass decoupled look-back prefix scan (tiles claimed in launch order
// through an atomic ticket so every predecessor is already resident).
#pragma once

#include "common.cuh"

namespace bgl {

// status word = flag (2 bits) << 62 | value (62 bits)
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

struct ScanState {
    uint64_t* status;   // [N][max_tiles]
    int64_t max_tiles;
    unsigned* ticket;   // 1 counter
};

// Bytes of scan state for N values over up to max_tiles tiles (ticket included).
inline size_t scan_state_bytes(int N, int64_t max_tiles) {
    return (size_t)N * (size_t)max_tiles * sizeof(uint64_t) + 256;
}

inline ScanState make_scan_state(void* base, int N, int64_t max_tiles) {
    ScanState s;
    s.status = reinterpret_cast<uint64_t*>(base);
    s.max_tiles = max_tiles;
    s.ticket = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(base) + (size_t)N * max_tiles * 8);
    return s;
}

inline int reset_scan_state(void* base, int N, int64_t max_tiles, cudaStream_t st) {
    return cuda_status(cudaMemsetAsync(base, 0, scan_state_bytes(N, max_tiles), st), "scan state reset");
}

__device__ __forceinline__ int64_t claim_tile(const ScanState& s, int64_t* smem_slot) {
    if (threadIdx.x == 0) *smem_slot = (int64_t)atomicAdd(s.ticket, 1u);
    __syncthreads();
    int64_t t = *smem_slot;
    __syncthreads();
    return t;
}

// All threads call with the tile aggregates agg[0..N); returns exclusive
// prefixes in prefix[0..N) (shared memory, visible to all threads on return).
template <int N>
__device__ __forceinline__ void lookback(const ScanState& s, int64_t tile, const int64_t* agg,
                                         int64_t* prefix /* smem[N] */) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < N; ++v) {
            uint64_t w = (tile == 0 ? kFlagInc : kFlagAgg) | ((uint64_t)agg[v] & kValMask);
            atomicExch((unsigned long long*)&s.status[v * s.max_tiles + tile], (unsigned long long)w);
            if (tile == 0) prefix[v] = 0;
        }
    }
    if (tile > 0 && warp_id() == 0) {
        const int lane = lane_id();
#pragma unroll
        for (int v = 0; v < N; ++v) {
            const uint64_t* st = s.status + v * s.max_tiles;
            int64_t acc = 0;
            int64_t j = tile - 1;
            while (true) {
                int64_t idx = j - lane;
                uint64_t w = kFlagInc;   // before tile 0: inclusive zero
                if (idx >= 0) {
                    do { w = ld_status(st + idx); } while ((w >> 62) == 0);
                }
                unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                int stop = inc ? __ffs(inc) - 1 : 31;
                int64_t val = lane <= stop ? (int64_t)(w & kValMask) : 0;
                acc += warp_sum_i64(val);
                if (inc) break;
                j -= 32;
            }
            if (lane == 0) {
                prefix[v] = acc;
                uint64_t w = kFlagInc | ((uint64_t)(acc + agg[v]) & kValMask);
                atomicExch((unsigned long long*)&s.status[v * s.max_tiles + tile], (unsigned long long)w);
            }
        }
    }
    __syncthreads();
}

}  // namespace bgl
