// K3/K4: BGL's dynamic FIFO feature cache, bit-exact with gnnio.cachesim's
// FIFO policy (FifoLevel cachesim.py:81-107; simulate cachesim.py:275-363).
//
// State (all device-resident):
//   rings   int32 [d][C]   node in each slot, -1 empty   (FifoLevel.slots)
//   hring   int32 [Ch]     shared host level
//   slot_of int32 [n]      slot of v in ring v % d, -1 absent (the paper's
//                          "contiguous 1D array as a hashmap")
//   hslot_of int32 [n]     slot in the host ring
//   tails   int64 [d+1]    next insertion slot per level
//   rows    [d*C][row_bytes] feature rows of the device rings
//
// One batch = lookup (classify every query against the pre-batch state)
// -> the caller gathers rows -> insert. The insert is the exact batch-
// parallel closed form of the sequential ring: with tail t
// and ascending miss list m_0..m_{M-1}, m_j lands in slot (t+j) % C and only
// j >= M-C survive; evictions = #occupied among the first min(M, C) slots +
// max(0, M-C); tail <- (t+M) % C. It is computed slot-centrically (one warp
// per touched slot), so no two writers ever race.
#include <algorithm>
#include <vector>

#include "cache.cuh"
#include "common.cuh"
#include "scan.cuh"

namespace bgl {

constexpr int kCThreads = 256;
constexpr int kCRounds = 4;
constexpr int kCTile = kCThreads * kCRounds;
constexpr int kMaxLevels = 65;   // d <= 64 plus the host level


__global__ void lookup_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int32_t worker,
                              int32_t shard, int32_t d, int64_t C, const int32_t* __restrict__ slot_of,
                              const int32_t* __restrict__ hslot_of, uint8_t* __restrict__ codes,
                              int64_t* __restrict__ src_row, int64_t* __restrict__ counters,
                              const uint8_t* __restrict__ home_of) {
    const int64_t n = *n_dev;
    int64_t c[4] = {0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        const int32_t h = home_of ? (int32_t)home_of[v] : v % d;
        const int32_t s = slot_of[v];
        uint8_t code;
        int64_t src = -1;
        if (s >= 0) {
            code = (h + shard == worker) ? kD : kP;
            src = (int64_t)h * C + s;
        } else if (hslot_of != nullptr && hslot_of[v] >= 0) {
            code = kH;
        } else {
            code = kM;
        }
        c[code]++;
        if (codes) codes[i] = code;
        if (src_row) src_row[i] = src;
    }
    __shared__ int64_t s_c[4];
    if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int64_t w = warp_sum_i64(c[k]);
        if (lane_id() == 0 && w) atomicAdd((unsigned long long*)&s_c[k], (unsigned long long)w);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&counters[0], (unsigned long long)(s_c[0] + s_c[1] + s_c[2] + s_c[3]));
    }
    if (threadIdx.x < 4 && s_c[threadIdx.x])
        atomicAdd((unsigned long long*)&counters[1 + threadIdx.x], (unsigned long long)s_c[threadIdx.x]);
}

// level of a sorted id: shard (dev-missed) and whether it is a full miss
__device__ __forceinline__ void classify(int32_t v, int32_t d, const int32_t* slot_of, const int32_t* hslot_of,
                                         const uint8_t* home_of, int* shard, bool* full) {
    *shard = -1;
    *full = false;
    if (slot_of[v] < 0) {
        *shard = home_of ? (int)home_of[v] : v % d;
        *full = (hslot_of == nullptr) || (hslot_of[v] < 0);
    }
}

__global__ void __launch_bounds__(kCThreads)
miss_count_kernel(const int32_t* __restrict__ sorted_ids, const int64_t* __restrict__ n_dev, int32_t d,
                  const int32_t* __restrict__ slot_of, const int32_t* __restrict__ hslot_of,
                  int64_t* __restrict__ tile_counts, const uint8_t* __restrict__ home_of) {
    __shared__ int64_t s_cnt[kMaxLevels];
    const int64_t n = *n_dev;
    const int64_t tile = blockIdx.x;
    for (int y = threadIdx.x; y <= d; y += blockDim.x) s_cnt[y] = 0;
    __syncthreads();
    if (tile * kCTile < n) {
        for (int r = 0; r < kCRounds; ++r) {
            int64_t e = tile * kCTile + r * kCThreads + threadIdx.x;
            if (e < n) {
                int sh;
                bool full;
                classify(sorted_ids[e], d, slot_of, hslot_of, home_of, &sh, &full);
                if (sh >= 0) atomicAdd((unsigned long long*)&s_cnt[sh], 1ull);
                if (full) atomicAdd((unsigned long long*)&s_cnt[d], 1ull);
            }
        }
    }
    __syncthreads();
    for (int y = threadIdx.x; y <= d; y += blockDim.x) tile_counts[tile * (d + 1) + y] = s_cnt[y];
}

// one block: exclusive scan of tile_counts per level, totals -> mcount
__global__ void miss_scan_kernel(int64_t* __restrict__ tile_counts, int64_t ntiles, int32_t d,
                                 int64_t* __restrict__ mcount) {
    __shared__ int64_t s_red[kCThreads / 32 + 1];
    for (int y = 0; y <= d; ++y) {
        int64_t carry = 0;
        for (int64_t b = 0; b < ntiles; b += blockDim.x) {
            int64_t t = b + threadIdx.x;
            int64_t v = t < ntiles ? tile_counts[t * (d + 1) + y] : 0;
            int64_t tot;
            int64_t ex = block_excl_scan(v, s_red, &tot);
            if (t < ntiles) tile_counts[t * (d + 1) + y] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) mcount[y] = carry;
    }
}

__global__ void __launch_bounds__(kCThreads)
miss_scatter_kernel(const int32_t* __restrict__ sorted_ids, const int64_t* __restrict__ n_dev, int32_t d,
                    const int32_t* __restrict__ slot_of, const int32_t* __restrict__ hslot_of,
                    const int64_t* __restrict__ tile_off, int32_t* __restrict__ lists, int64_t list_cap,
                    const uint8_t* __restrict__ home_of) {
    constexpr int NW = kCThreads / 32;
    __shared__ int32_t s_w[NW][kMaxLevels];
    __shared__ int64_t s_run[kMaxLevels];
    const int64_t n = *n_dev;
    const int64_t tile = blockIdx.x;
    if (tile * kCTile >= n) return;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    for (int y = threadIdx.x; y <= d; y += blockDim.x) s_run[y] = tile_off[tile * (d + 1) + y];
    __syncthreads();
    for (int r = 0; r < kCRounds; ++r) {
        int64_t e = tile * kCTile + r * kCThreads + threadIdx.x;
        int sh = -1;
        bool full = false;
        if (e < n) classify(sorted_ids[e], d, slot_of, hslot_of, home_of, &sh, &full);
        int my_rank_sh = 0, my_rank_h = 0;
        for (int y = 0; y < d; ++y) {
            unsigned m = __ballot_sync(0xffffffffu, sh == y);
            if (sh == y) my_rank_sh = __popc(m & lt);
            if (lane == 0) s_w[wid][y] = __popc(m);
        }
        {
            unsigned m = __ballot_sync(0xffffffffu, full);
            if (full) my_rank_h = __popc(m & lt);
            if (lane == 0) s_w[wid][d] = __popc(m);
        }
        __syncthreads();
        if (sh >= 0) {
            int64_t pos = s_run[sh] + my_rank_sh;
            for (int w = 0; w < wid; ++w) pos += s_w[w][sh];
            lists[(int64_t)sh * list_cap + pos] = (int32_t)e;
        }
        if (full) {
            int64_t pos = s_run[d] + my_rank_h;
            for (int w = 0; w < wid; ++w) pos += s_w[w][d];
            lists[(int64_t)d * list_cap + pos] = (int32_t)e;
        }
        __syncthreads();
        for (int y = threadIdx.x; y <= d; y += blockDim.x) {
            int64_t add = 0;
            for (int w = 0; w < NW; ++w) add += s_w[w][y];
            s_run[y] += add;
        }
        __syncthreads();
    }
}

// Single-pass lookup + insert-list compaction for one device shard (d == 1)
// and an already sorted, distinct batch: classify, count and write the two
// ascending lists (device-missed, full-missed) with a decoupled look-back.
__global__ void __launch_bounds__(kCThreads)
lookup_fused_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int32_t worker, int32_t shard,
                    int64_t C,
                    const int32_t* __restrict__ slot_of, const int32_t* __restrict__ hslot_of,
                    uint8_t* __restrict__ codes, int64_t* __restrict__ src_row, int64_t* __restrict__ counters,
                    ScanState ss, int32_t* __restrict__ lists, int64_t list_cap, int64_t* __restrict__ mcount,
                    int32_t* __restrict__ miss_pos, int64_t* __restrict__ miss_count) {
    constexpr int NW = kCThreads / 32;
    __shared__ int32_t s_w[2][kCRounds][NW];
    __shared__ int64_t s_c[4];
    __shared__ int64_t s_agg[2], s_pre[2], s_slot;
    const int64_t n = *n_dev;
    const int64_t ntiles = n > 0 ? ceil_div(n, kCTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
    unsigned bm_d[kCRounds], bm_f[kCRounds];
    int64_t c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < kCRounds; ++r) {
        const int64_t e = tile * kCTile + r * kCThreads + threadIdx.x;
        bool dm = false, fm = false;
        if (e < n) {
            const int32_t v = ids[e];
            const int32_t s = slot_of[v];
            uint8_t code;
            int64_t src = -1;
            if (s >= 0) {
                code = (worker == shard) ? kD : kP;
                src = s;
            } else {
                dm = true;
                fm = hslot_of == nullptr || hslot_of[v] < 0;
                code = fm ? kM : kH;
            }
            c[code]++;
            if (codes) codes[e] = code;
            if (src_row) src_row[e] = src;
        }
        bm_d[r] = __ballot_sync(0xffffffffu, dm);
        bm_f[r] = __ballot_sync(0xffffffffu, fm);
        if (lane == 0) {
            s_w[0][r][wid] = __popc(bm_d[r]);
            s_w[1][r][wid] = __popc(bm_f[r]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int64_t w = warp_sum_i64(c[k]);
        if (lane == 0 && w) atomicAdd((unsigned long long*)&s_c[k], (unsigned long long)w);
    }
    if (threadIdx.x < 2) {
        int64_t t = 0;
        for (int r = 0; r < kCRounds; ++r)
            for (int w = 0; w < NW; ++w) t += s_w[threadIdx.x][r][w];
        s_agg[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&counters[0], (unsigned long long)(s_c[0] + s_c[1] + s_c[2] + s_c[3]));
        for (int k = 0; k < 4; ++k)
            if (s_c[k]) atomicAdd((unsigned long long*)&counters[1 + k], (unsigned long long)s_c[k]);
    }
    lookback<2>(ss, tile, s_agg, s_pre);
    int64_t run_d = s_pre[0], run_f = s_pre[1];
#pragma unroll
    for (int r = 0; r < kCRounds; ++r) {
        const int64_t e = tile * kCTile + r * kCThreads + threadIdx.x;
        int64_t pd = run_d + __popc(bm_d[r] & lt), pf = run_f + __popc(bm_f[r] & lt);
        for (int w = 0; w < wid; ++w) {
            pd += s_w[0][r][w];
            pf += s_w[1][r][w];
        }
        if ((bm_d[r] >> lane) & 1u) {
            lists[pd] = (int32_t)e;
            if (miss_pos) miss_pos[pd] = (int32_t)e;   // caller-owned copy for the compacted miss gather
        }
        if ((bm_f[r] >> lane) & 1u) lists[list_cap + pf] = (int32_t)e;
        for (int w = 0; w < NW; ++w) {
            run_d += s_w[0][r][w];
            run_f += s_w[1][r][w];
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        mcount[0] = s_pre[0] + s_agg[0];
        mcount[1] = s_pre[1] + s_agg[1];
        if (miss_count) *miss_count = s_pre[0] + s_agg[0];
    }
}

// warp per touched slot r of level y (= blockIdx.y; y == d is the host ring)
__global__ void insert_kernel(const int32_t* __restrict__ sorted_ids, int32_t d, int64_t C, int64_t Ch,
                              int32_t* __restrict__ rings, int32_t* __restrict__ hring, int32_t* __restrict__ slot_of,
                              int32_t* __restrict__ hslot_of, const int64_t* __restrict__ tails,
                              const int64_t* __restrict__ mcount, const int32_t* __restrict__ lists, int64_t list_cap,
                              const unsigned char* __restrict__ batch_rows, unsigned char* __restrict__ rows,
                              int64_t rb, int64_t* __restrict__ counters, int32_t* __restrict__ plan,
                              int64_t plan_stride, int64_t* __restrict__ level_stats) {
    const int y = blockIdx.y;
    const bool host = (y == d);
    const int64_t cap = host ? Ch : C;
    if (cap == 0) return;
    const int64_t M = mcount[y];
    const int64_t lim = M < cap ? M : cap;
    const int64_t t0 = tails[y];
    int32_t* ring = host ? hring : rings + (int64_t)y * C;
    int32_t* index = host ? hslot_of : slot_of;
    const int32_t* list = lists + (int64_t)y * list_cap;
    const int lane = lane_id();
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t ev = 0;
    for (int64_t r = gw; r < lim; r += nw) {
        const int64_t slot = (t0 + r) % cap;
        const int64_t j = r + cap * ((M - 1 - r) / cap);   // last miss landing in this slot
        const int32_t pos = list[j];
        const int32_t v = sorted_ids[pos];
        if (lane == 0) {
            const int32_t old = ring[slot];
            if (old >= 0) {
                index[old] = -1;
                ++ev;
            }
            ring[slot] = v;
            index[v] = (int32_t)slot;
            if (!host && plan != nullptr) {   // deferred row copy (bgl_cache_copy_rows)
                plan[2 * ((int64_t)y * plan_stride + r)] = pos;
                plan[2 * ((int64_t)y * plan_stride + r) + 1] = (int32_t)slot;
            }
        }
        if (!host && batch_rows != nullptr && plan == nullptr) {
            const unsigned char* src = batch_rows + (int64_t)pos * rb;
            unsigned char* dst = rows + ((int64_t)y * C + slot) * rb;
            if ((rb & 15) == 0) {
                for (int64_t b = (int64_t)lane * 16; b < rb; b += 32 * 16)
                    *reinterpret_cast<uint4*>(dst + b) = __ldg(reinterpret_cast<const uint4*>(src + b));
            } else {
                for (int64_t b = (int64_t)lane * 4; b < rb; b += 32 * 4)
                    *reinterpret_cast<uint32_t*>(dst + b) = __ldg(reinterpret_cast<const uint32_t*>(src + b));
            }
        }
    }
    if (lane == 0 && ev) {
        atomicAdd((unsigned long long*)&counters[6], (unsigned long long)ev);
        atomicAdd((unsigned long long*)&level_stats[2 * y + 1], (unsigned long long)ev);
    }
}

// The same insert with one THREAD per touched slot: index/ring/plan updates
// only (no row copy), so a warp per slot would leave 31 lanes idle.
__global__ void insert_index_kernel(const int32_t* __restrict__ sorted_ids, int32_t d, int64_t C, int64_t Ch,
                                    int32_t* __restrict__ rings, int32_t* __restrict__ hring,
                                    int32_t* __restrict__ slot_of, int32_t* __restrict__ hslot_of,
                                    const int64_t* __restrict__ tails, const int64_t* __restrict__ mcount,
                                    const int32_t* __restrict__ lists, int64_t list_cap,
                                    int64_t* __restrict__ counters, int32_t* __restrict__ plan, int64_t plan_stride,
                                    int64_t* __restrict__ level_stats) {
    const int y = blockIdx.y;
    const bool host = (y == d);
    const int64_t cap = host ? Ch : C;
    if (cap == 0) return;
    const int64_t M = mcount[y];
    const int64_t lim = M < cap ? M : cap;
    const int64_t t0 = tails[y];
    int32_t* ring = host ? hring : rings + (int64_t)y * C;
    int32_t* index = host ? hslot_of : slot_of;
    const int32_t* list = lists + (int64_t)y * list_cap;
    int64_t ev = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < lim; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = (t0 + r) % cap;
        const int64_t j = r + cap * ((M - 1 - r) / cap);   // last miss landing in this slot
        const int32_t pos = list[j];
        const int32_t v = sorted_ids[pos];
        const int32_t old = ring[slot];
        if (old >= 0) {
            index[old] = -1;
            ++ev;
        }
        ring[slot] = v;
        index[v] = (int32_t)slot;
        if (!host && plan != nullptr) {
            plan[2 * ((int64_t)y * plan_stride + r)] = pos;
            plan[2 * ((int64_t)y * plan_stride + r) + 1] = (int32_t)slot;
        }
    }
    const int64_t wev = warp_sum_i64(ev);
    if (lane_id() == 0 && wev) {
        atomicAdd((unsigned long long*)&counters[6], (unsigned long long)wev);
        atomicAdd((unsigned long long*)&level_stats[2 * y + 1], (unsigned long long)wev);
    }
}

__global__ void insert_finalize_kernel(int32_t d, int64_t C, int64_t Ch, int64_t* __restrict__ tails,
                                       const int64_t* __restrict__ mcount, int64_t* __restrict__ counters,
                                       int64_t* __restrict__ plan_count, int64_t* __restrict__ level_stats) {
    if (threadIdx.x != 0) return;
    int64_t ins = 0, ev = 0;
    for (int y = 0; y <= d; ++y) {
        const int64_t cap = (y == d) ? Ch : C;
        const int64_t M = mcount[y];
        if (plan_count && y < d) plan_count[y] = M < cap ? M : cap;
        if (cap == 0) continue;
        tails[y] = (tails[y] + M) % cap;
        ins += M;
        ev += M > cap ? M - cap : 0;
        level_stats[2 * y] += M;                       // every insert of a distinct miss counts (cachesim.py:104)
        level_stats[2 * y + 1] += M > cap ? M - cap : 0;   // inserts evicted by later inserts of the batch
    }
    counters[5] += ins;
    counters[6] += ev;
}

// deferred survivor row copy: plan[y][r] = (batch position, ring slot); the
// row of batch position p is batch_rows[row_index ? row_index[p] : p]
__global__ void copy_rows_kernel(const int32_t* __restrict__ plan, const int64_t* __restrict__ plan_count,
                                 int64_t stride, int64_t C, const unsigned char* __restrict__ batch_rows,
                                 unsigned char* __restrict__ rows, int64_t rb, const int32_t* __restrict__ row_index) {
    const int y = blockIdx.y;
    const int64_t cnt = plan_count[y];
    const int lane = lane_id();
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if ((rb & 15) == 0 && rb <= 512) {   // one 16-B piece per lane, two rows in flight per warp
        const int64_t nr = (cnt + 1) >> 1;
        for (int64_t r2 = gw; r2 < nr; r2 += nw) {
            const int64_t ra = r2, rb2 = r2 + nr;
            const bool two = rb2 < cnt;
            const int2 pa = *reinterpret_cast<const int2*>(plan + 2 * ((int64_t)y * stride + ra));
            int2 pb = make_int2(0, 0);
            if (two) pb = *reinterpret_cast<const int2*>(plan + 2 * ((int64_t)y * stride + rb2));
            const int64_t sa = row_index ? (int64_t)row_index[pa.x] : (int64_t)pa.x;
            const int64_t sb = two ? (row_index ? (int64_t)row_index[pb.x] : (int64_t)pb.x) : 0;
            const int64_t b = (int64_t)lane * 16;
            if (b < rb) {
                const uint4 va = *reinterpret_cast<const uint4*>(batch_rows + sa * rb + b);
                uint4 vb = make_uint4(0, 0, 0, 0);
                if (two) vb = *reinterpret_cast<const uint4*>(batch_rows + sb * rb + b);
                *reinterpret_cast<uint4*>(rows + ((int64_t)y * C + pa.y) * rb + b) = va;
                if (two) *reinterpret_cast<uint4*>(rows + ((int64_t)y * C + pb.y) * rb + b) = vb;
            }
        }
        return;
    }
    for (int64_t r = gw; r < cnt; r += nw) {
        const int32_t pos = plan[2 * ((int64_t)y * stride + r)];
        const int32_t slot = plan[2 * ((int64_t)y * stride + r) + 1];
        const int64_t src_row = row_index ? (int64_t)row_index[pos] : (int64_t)pos;
        const unsigned char* src = batch_rows + src_row * rb;
        unsigned char* dst = rows + ((int64_t)y * C + slot) * rb;
        if ((rb & 15) == 0) {
            for (int64_t b = (int64_t)lane * 16; b < rb; b += 32 * 16)
                *reinterpret_cast<uint4*>(dst + b) = *reinterpret_cast<const uint4*>(src + b);
        } else {
            for (int64_t b = (int64_t)lane * 4; b < rb; b += 32 * 4)
                *reinterpret_cast<uint32_t*>(dst + b) = *reinterpret_cast<const uint32_t*>(src + b);
        }
    }
}

// Bulk survivor copy (TMA): the survivors of a level are ascending batch
// positions landing in consecutive ring slots (t + j) % C (cachesim.py:101-103),
// so the destination is one contiguous run per level (two at the ring's wrap).
// A warp takes kCopyChunk plan entries: every lane bulk-loads its row
// (cp.async.bulk global -> shared, completion on the warp's mbarrier), then
// every lane that starts a run of consecutive slots issues ONE bulk store of
// the whole run (shared -> global). The batch rows are read row by row (they
// sit between the batch's hits), the ring is written in long contiguous
// stores; no registers carry the bytes. Needs row_bytes % 16 == 0.
constexpr int kCopyChunk = 16;
constexpr int kCopyWarps = 8;

__device__ __forceinline__ unsigned cache_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kCopyWarps * 32)
copy_rows_bulk_kernel(const int32_t* __restrict__ plan, const int64_t* __restrict__ plan_count, int64_t stride,
                      int64_t C, const unsigned char* __restrict__ batch_rows, unsigned char* __restrict__ rows,
                      int64_t rb, const int32_t* __restrict__ row_index) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kCopyWarps];
    const int y = blockIdx.y;
    const int lane = lane_id(), wid = warp_id();
    unsigned char* stage = smem + (int64_t)wid * kCopyChunk * rb;
    const unsigned bar = cache_smem_u32(&bars[wid]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t cnt = plan_count[y];
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lt = (1u << lane) - 1u;
    unsigned phase = 0;
    for (int64_t j0 = w * kCopyChunk; j0 < cnt; j0 += nw * kCopyChunk) {
        const int m = (int)((cnt - j0) < kCopyChunk ? (cnt - j0) : kCopyChunk);
        int32_t slot = -1;
        int64_t src = 0;
        if (lane < m) {
            const int2 pe = *reinterpret_cast<const int2*>(plan + 2 * ((int64_t)y * stride + j0 + lane));
            slot = pe.y;
            src = row_index ? (int64_t)__ldg(row_index + pe.x) : (int64_t)pe.x;
        }
        // the previous chunk's stores must have read the stage before it is refilled
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"((unsigned)(m * rb))
                         : "memory");
        __syncwarp();
        if (lane < m)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(cache_smem_u32(stage + (int64_t)lane * rb)), "l"(batch_rows + src * rb),
                            "r"((unsigned)rb), "r"(bar) : "memory");
        const int32_t ps = __shfl_up_sync(0xffffffffu, slot, 1);
        const bool start = lane < m && (lane == 0 || ps + 1 != slot);
        const unsigned sm = __ballot_sync(0xffffffffu, start);
        const unsigned after = sm & ~((lt << 1) | 1u);
        const int next = after ? __ffs(after) - 1 : m;
        asm volatile("{\n.reg .pred P;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}"
                     :: "r"(bar), "r"(phase) : "memory");
        phase ^= 1u;
        if (start)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(rows + ((int64_t)y * C + slot) * rb), "r"(cache_smem_u32(stage + (int64_t)lane * rb)),
                            "r"((unsigned)((next - lane) * rb)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int alloc_fill(void** p, size_t bytes, int byte, const char* what) {
    if (bytes == 0) {
        *p = nullptr;
        return BGL_OK;
    }
    BGL_TRY(cuda_status(cudaMalloc(p, bytes), what));
    return cuda_status(cudaMemset(*p, byte, bytes), what);
}

}  // namespace bgl

using namespace bgl;

namespace {

int launch_copy_rows(const bgl_cache* c, const int32_t* plan, const int64_t* plan_count, int64_t stride,
                     const void* batch_rows, const int32_t* row_index, cudaStream_t st) {
    // BGL_COPY_BULK=0: the register-staged warp-per-row copy (A/B)
    static const bool bulk_env = [] {
        const char* e = getenv("BGL_COPY_BULK");
        return !(e && e[0] == '0');
    }();
    // (row_index != NULL: the multi-GPU path reads the rows from another GPU's
    // output over peer memory -- kept on plain loads/stores there)
    const bool bulk = bulk_env && row_index == nullptr && (c->rb % 16) == 0 && ((uintptr_t)batch_rows % 16) == 0 &&
                      c->rb * kCopyChunk * kCopyWarps <= 200 * 1024;
    if (bulk) {
        const size_t smem = (size_t)c->rb * kCopyChunk * kCopyWarps;
        if (smem > 48 * 1024)
            BGL_TRY(cuda_status(cudaFuncSetAttribute(copy_rows_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem), "cudaFuncSetAttribute(copy_rows_bulk)"));
        unsigned gx = (unsigned)std::min<int64_t>(ceil_div(stride, (int64_t)kCopyChunk * kCopyWarps),
                                                  (int64_t)kNumSMs * 4);
        dim3 grid(std::max(gx, 1u), c->d);
        copy_rows_bulk_kernel<<<grid, kCopyWarps * 32, smem, st>>>(plan, plan_count, stride, c->C,
                                                                   (const unsigned char*)batch_rows, c->rows, c->rb,
                                                                   row_index);
        return launch_status("copy_rows_bulk_kernel");
    }
    dim3 grid(grid_for(stride * 32, 256, 8), c->d);
    copy_rows_kernel<<<grid, 256, 0, st>>>(plan, plan_count, stride, c->C, (const unsigned char*)batch_rows, c->rows,
                                           c->rb, row_index);
    return launch_status("copy_rows_kernel");
}

void free_cache(bgl_cache* c) {
    cudaFree(c->slot_of);
    cudaFree(c->hslot_of);
    cudaFree(c->rings);
    cudaFree(c->hring);
    cudaFree(c->tails);
    cudaFree(c->mcount);
    cudaFree(c->rows);
    cudaFree(c->lists);
    cudaFree(c->tile_counts);
    cudaFree(c->level_stats);
    cudaFree(c->lastq);
    cudaFree(c->freq);
    cudaFree(c->tick);
    cudaFree(c->level_tick);
    cudaFree(c->md_stats);
}

}  // namespace

extern "C" {

int bgl_cache_create(int64_t num_nodes, int32_t num_shards, int64_t shard_capacity, int64_t host_capacity,
                     int64_t row_bytes, bgl_cache_t* out) {
    BGL_CHECK_ARG(out, "bgl_cache_create: null out");
    BGL_CHECK_ARG(num_shards >= 1 && num_shards <= kMaxLevels - 1, "num_devices must be in [1, 64]");
    BGL_CHECK_ARG(shard_capacity >= 0 && host_capacity >= 0, "capacities must be >= 0");
    BGL_CHECK_ARG(shard_capacity < (1ll << 31) && host_capacity < (1ll << 31), "capacity must be < 2^31");
    BGL_CHECK_ARG(num_nodes >= 1 && num_nodes < (1ll << 31), "num_nodes must be in [1, 2^31)");
    BGL_CHECK_ARG(row_bytes >= 0 && row_bytes % 4 == 0, "row_bytes must be a multiple of 4");
    bgl_cache* c = new bgl_cache();
    c->n = num_nodes;
    c->d = num_shards;
    c->C = shard_capacity;
    c->Ch = host_capacity;
    c->rb = row_bytes;
    int st = BGL_OK;
    do {
        if ((st = alloc_fill((void**)&c->slot_of, num_nodes * 4, 0xFF, "cache index")) != BGL_OK) break;
        if (host_capacity > 0 &&
            (st = alloc_fill((void**)&c->hslot_of, num_nodes * 4, 0xFF, "cache host index")) != BGL_OK) break;
        if ((st = alloc_fill((void**)&c->rings, (size_t)num_shards * shard_capacity * 4, 0xFF, "cache rings")) != BGL_OK) break;
        if ((st = alloc_fill((void**)&c->hring, (size_t)host_capacity * 4, 0xFF, "cache host ring")) != BGL_OK) break;
        if ((st = alloc_fill((void**)&c->tails, (size_t)(num_shards + 1) * 8, 0, "cache tails")) != BGL_OK) break;
        if ((st = alloc_fill((void**)&c->mcount, (size_t)(num_shards + 1) * 8, 0, "cache mcount")) != BGL_OK) break;
        if ((st = alloc_fill((void**)&c->level_stats, (size_t)(num_shards + 1) * 16, 0, "cache level stats")) != BGL_OK)
            break;
        if (row_bytes > 0 &&
            (st = alloc_fill((void**)&c->rows, (size_t)num_shards * shard_capacity * row_bytes, 0, "cache rows")) != BGL_OK)
            break;
    } while (0);
    if (st != BGL_OK) {
        free_cache(c);
        delete c;
        return st;
    }
    *out = c;
    return BGL_OK;
}

int bgl_cache_destroy(bgl_cache_t c) {
    if (!c) return BGL_OK;
    free_cache(c);
    delete c;
    return BGL_OK;
}

void* bgl_cache_rows(bgl_cache_t c) { return c ? c->rows : nullptr; }

int bgl_cache_reserve_nodes(bgl_cache_t c, int64_t num_nodes, void* stream) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_CHECK_ARG(num_nodes < (1ll << 31), "num_nodes must be < 2^31");
    if (num_nodes <= c->n) return BGL_OK;
    cudaStream_t st = as_stream(stream);
    BGL_TRY(cuda_status(cudaStreamSynchronize(st), "reserve sync"));
    int32_t* arrs[2] = {c->slot_of, c->hslot_of};
    for (int a = 0; a < 2; ++a) {
        if (!arrs[a]) continue;
        int32_t* nw = nullptr;
        BGL_TRY(alloc_fill((void**)&nw, num_nodes * 4, 0xFF, "cache index grow"));
        BGL_TRY(cuda_status(cudaMemcpy(nw, arrs[a], c->n * 4, cudaMemcpyDeviceToDevice), "cache index copy"));
        cudaFree(arrs[a]);
        arrs[a] = nw;
    }
    c->slot_of = arrs[0];
    c->hslot_of = arrs[1];
    BGL_TRY(bgl_cache_ordered_resize(c, num_nodes, nullptr, st));
    c->n = num_nodes;
    return BGL_OK;
}

int bgl_cache_reserve_batch(bgl_cache_t c, int64_t max_batch) {
    BGL_CHECK_ARG(c, "null cache");
    if (max_batch <= c->list_cap) return BGL_OK;
    BGL_TRY(cuda_status(cudaDeviceSynchronize(), "reserve batch sync"));
    cudaFree(c->lists);
    cudaFree(c->tile_counts);
    c->lists = nullptr;
    c->tile_counts = nullptr;
    int64_t cap = std::max<int64_t>(max_batch, 1024);
    c->max_tiles = ceil_div(cap, kCTile);
    BGL_TRY(cuda_status(cudaMalloc((void**)&c->lists, (size_t)(c->d + 1) * cap * 4), "cache lists"));
    // tile counts of the generic path; doubles as the look-back state of the fused one
    BGL_TRY(cuda_status(cudaMalloc((void**)&c->tile_counts, (size_t)(c->d + 1) * c->max_tiles * 8 + 256),
                        "cache tiles"));
    c->list_cap = cap;
    return BGL_OK;
}

int bgl_cache_reset(bgl_cache_t c, void* stream) {
    BGL_CHECK_ARG(c, "null cache");
    cudaStream_t st = as_stream(stream);
    BGL_TRY(cuda_status(cudaMemsetAsync(c->slot_of, 0xFF, c->n * 4, st), "reset"));
    if (c->hslot_of) BGL_TRY(cuda_status(cudaMemsetAsync(c->hslot_of, 0xFF, c->n * 4, st), "reset"));
    if (c->rings) BGL_TRY(cuda_status(cudaMemsetAsync(c->rings, 0xFF, (size_t)c->d * c->C * 4, st), "reset"));
    if (c->hring) BGL_TRY(cuda_status(cudaMemsetAsync(c->hring, 0xFF, (size_t)c->Ch * 4, st), "reset"));
    BGL_TRY(cuda_status(cudaMemsetAsync(c->level_stats, 0, (size_t)(c->d + 1) * 16, st), "reset"));
    return cuda_status(cudaMemsetAsync(c->tails, 0, (size_t)(c->d + 1) * 8, st), "reset");
}

int bgl_cache_lookup(bgl_cache_t c, const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t worker,
                     const int32_t* sorted_ids, const int64_t* n_sorted_dev, int64_t max_sorted, uint8_t* codes,
                     int64_t* src_row, int64_t* counters, void* stream) {
    BGL_CHECK_ARG(c && ids && n_dev && sorted_ids && n_sorted_dev && counters, "bgl_cache_lookup: null pointer");
    const int32_t nglobal = c->global_shards > 0 ? c->global_shards : c->d;
    BGL_CHECK_ARG(worker >= 0 && worker < nglobal, "worker device out of range");
    BGL_CHECK_ARG(max_sorted <= c->list_cap, "batch larger than reserved (call bgl_cache_reserve_batch)");
    cudaStream_t st = as_stream(stream);
    if (c->d == 1 && ids == sorted_ids && n_dev == n_sorted_dev) {
        const int64_t ntiles = std::max<int64_t>(1, ceil_div(max_sorted, kCTile));
        BGL_TRY(reset_scan_state(c->tile_counts, 2, ntiles, st));
        lookup_fused_kernel<<<(unsigned)ntiles, kCThreads, 0, st>>>(
            ids, n_dev, worker, c->shard_index, c->C, c->slot_of, c->hslot_of, codes, src_row, counters,
            make_scan_state(c->tile_counts, 2, ntiles), c->lists, c->list_cap, c->mcount, nullptr, nullptr);
        return launch_status("lookup_fused_kernel");
    }
    if (max_n > 0) {
        lookup_kernel<<<grid_for(max_n, 256), 256, 0, st>>>(ids, n_dev, worker, c->shard_index, c->d, c->C, c->slot_of, c->hslot_of,
                                                            codes, src_row, counters, c->home_of);
        BGL_TRY(launch_status("lookup_kernel"));
    }
    const int64_t ntiles = std::max<int64_t>(1, ceil_div(max_sorted, kCTile));
    miss_count_kernel<<<(unsigned)ntiles, kCThreads, 0, st>>>(sorted_ids, n_sorted_dev, c->d, c->slot_of,
                                                              c->hslot_of, c->tile_counts, c->home_of);
    BGL_TRY(launch_status("miss_count_kernel"));
    miss_scan_kernel<<<1, kCThreads, 0, st>>>(c->tile_counts, ntiles, c->d, c->mcount);
    BGL_TRY(launch_status("miss_scan_kernel"));
    miss_scatter_kernel<<<(unsigned)ntiles, kCThreads, 0, st>>>(sorted_ids, n_sorted_dev, c->d, c->slot_of,
                                                                c->hslot_of, c->tile_counts, c->lists, c->list_cap,
                                                                c->home_of);
    return launch_status("miss_scatter_kernel");
}

int bgl_cache_lookup_misses(bgl_cache_t c, const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t worker,
                            uint8_t* codes, int64_t* src_row, int64_t* counters, int32_t* miss_pos,
                            int64_t* miss_count, void* stream) {
    BGL_CHECK_ARG(c && ids && n_dev && counters && miss_pos && miss_count, "bgl_cache_lookup_misses: null pointer");
    BGL_CHECK_ARG(c->d == 1, "bgl_cache_lookup_misses: single-shard handles only (use bgl_cache_lookup)");
    const int32_t nglobal = c->global_shards > 0 ? c->global_shards : c->d;
    BGL_CHECK_ARG(worker >= 0 && worker < nglobal, "worker device out of range");
    BGL_CHECK_ARG(max_n <= c->list_cap, "batch larger than reserved (call bgl_cache_reserve_batch)");
    cudaStream_t st = as_stream(stream);
    const int64_t ntiles = std::max<int64_t>(1, ceil_div(max_n, kCTile));
    BGL_TRY(reset_scan_state(c->tile_counts, 2, ntiles, st));
    lookup_fused_kernel<<<(unsigned)ntiles, kCThreads, 0, st>>>(
        ids, n_dev, worker, c->shard_index, c->C, c->slot_of, c->hslot_of, codes, src_row, counters,
        make_scan_state(c->tile_counts, 2, ntiles), c->lists, c->list_cap, c->mcount, miss_pos, miss_count);
    return launch_status("lookup_fused_kernel");
}

int bgl_cache_insert(bgl_cache_t c, const int32_t* sorted_ids, int64_t max_sorted, const void* batch_rows,
                     int64_t* counters, void* stream) {
    BGL_CHECK_ARG(c && sorted_ids && counters, "bgl_cache_insert: null pointer");
    BGL_CHECK_ARG(batch_rows == nullptr || c->rb > 0, "cache was created without feature rows");
    cudaStream_t st = as_stream(stream);
    const int64_t cap = std::max(c->C, c->Ch);
    const int64_t work = std::min<int64_t>(max_sorted, cap);
    if (work > 0) {
        const int threads = 256;
        unsigned gx = grid_for(work * 32, threads, 8);
        dim3 grid(gx, c->d + 1);
        insert_kernel<<<grid, threads, 0, st>>>(sorted_ids, c->d, c->C, c->Ch, c->rings, c->hring, c->slot_of,
                                                c->hslot_of, c->tails, c->mcount, c->lists, c->list_cap,
                                                (const unsigned char*)batch_rows, c->rows, c->rb, counters, nullptr, 0,
                                                c->level_stats);
        BGL_TRY(launch_status("insert_kernel"));
    }
    insert_finalize_kernel<<<1, 32, 0, st>>>(c->d, c->C, c->Ch, c->tails, c->mcount, counters, nullptr,
                                             c->level_stats);
    return launch_status("insert_finalize_kernel");
}

int64_t bgl_cache_plan_stride(bgl_cache_t c, int64_t max_sorted) {
    return c ? std::max<int64_t>(1, std::min<int64_t>(max_sorted, c->C)) : 0;
}

int bgl_cache_insert_plan(bgl_cache_t c, const int32_t* sorted_ids, int64_t max_sorted, int32_t* plan,
                          int64_t* plan_count, int64_t* counters, void* stream) {
    BGL_CHECK_ARG(c && sorted_ids && plan && plan_count && counters, "bgl_cache_insert_plan: null pointer");
    cudaStream_t st = as_stream(stream);
    const int64_t stride = bgl_cache_plan_stride(c, max_sorted);
    const int64_t work = std::min<int64_t>(max_sorted, std::max(c->C, c->Ch));
    if (work > 0) {
        dim3 grid(grid_for(work, 256, 8), c->d + 1);
        insert_index_kernel<<<grid, 256, 0, st>>>(sorted_ids, c->d, c->C, c->Ch, c->rings, c->hring, c->slot_of,
                                                  c->hslot_of, c->tails, c->mcount, c->lists, c->list_cap,
                                                  counters, plan, stride, c->level_stats);
        BGL_TRY(launch_status("insert_index_kernel"));
    }
    insert_finalize_kernel<<<1, 32, 0, st>>>(c->d, c->C, c->Ch, c->tails, c->mcount, counters, plan_count,
                                             c->level_stats);
    return launch_status("insert_finalize_kernel");
}

int bgl_cache_copy_rows(bgl_cache_t c, const int32_t* plan, const int64_t* plan_count, int64_t max_sorted,
                        const void* batch_rows, void* stream) {
    BGL_CHECK_ARG(c && plan && plan_count && batch_rows, "bgl_cache_copy_rows: null pointer");
    BGL_CHECK_ARG(c->rb > 0, "cache was created without feature rows");
    const int64_t stride = bgl_cache_plan_stride(c, max_sorted);
    if (c->C == 0 || max_sorted <= 0) return BGL_OK;
    return launch_copy_rows(c, plan, plan_count, stride, batch_rows, nullptr, as_stream(stream));
}

int bgl_cache_copy_rows_indexed(bgl_cache_t c, const int32_t* plan, const int64_t* plan_count, int64_t max_sorted,
                                const void* batch_rows, const int32_t* row_index, void* stream) {
    BGL_CHECK_ARG(c && plan && plan_count && batch_rows && row_index, "bgl_cache_copy_rows_indexed: null pointer");
    BGL_CHECK_ARG(c->rb > 0, "cache was created without feature rows");
    const int64_t stride = bgl_cache_plan_stride(c, max_sorted);
    if (c->C == 0 || max_sorted <= 0) return BGL_OK;
    return launch_copy_rows(c, plan, plan_count, stride, batch_rows, row_index, as_stream(stream));
}

int bgl_cache_level_stats(bgl_cache_t c, int64_t* out_host) {
    BGL_CHECK_ARG(c && out_host, "bgl_cache_level_stats: null pointer");
    BGL_TRY(cuda_status(cudaDeviceSynchronize(), "level stats sync"));
    return cuda_status(cudaMemcpy(out_host, c->level_stats, (size_t)(c->d + 1) * 16, cudaMemcpyDeviceToHost),
                       "level stats copy");
}

int bgl_cache_export(bgl_cache_t c, int64_t* dev_slots_host, int64_t* dev_tails_host, int64_t* host_slots_host,
                     int64_t* host_tail_host) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_TRY(cuda_status(cudaDeviceSynchronize(), "export sync"));
    std::vector<int32_t> tmp;
    if (dev_slots_host && c->C > 0) {
        tmp.resize((size_t)c->d * c->C);
        BGL_TRY(cuda_status(cudaMemcpy(tmp.data(), c->rings, tmp.size() * 4, cudaMemcpyDeviceToHost), "export"));
        for (size_t i = 0; i < tmp.size(); ++i) dev_slots_host[i] = tmp[i];
    }
    std::vector<int64_t> tails(c->d + 1);
    BGL_TRY(cuda_status(cudaMemcpy(tails.data(), c->tails, tails.size() * 8, cudaMemcpyDeviceToHost), "export"));
    if (dev_tails_host)
        for (int i = 0; i < c->d; ++i) dev_tails_host[i] = tails[i];
    if (host_tail_host) *host_tail_host = tails[c->d];
    if (host_slots_host && c->Ch > 0) {
        tmp.resize((size_t)c->Ch);
        BGL_TRY(cuda_status(cudaMemcpy(tmp.data(), c->hring, tmp.size() * 4, cudaMemcpyDeviceToHost), "export"));
        for (size_t i = 0; i < tmp.size(); ++i) host_slots_host[i] = tmp[i];
    }
    return BGL_OK;
}

}  // extern "C"

extern "C" int bgl_cache_set_shard(bgl_cache_t c, int32_t shard_index, int32_t num_global_shards) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_CHECK_ARG(num_global_shards >= 1 && shard_index >= 0 && shard_index < num_global_shards,
                  "shard index out of range");
    BGL_CHECK_ARG(c->d == 1 || num_global_shards == c->d, "a multi-shard handle is its own global sharding");
    c->shard_index = shard_index;
    c->global_shards = num_global_shards;
    return BGL_OK;
}

namespace bgl {
// ring[r] = nodes[r], index[nodes[r]] = r (static warm-up: rings filled once)
__global__ void warm_kernel(const int32_t* __restrict__ nodes, int64_t count, int32_t* __restrict__ ring,
                            int32_t* __restrict__ index) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = nodes[r];
        ring[r] = v;
        index[v] = (int32_t)r;
    }
}
}  // namespace bgl

extern "C" int bgl_cache_warm(bgl_cache_t c, const int32_t* dev_nodes, const int64_t* dev_counts_host,
                              const int32_t* host_nodes, int64_t n_host, void* stream) {
    BGL_CHECK_ARG(c, "null cache");
    cudaStream_t st = as_stream(stream);
    BGL_TRY(bgl_cache_reset(c, stream));
    int64_t off = 0;
    for (int h = 0; h < c->d; ++h) {
        const int64_t cnt = dev_counts_host ? dev_counts_host[h] : 0;
        BGL_CHECK_ARG(cnt >= 0 && cnt <= c->C, "more warm nodes than shard capacity");
        if (cnt > 0) {
            warm_kernel<<<grid_for(cnt, 256), 256, 0, st>>>(dev_nodes + off, cnt, c->rings + (int64_t)h * c->C,
                                                            c->slot_of);
            BGL_TRY(launch_status("warm_kernel"));
        }
        off += cnt;
    }
    BGL_CHECK_ARG(n_host >= 0 && n_host <= c->Ch, "more warm nodes than host capacity");
    if (n_host > 0) {
        warm_kernel<<<grid_for(n_host, 256), 256, 0, st>>>(host_nodes, n_host, c->hring, c->hslot_of);
        BGL_TRY(launch_status("warm_kernel"));
    }
    return BGL_OK;
}

// ---------------------------------------------------------------- sparse node IDs
// Traces whose node IDs are sparse int64 run on dense ranks (bgl_hash_unique:
// the rank order is the ID order, so every ascending insert list is the
// reference's); the shard of a rank is then home_of[rank] = ID % d instead of
// rank % d, and a growing key set remaps the rings' ranks and rebuilds the
// index from them.
namespace bgl {
__global__ void remap_ring_kernel(int32_t* __restrict__ ring, int64_t len, const int32_t* __restrict__ old_to_new,
                                  int32_t* __restrict__ index) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < len; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ring[s];
        if (v < 0) continue;
        const int32_t w = old_to_new ? old_to_new[v] : v;
        ring[s] = w;
        index[w] = (int32_t)s;
    }
}
}  // namespace bgl

extern "C" int bgl_cache_set_home_map(bgl_cache_t c, const uint8_t* home_of) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_CHECK_ARG(home_of == nullptr || c->d <= 255, "home map needs num_devices <= 255");
    c->home_of = home_of;
    return BGL_OK;
}

extern "C" int bgl_cache_remap(bgl_cache_t c, const int32_t* old_to_new, int64_t new_num_nodes, void* stream) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_CHECK_ARG(new_num_nodes >= 1 && new_num_nodes < (1ll << 31), "num_nodes must be in [1, 2^31)");
    cudaStream_t st = as_stream(stream);
    // LRU / LFU per-node state follows its residents to their new ranks
    BGL_TRY(bgl_cache_ordered_resize(c, std::max(new_num_nodes, c->n), old_to_new, st));
    if (new_num_nodes > c->n) {
        BGL_TRY(cuda_status(cudaStreamSynchronize(st), "remap sync"));
        int32_t* arrs[2] = {c->slot_of, c->hslot_of};
        for (int a = 0; a < 2; ++a) {
            if (!arrs[a]) continue;
            cudaFree(arrs[a]);
            arrs[a] = nullptr;
            BGL_TRY(alloc_fill((void**)&arrs[a], new_num_nodes * 4, 0xFF, "cache index remap"));
        }
        c->slot_of = arrs[0];
        c->hslot_of = arrs[1];
        c->n = new_num_nodes;
    } else {
        BGL_TRY(cuda_status(cudaMemsetAsync(c->slot_of, 0xFF, c->n * 4, st), "remap reset"));
        if (c->hslot_of) BGL_TRY(cuda_status(cudaMemsetAsync(c->hslot_of, 0xFF, c->n * 4, st), "remap reset"));
    }
    for (int y = 0; y < c->d; ++y) {
        if (c->C == 0) break;
        remap_ring_kernel<<<grid_for(c->C, 256), 256, 0, st>>>(c->rings + (int64_t)y * c->C, c->C, old_to_new,
                                                               c->slot_of);
        BGL_TRY(launch_status("remap_ring_kernel"));
    }
    if (c->Ch > 0) {
        remap_ring_kernel<<<grid_for(c->Ch, 256), 256, 0, st>>>(c->hring, c->Ch, old_to_new, c->hslot_of);
        BGL_TRY(launch_status("remap_ring_kernel"));
    }
    return BGL_OK;
}
