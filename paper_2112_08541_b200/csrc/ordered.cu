// LRU and LFU levels of gnnio.cachesim (LruLevel cachesim.py:110-133,
// LfuLevel :136-175) on the device, bit-exact with the reference's
// sequential levels through simulate (cachesim.py:275-363).
//
// Residency inside a batch is the pre-batch one (inserts come after the
// batch, :341-344), so the batch's lookup is the FIFO engine's
// (bgl_cache_lookup: codes + the ascending insert lists per level); hits only
// reorder (LRU move_to_end, :118-120) or count (LFU freq += 1, :150-153).
// Each level keeps its residents as an ordered list in the ring buffer
// (rings / hring, length in tails[y]) and residency in slot_of / hslot_of
// (0 = resident, -1 = absent). One CTA per level applies the batch in
// closed form (oracle/cache_oracle.py OrderedLevel, pinned against the
// reference by tests/golden/ordered.npz):
//   LRU: list in recency order. S = [residents not hit] ++ [hit nodes by
//        their LAST hit of the batch] ++ [inserts, ascending]; each insert
//        evicts the front when full, so e = max(0, len0 + M - C) and the new
//        list is S[e:].
//   LFU: list in insertion-tick order, eviction at the min (freq, tick)
//        (the lazy heap's valid top, :157-163). An insert's key (1, T + j)
//        is above every freq-1 resident and below every freq >= 2 one, so the
//        evictions are the first e of [freq-1 residents] ++ [inserts] --
//        unless the level is full at the first insert with no freq-1
//        resident: then the first eviction is the min-(freq, tick) resident
//        and the next e - 1 are inserts.
// Per level: insertions += M, evictions += e, metadata_updates += hits + M
// (capacity 0: inserts are no-ops, :122, :156).
#include <algorithm>
#include <vector>

#include "cache.cuh"
#include "common.cuh"

namespace bgl {

constexpr int kOThreads = 1024;
constexpr int kOWarps = kOThreads / 32;

__device__ __forceinline__ int level_of(int32_t v, uint8_t code, int32_t d, const uint8_t* home_of) {
    if (code == kH) return d;
    return home_of ? (int)home_of[v] : (int)(v % d);
}

// hits of the batch: LRU records each node's last hit position, LFU adds the
// hit to the node's frequency on that level; metadata updates per level
__global__ void ordered_hits_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                    const uint8_t* __restrict__ codes, int32_t d, int32_t policy,
                                    const uint8_t* __restrict__ home_of, int32_t* __restrict__ lastq,
                                    int32_t* __restrict__ freq, int64_t nn, int64_t* __restrict__ md_stats,
                                    int64_t* __restrict__ counters) {
    const int64_t n = *n_dev;
    int64_t hits = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t code = codes[i];
        if (code == kM) continue;
        const int32_t v = ids[i];
        const int y = level_of(v, code, d, home_of);
        if (policy == 1) atomicMax(lastq + (y == d ? nn : 0) + v, (int32_t)i);
        else atomicAdd(freq + (y == d ? nn : 0) + v, 1);
        atomicAdd((unsigned long long*)(md_stats + y), 1ull);
        ++hits;
    }
    hits = warp_sum_i64(hits);
    if (lane_id() == 0 && hits) atomicAdd((unsigned long long*)(counters + 7), (unsigned long long)hits);
}

__global__ void ordered_reset_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                     const uint8_t* __restrict__ codes, int32_t* __restrict__ lastq, int64_t nn) {
    const int64_t n = *n_dev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t code = codes[i];
        if (code != kM) lastq[(code == kH ? nn : 0) + ids[i]] = -1;
    }
}

// block-wide exclusive scan of 0/1 flags; returns the prefix, *total the sum
__device__ __forceinline__ int block_flag_scan(bool f, int* s_w, int* total) {
    const int lane = lane_id(), wid = warp_id();
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_w[wid] = __popc(m);
    __syncthreads();
    if (wid == 0) {
        const int x = s_w[lane];
        int inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        s_w[lane] = inc - x;
        if (lane == 31) s_w[32] = inc;
    }
    __syncthreads();
    const int r = s_w[wid] + __popc(m & ((1u << lane) - 1u));
    *total = s_w[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ uint64_t block_min_u64(uint64_t v, uint64_t* s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u < v ? u : v;
    }
    if (lane_id() == 0) s[warp_id()] = v;
    __syncthreads();
    if (warp_id() == 0) {
        v = s[lane_id()];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t u = __shfl_xor_sync(0xffffffffu, v, o);
            v = u < v ? u : v;
        }
        if (lane_id() == 0) s[0] = v;
    }
    __syncthreads();
    v = s[0];
    __syncthreads();
    return v;
}

// one CTA per level (blockIdx.x == d: the shared host level)
__global__ void __launch_bounds__(kOThreads)
ordered_update_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                      const uint8_t* __restrict__ codes, const int32_t* __restrict__ sorted_ids, int32_t d,
                      int64_t C, int64_t Ch, int32_t policy, const uint8_t* __restrict__ home_of,
                      int32_t* __restrict__ rings, int32_t* __restrict__ hring, int32_t* __restrict__ slot_of,
                      int32_t* __restrict__ hslot_of, int64_t* __restrict__ tails, const int64_t* __restrict__ mcount,
                      const int32_t* __restrict__ lists, int64_t list_cap, const int32_t* lastq,
                      int32_t* __restrict__ freq, int64_t* __restrict__ tick, int64_t nn,
                      int64_t* __restrict__ level_tick, int64_t* __restrict__ level_stats,
                      int64_t* __restrict__ md_stats, int64_t* __restrict__ counters) {
    __shared__ int s_w[33];
    __shared__ uint64_t s_min[32];
    const int y = blockIdx.x;
    const bool host = y == d;
    const int64_t cap = host ? Ch : C;
    if (cap == 0) return;                       // never resident, inserts are no-ops
    int32_t* log = host ? hring : rings + (int64_t)y * C;
    int32_t* member = host ? hslot_of : slot_of;
    const int64_t len0 = tails[y];
    const int64_t M = mcount[y];
    const int32_t* list = lists + (int64_t)y * list_cap;
    const int64_t e = len0 + M > cap ? len0 + M - cap : 0;
    const int tid = threadIdx.x;
    int64_t out = 0;                            // position in S (before dropping the first e)
    if (policy == 1) {
        // a node may sit on its device level and on the host level: each level kind has its own last-hit array
        lastq += host ? nn : 0;
        // S part 1: residents not hit this batch, recency order (in place: writes trail reads)
        for (int64_t b = 0; b < len0; b += kOThreads) {
            const int64_t t = b + tid;
            const int32_t v = t < len0 ? log[t] : -1;
            const bool keep = t < len0 && lastq[v] < 0;
            int tot;
            const int r = block_flag_scan(keep, s_w, &tot);
            if (keep) {
                const int64_t p = out + r;
                if (p < e) member[v] = -1;      // evicted
                else log[p - e] = v;
            }
            out += tot;
        }
        // S part 2: hit nodes in the order of their last hit
        const int64_t n = *n_dev;
        for (int64_t b = 0; b < n; b += kOThreads) {
            const int64_t i = b + tid;
            bool last = false;
            int32_t v = 0;
            if (i < n) {
                const uint8_t code = codes[i];
                if (code != kM) {
                    v = ids[i];
                    last = level_of(v, code, d, home_of) == y && lastq[v] == (int32_t)i;
                }
            }
            int tot;
            const int r = block_flag_scan(last, s_w, &tot);
            if (last) {
                const int64_t p = out + r;
                if (p < e) member[v] = -1;
                else log[p - e] = v;
            }
            out += tot;
        }
        // S part 3: the inserts, ascending
        for (int64_t j = tid; j < M; j += kOThreads) {
            const int32_t v = sorted_ids[list[j]];
            const int64_t p = out + j;
            if (p >= e) {
                log[p - e] = v;
                member[v] = 0;
            }
        }
    } else {
        int32_t* fq = freq + (host ? nn : 0);
        int64_t* tk = tick + (host ? nn : 0);
        const int64_t k0 = cap > len0 ? cap - len0 : 0;
        // freq-1 residents
        int64_t nA = 0;
        for (int64_t b = 0; b < len0; b += kOThreads) {
            const int64_t t = b + tid;
            int tot;
            block_flag_scan(t < len0 && fq[log[t]] == 1, s_w, &tot);
            nA += tot;
        }
        const bool special = e >= 1 && k0 == 0 && nA == 0;
        int64_t victim = -1;                    // special: position of the min (freq, tick) resident
        if (special) {
            uint64_t best = ~0ull;
            for (int64_t t = tid; t < len0; t += kOThreads) {
                const int32_t v = log[t];
                const uint64_t key = ((uint64_t)fq[v] << 40) | (uint64_t)tk[v];
                if (key < best) best = key;
            }
            best = block_min_u64(best, s_min);
            for (int64_t t = tid; t < len0; t += kOThreads) {
                const int32_t v = log[t];
                if ((((uint64_t)fq[v] << 40) | (uint64_t)tk[v]) == best) victim = t;
            }
            // a unique tick makes the key unique: exactly one thread found it
            if (victim >= 0) s_min[0] = (uint64_t)victim;
            __syncthreads();
            victim = (int64_t)s_min[0];
            __syncthreads();
        }
        const int64_t eA = special ? 0 : (e < nA ? e : nA);   // freq-1 residents evicted
        const int64_t eX = special ? e - 1 : e - eA;          // inserts evicted
        // residents: drop the evicted, keep the tick order (in place)
        int64_t seenA = 0;
        for (int64_t b = 0; b < len0; b += kOThreads) {
            const int64_t t = b + tid;
            const int32_t v = t < len0 ? log[t] : -1;
            const bool isA = t < len0 && fq[v] == 1;
            int totA;
            const int64_t rA = seenA + block_flag_scan(isA, s_w, &totA);
            const bool gone = t < len0 && (special ? t == victim : (isA && rA < eA));
            int tot;
            const int r = block_flag_scan(t < len0 && !gone, s_w, &tot);
            if (gone) {
                member[v] = -1;
                fq[v] = 0;
            } else if (t < len0) {
                log[out + r] = v;
            }
            out += tot;
            seenA += totA;
        }
        // inserts: key (1, T + 1 + j); the first eX are evicted again at once
        const int64_t T = level_tick[y];
        for (int64_t j = tid; j < M; j += kOThreads) {
            const int32_t v = sorted_ids[list[j]];
            if (j >= eX) {
                log[out + j - eX] = v;
                member[v] = 0;
                fq[v] = 1;
                tk[v] = T + 1 + j;
            }
        }
        __syncthreads();
        if (tid == 0) level_tick[y] = T + M;
    }
    // clear the list past its new end, then the counters
    __syncthreads();
    const int64_t len1 = len0 + M - e;
    for (int64_t t = len1 + tid; t < len0; t += kOThreads) log[t] = -1;
    if (tid == 0) {
        tails[y] = len1;
        atomicAdd((unsigned long long*)(counters + 5), (unsigned long long)M);
        atomicAdd((unsigned long long*)(counters + 6), (unsigned long long)e);
        atomicAdd((unsigned long long*)(counters + 7), (unsigned long long)M);
        level_stats[2 * y] += M;
        level_stats[2 * y + 1] += e;
        md_stats[y] += M;
    }
}

// move the LFU state of every resident (on the level's list) to its new rank
__global__ void ordered_rename_kernel(const int32_t* __restrict__ log, const int64_t* __restrict__ len_dev,
                                      const int32_t* __restrict__ map, const int32_t* __restrict__ fq_old,
                                      const int64_t* __restrict__ tk_old, int32_t* __restrict__ fq_new,
                                      int64_t* __restrict__ tk_new) {
    const int64_t len = *len_dev;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = log[t];
        const int32_t w = map ? map[v] : v;
        fq_new[w] = fq_old[v];
        tk_new[w] = tk_old[v];
    }
}

}  // namespace bgl

using namespace bgl;

// Resize the per-node LRU / LFU arrays to new_n nodes; map != NULL renames
// every resident v to map[v] (sparse IDs: the key set grew). Called by
// bgl_cache_reserve_nodes / bgl_cache_remap before the lists are renamed.
int bgl_cache_ordered_resize(bgl_cache_t c, int64_t new_n, const int32_t* map, cudaStream_t st) {
    if (c->policy == 0) return BGL_OK;
    BGL_TRY(cuda_status(cudaStreamSynchronize(st), "ordered resize sync"));
    int32_t* lq = nullptr;
    BGL_TRY(alloc_fill((void**)&lq, 2 * new_n * 4, 0xFF, "lru last-hit"));
    cudaFree(c->lastq);
    c->lastq = lq;
    int32_t* fq = nullptr;
    int64_t* tk = nullptr;
    BGL_TRY(alloc_fill((void**)&fq, 2 * new_n * 4, 0, "lfu freq"));
    BGL_TRY(alloc_fill((void**)&tk, 2 * new_n * 8, 0, "lfu tick"));
    if (c->freq) {
        for (int y = 0; y <= c->d; ++y) {
            const bool host = y == c->d;
            const int64_t cap = host ? c->Ch : c->C;
            if (cap == 0) continue;
            const int32_t* log = host ? c->hring : c->rings + (int64_t)y * c->C;
            const int64_t o0 = host ? c->n : 0, o1 = host ? new_n : 0;
            ordered_rename_kernel<<<grid_for(cap, 256), 256, 0, st>>>(log, c->tails + y, map, c->freq + o0,
                                                                      c->tick + o0, fq + o1, tk + o1);
            BGL_TRY(launch_status("ordered_rename_kernel"));
        }
        BGL_TRY(cuda_status(cudaStreamSynchronize(st), "ordered resize copy"));
    }
    cudaFree(c->freq);
    cudaFree(c->tick);
    c->freq = fq;
    c->tick = tk;
    return BGL_OK;
}

extern "C" {

int bgl_cache_set_policy(bgl_cache_t c, int32_t policy) {
    BGL_CHECK_ARG(c, "null cache");
    BGL_CHECK_ARG(policy >= 0 && policy <= 2, "policy must be 0 (fifo), 1 (lru) or 2 (lfu)");
    BGL_CHECK_ARG(c->rb == 0 || policy == 0, "LRU / LFU levels carry no feature rows");
    if (policy == c->policy) return BGL_OK;
    BGL_CHECK_ARG(c->policy == 0, "the policy of a cache is set once");
    c->policy = policy;
    if (policy == 0) return BGL_OK;
    BGL_TRY(alloc_fill((void**)&c->level_tick, (size_t)(c->d + 1) * 8, 0, "lfu level ticks"));
    BGL_TRY(alloc_fill((void**)&c->md_stats, (size_t)(c->d + 1) * 8, 0, "metadata stats"));
    return bgl_cache_ordered_resize(c, c->n, nullptr, 0);
}

int bgl_cache_update_ordered(bgl_cache_t c, const int32_t* ids, const int64_t* n_dev, int64_t max_n,
                             const uint8_t* codes, const int32_t* sorted_ids, int64_t* counters, void* stream) {
    BGL_CHECK_ARG(c && ids && n_dev && codes && sorted_ids && counters, "bgl_cache_update_ordered: null pointer");
    BGL_CHECK_ARG(c->policy == 1 || c->policy == 2, "bgl_cache_update_ordered: LRU / LFU caches only");
    cudaStream_t st = as_stream(stream);
    if (max_n > 0) {
        ordered_hits_kernel<<<grid_for(max_n, 256), 256, 0, st>>>(ids, n_dev, codes, c->d, c->policy, c->home_of,
                                                                 c->lastq, c->freq, c->n, c->md_stats, counters);
        BGL_TRY(launch_status("ordered_hits_kernel"));
    }
    ordered_update_kernel<<<c->d + 1, kOThreads, 0, st>>>(
        ids, n_dev, codes, sorted_ids, c->d, c->C, c->Ch, c->policy, c->home_of, c->rings, c->hring, c->slot_of,
        c->hslot_of, c->tails, c->mcount, c->lists, c->list_cap, c->lastq, c->freq, c->tick, c->n, c->level_tick,
        c->level_stats, c->md_stats, counters);
    BGL_TRY(launch_status("ordered_update_kernel"));
    if (c->policy == 1 && max_n > 0) {
        ordered_reset_kernel<<<grid_for(max_n, 256), 256, 0, st>>>(ids, n_dev, codes, c->lastq, c->n);
        BGL_TRY(launch_status("ordered_reset_kernel"));
    }
    return BGL_OK;
}

int bgl_cache_export_ordered(bgl_cache_t c, int32_t level, int64_t* list_host, int64_t* len_host, int64_t* freq_host,
                             int64_t* tick_host, int64_t* level_tick_host, int64_t* md_host) {
    BGL_CHECK_ARG(c && list_host && len_host, "bgl_cache_export_ordered: null pointer");
    BGL_CHECK_ARG(level >= 0 && level <= c->d, "level out of range");
    BGL_TRY(cuda_status(cudaDeviceSynchronize(), "export sync"));
    const bool host = level == c->d;
    const int64_t cap = host ? c->Ch : c->C;
    int64_t len = 0;
    BGL_TRY(cuda_status(cudaMemcpy(&len, c->tails + level, 8, cudaMemcpyDeviceToHost), "export len"));
    if (cap == 0) len = 0;
    *len_host = len;
    if (md_host) {
        *md_host = 0;
        if (c->md_stats)
            BGL_TRY(cuda_status(cudaMemcpy(md_host, c->md_stats + level, 8, cudaMemcpyDeviceToHost), "export md"));
    }
    if (c->policy == 0 || len == 0) {
        if (level_tick_host) *level_tick_host = 0;
        if (level_tick_host && c->level_tick)
            BGL_TRY(cuda_status(cudaMemcpy(level_tick_host, c->level_tick + level, 8, cudaMemcpyDeviceToHost), "tick"));
        return BGL_OK;
    }
    std::vector<int32_t> lst(len);
    const int32_t* src = host ? c->hring : c->rings + (int64_t)level * c->C;
    BGL_TRY(cuda_status(cudaMemcpy(lst.data(), src, len * 4, cudaMemcpyDeviceToHost), "export list"));
    for (int64_t i = 0; i < len; ++i) list_host[i] = lst[i];
    if (c->policy == 2 && (freq_host || tick_host)) {
        const int64_t off = host ? c->n : 0;
        std::vector<int32_t> fq(c->n);
        std::vector<int64_t> tk(c->n);
        BGL_TRY(cuda_status(cudaMemcpy(fq.data(), c->freq + off, c->n * 4, cudaMemcpyDeviceToHost), "export freq"));
        BGL_TRY(cuda_status(cudaMemcpy(tk.data(), c->tick + off, c->n * 8, cudaMemcpyDeviceToHost), "export tick"));
        for (int64_t i = 0; i < len; ++i) {
            if (freq_host) freq_host[i] = fq[lst[i]];
            if (tick_host) tick_host[i] = tk[lst[i]];
        }
    }
    if (level_tick_host) {
        *level_tick_host = 0;
        if (c->level_tick)
            BGL_TRY(cuda_status(cudaMemcpy(level_tick_host, c->level_tick + level, 8, cudaMemcpyDeviceToHost), "tick"));
    }
    return BGL_OK;
}

}  // extern "C"
