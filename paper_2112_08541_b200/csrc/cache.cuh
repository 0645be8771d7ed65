// The FIFO / LRU / LFU cache handle shared by cache.cu and ordered.cu.
#pragma once

#include "common.cuh"

struct bgl_cache {
    int64_t n = 0;          // node-ID space of the index
    int32_t d = 1;
    int64_t C = 0, Ch = 0, rb = 0;
    int32_t* slot_of = nullptr;   // FIFO: slot in ring v % d; LRU/LFU: 0 = resident; -1 absent
    int32_t* hslot_of = nullptr;
    int32_t* rings = nullptr;     // FIFO: ring slots; LRU/LFU: the level's resident list (eviction order)
    int32_t* hring = nullptr;
    int64_t* tails = nullptr;     // [d+1] FIFO: next slot; LRU/LFU: resident count
    int64_t* mcount = nullptr;    // [d+1] misses per level in the current batch
    unsigned char* rows = nullptr;
    int32_t* lists = nullptr;     // [(d+1)][list_cap] positions into sorted_ids
    int64_t list_cap = 0;
    int64_t* tile_counts = nullptr;   // [max_tiles][d+1] (exclusive offsets after scan)
    int64_t max_tiles = 0;
    int32_t shard_index = 0;     // global shard of this handle (multi-GPU: rank)
    int32_t global_shards = 0;   // 0 = d (single process)
    int64_t* level_stats = nullptr;   // [d+1][2] insertions, evictions per level (_Level counters, cachesim.py:45-49)
    const uint8_t* home_of = nullptr; // sparse IDs: shard of each dense rank (caller-owned); null = v % d
    // LRU / LFU (ordered.cu): policy 0 = FIFO, 1 = LRU, 2 = LFU
    int32_t policy = 0;
    int32_t* lastq = nullptr;     // [2][n] LRU: last query index of a hit on the device / host level in the batch, -1 otherwise
    int32_t* freq = nullptr;      // [2][n] LFU: frequency on the node's device level / on the host level
    int64_t* tick = nullptr;      // [2][n] LFU: insertion tick on the device level / the host level
    int64_t* level_tick = nullptr;    // [d+1] LFU: ticks handed out per level (LfuLevel.tick)
    int64_t* md_stats = nullptr;  // [d+1] metadata updates per level (_Level.metadata_updates)
};

namespace bgl {
enum : uint8_t { kD = 0, kP = 1, kH = 2, kM = 3 };
int alloc_fill(void** p, size_t bytes, int byte, const char* what);
}  // namespace bgl

// ordered.cu: resize / rename the per-node LRU / LFU arrays (no-op for FIFO)
int bgl_cache_ordered_resize(bgl_cache* c, int64_t new_n, const int32_t* map, cudaStream_t st);
