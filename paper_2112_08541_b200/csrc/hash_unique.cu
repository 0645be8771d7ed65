// Sparse-ID dedup/relabel: a GPU open-addressing hash table (the north_star's
// "GPU open-addressing hash table for unique and relabel") for int64 node IDs
// that are not dense in [0, 2^31).
//
// Semantics = np.unique(keys, return_inverse=True): the distinct keys in
// ascending order plus every key's rank (gnnio/sampler.py:115,157 take the
// sorted distinct set; gnnio's FifoLevel, cachesim.py:81-107, is a dict, so its
// simulate, cachesim.py:275-363, accepts any int64 node ID). The dense path
// (unique.cu: one bit per node, sorted without a sort) stays the default for
// graph node IDs; this one serves traces whose IDs are sparse or >= 2^31.
//
//   1. insert: one thread per key, linear probing from fmix64(key), claim an
//      empty slot with a 64-bit atomicCAS (EMPTY = ~0); the key's table slot
//      is kept for the relabel.
//   2. compact: occupied slots -> unordered distinct list (warp-aggregated
//      atomic append); the slot remembers its list index.
//   3. sort: LSD radix sort of the U distinct keys (8-bit digits, only the
//      passes the caller's key_bits need), each pass a per-tile digit
//      histogram, one digit-major exclusive scan, and a stable scatter (warp
//      __match_any_sync ranks + per-warp digit counts in shared memory).
//   4. rank: rank_of_list[list index] = sorted position; keys -> rank through
//      their table slot.
// Table size = next power of two >= 2 * max_n (load factor <= 0.5), L2-
// resident up to ~4M keys.
#include <algorithm>

#include "common.cuh"

namespace bgl {

constexpr uint64_t kHEmpty = ~0ull;
constexpr int kHThreads = 256;
constexpr int kHItems = 8;                      // keys per thread per radix tile
constexpr int kHTile = kHThreads * kHItems;     // 2048 keys
constexpr int kHRadix = 256;

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

struct HashWs {
    uint64_t* tab;        // [T] keys
    int32_t* tidx;        // [T] list index of the slot's key
    int32_t* qslot;       // [max_n] table slot of each query key
    uint64_t* k0;         // [max_n] distinct keys (ping)
    uint64_t* k1;         // [max_n] (pong)
    int32_t* v0;          // [max_n] list index carried through the sort
    int32_t* v1;
    int32_t* rank_of;     // [max_n] list index -> rank
    uint32_t* hist;       // [kHRadix][max_tiles]
    int64_t* count;       // [1] distinct keys (list length)
    int64_t T, max_n, max_tiles;
};

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

static int64_t table_size(int64_t max_n) {
    int64_t T = 1024;
    while (T < 2 * max_n) T <<= 1;
    return T;
}

static HashWs carve_hash(void* ws, int64_t max_n) {
    HashWs h;
    h.max_n = std::max<int64_t>(max_n, 1);
    h.T = table_size(h.max_n);
    h.max_tiles = ceil_div(h.max_n, kHTile);
    char* p = reinterpret_cast<char*>(ws);
    h.tab = reinterpret_cast<uint64_t*>(p);   p += a256(h.T * 8);
    h.tidx = reinterpret_cast<int32_t*>(p);   p += a256(h.T * 4);
    h.qslot = reinterpret_cast<int32_t*>(p);  p += a256(h.max_n * 4);
    h.k0 = reinterpret_cast<uint64_t*>(p);    p += a256(h.max_n * 8);
    h.k1 = reinterpret_cast<uint64_t*>(p);    p += a256(h.max_n * 8);
    h.v0 = reinterpret_cast<int32_t*>(p);     p += a256(h.max_n * 4);
    h.v1 = reinterpret_cast<int32_t*>(p);     p += a256(h.max_n * 4);
    h.rank_of = reinterpret_cast<int32_t*>(p); p += a256(h.max_n * 4);
    h.hist = reinterpret_cast<uint32_t*>(p);  p += a256((size_t)kHRadix * h.max_tiles * 4);
    h.count = reinterpret_cast<int64_t*>(p);
    return h;
}

__global__ void hash_insert_kernel(const int64_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ tab,
                                   int64_t T, int32_t* __restrict__ qslot) {
    const uint64_t mask = (uint64_t)T - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = (unsigned long long)keys[i];
        uint64_t h = fmix64(k) & mask;
        while (true) {
            const unsigned long long cur = tab[h];
            if (cur == k) break;
            if (cur == kHEmpty) {
                const unsigned long long prev = atomicCAS(tab + h, kHEmpty, k);
                if (prev == kHEmpty || prev == k) break;
            }
            h = (h + 1) & mask;
        }
        qslot[i] = (int32_t)h;
    }
}

// occupied slots -> list (unordered; the sort below fixes the order)
__global__ void hash_compact_kernel(const uint64_t* __restrict__ tab, int64_t T, int32_t* __restrict__ tidx,
                                    uint64_t* __restrict__ klist, int32_t* __restrict__ vlist,
                                    unsigned long long* __restrict__ count) {
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // every lane of a warp runs the same number of iterations (T is a multiple of 32)
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < T; s += stride) {
        const uint64_t k = tab[s];
        const bool occ = k != kHEmpty;
        const unsigned bm = __ballot_sync(0xffffffffu, occ);
        unsigned long long base = 0;
        if (lane == 0 && bm) base = atomicAdd(count, (unsigned long long)__popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (occ) {
            const int32_t pos = (int32_t)(base + __popc(bm & lt));
            klist[pos] = k;
            vlist[pos] = pos;
            tidx[s] = pos;
        }
    }
}

__global__ void __launch_bounds__(kHThreads)
radix_hist_kernel(const uint64_t* __restrict__ k, const int64_t* __restrict__ count, int shift,
                  uint32_t* __restrict__ hist, int64_t ntiles) {
    __shared__ uint32_t s_h[kHRadix];
    const int64_t n = *count;
    const int64_t tile = blockIdx.x;
    s_h[threadIdx.x] = 0;
    __syncthreads();
    for (int r = 0; r < kHItems; ++r) {
        const int64_t i = tile * kHTile + (int64_t)r * kHThreads + threadIdx.x;
        if (i < n) atomicAdd(&s_h[(k[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + tile] = s_h[threadIdx.x];
}

// one CTA: exclusive scan of the digit-major histogram (digit d's tiles are
// contiguous, so the scanned entry is the global offset of (d, tile))
__global__ void __launch_bounds__(1024) radix_scan_kernel(uint32_t* __restrict__ hist, int64_t total) {
    __shared__ uint32_t s_red[1024 / 32 + 1];
    uint32_t carry = 0;
    for (int64_t b = 0; b < total; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const uint32_t v = i < total ? hist[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(v, s_red, &tot);
        if (i < total) hist[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(kHThreads)
radix_scatter_kernel(const uint64_t* __restrict__ kin, const int32_t* __restrict__ vin,
                     uint64_t* __restrict__ kout, int32_t* __restrict__ vout, const int64_t* __restrict__ count,
                     int shift, const uint32_t* __restrict__ hist, int64_t ntiles) {
    constexpr int NW = kHThreads / 32;
    __shared__ uint32_t s_base[kHRadix];
    __shared__ uint32_t s_wc[NW][kHRadix];
    const int64_t n = *count;
    const int64_t tile = blockIdx.x;
    if (tile * kHTile >= n) return;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    s_base[threadIdx.x] = hist[(int64_t)threadIdx.x * ntiles + tile];
    for (int r = 0; r < kHItems; ++r) {
        for (int x = threadIdx.x; x < NW * kHRadix; x += kHThreads) (&s_wc[0][0])[x] = 0;
        __syncthreads();
        const int64_t i = tile * kHTile + (int64_t)r * kHThreads + threadIdx.x;
        const bool has = i < n;
        uint64_t key = 0;
        int32_t val = 0;
        unsigned dg = kHRadix;                 // sentinel digit for lanes past the end
        if (has) {
            key = kin[i];
            val = vin[i];
            dg = (unsigned)(key >> shift) & 255u;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const int rk = __popc(peers & lt);
        if (has && rk == 0) s_wc[wid][dg] = (uint32_t)__popc(peers);
        __syncthreads();
        if (has) {
            uint32_t pos = s_base[dg] + (uint32_t)rk;
            for (int w = 0; w < wid; ++w) pos += s_wc[w][dg];
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        uint32_t add = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) add += s_wc[w][threadIdx.x];
        s_base[threadIdx.x] += add;
        __syncthreads();
    }
}

__global__ void hash_rank_kernel(const uint64_t* __restrict__ ksorted, const int32_t* __restrict__ vsorted,
                                 const int64_t* __restrict__ count, int32_t* __restrict__ rank_of,
                                 int64_t* __restrict__ uniq_out) {
    const int64_t n = *count;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rank_of[vsorted[i]] = (int32_t)i;
        if (uniq_out) uniq_out[i] = (int64_t)ksorted[i];
    }
}

__global__ void hash_relabel_kernel(const int32_t* __restrict__ qslot, const int32_t* __restrict__ tidx,
                                    const int32_t* __restrict__ rank_of, int64_t n, int32_t* __restrict__ rank_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rank_out[i] = rank_of[tidx[qslot[i]]];
}

__global__ void key_home_kernel(const int64_t* __restrict__ keys, const int64_t* __restrict__ n_dev, int64_t max_n,
                                int32_t d, uint8_t* __restrict__ home) {
    const int64_t n = n_dev ? *n_dev : max_n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        home[i] = (uint8_t)(keys[i] % d);
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_hash_unique_workspace(int64_t max_n) {
    const int64_t m = std::max<int64_t>(max_n, 1);
    const int64_t T = table_size(m);
    return a256(T * 8) + a256(T * 4) + a256(m * 4) * 4 + a256(m * 8) * 2 +
           a256((size_t)kHRadix * ceil_div(m, kHTile) * 4) + 256;
}

int bgl_hash_unique(const int64_t* keys, int64_t n, int32_t key_bits, void* workspace, int64_t* uniq_out,
                    int64_t* num_uniq_dev, int32_t* rank_out, void* stream) {
    BGL_CHECK_ARG(n >= 0 && n < (1ll << 31), "bgl_hash_unique: n must be in [0, 2^31)");
    BGL_CHECK_ARG(key_bits >= 0 && key_bits <= 64, "bgl_hash_unique: key_bits must be in [0, 64]");
    BGL_CHECK_ARG(workspace && num_uniq_dev && (n == 0 || keys), "bgl_hash_unique: null pointer");
    cudaStream_t st = as_stream(stream);
    HashWs h = carve_hash(workspace, n);
    BGL_TRY(cuda_status(cudaMemsetAsync(h.tab, 0xFF, h.T * 8, st), "hash table reset"));
    BGL_TRY(cuda_status(cudaMemsetAsync(h.count, 0, 8, st), "hash count reset"));
    if (n > 0) {
        hash_insert_kernel<<<grid_for(n, 256), 256, 0, st>>>(keys, n, (unsigned long long*)h.tab, h.T, h.qslot);
        BGL_TRY(launch_status("hash_insert_kernel"));
        hash_compact_kernel<<<grid_for(h.T, 256), 256, 0, st>>>(h.tab, h.T, h.tidx, h.k0, h.v0,
                                                                (unsigned long long*)h.count);
        BGL_TRY(launch_status("hash_compact_kernel"));
        const int bits = key_bits == 0 ? 64 : key_bits;
        const int passes = (int)ceil_div(bits, 8);
        const int64_t ntiles = ceil_div(n, kHTile);
        uint64_t *ka = h.k0, *kb = h.k1;
        int32_t *va = h.v0, *vb = h.v1;
        for (int p = 0; p < passes; ++p) {
            radix_hist_kernel<<<(unsigned)ntiles, kHThreads, 0, st>>>(ka, h.count, 8 * p, h.hist, ntiles);
            BGL_TRY(launch_status("radix_hist_kernel"));
            radix_scan_kernel<<<1, 1024, 0, st>>>(h.hist, (int64_t)kHRadix * ntiles);
            BGL_TRY(launch_status("radix_scan_kernel"));
            radix_scatter_kernel<<<(unsigned)ntiles, kHThreads, 0, st>>>(ka, va, kb, vb, h.count, 8 * p, h.hist,
                                                                        ntiles);
            BGL_TRY(launch_status("radix_scatter_kernel"));
            std::swap(ka, kb);
            std::swap(va, vb);
        }
        hash_rank_kernel<<<grid_for(n, 256), 256, 0, st>>>(ka, va, h.count, h.rank_of, uniq_out);
        BGL_TRY(launch_status("hash_rank_kernel"));
        if (rank_out) {
            hash_relabel_kernel<<<grid_for(n, 256), 256, 0, st>>>(h.qslot, h.tidx, h.rank_of, n, rank_out);
            BGL_TRY(launch_status("hash_relabel_kernel"));
        }
    }
    return cuda_status(cudaMemcpyAsync(num_uniq_dev, h.count, 8, cudaMemcpyDeviceToDevice, st), "hash count copy");
}

int bgl_key_home(const int64_t* keys, const int64_t* n_dev, int64_t max_n, int32_t num_shards, uint8_t* home,
                 void* stream) {
    BGL_CHECK_ARG(num_shards >= 1 && num_shards <= 255, "bgl_key_home: num_shards must be in [1, 255]");
    BGL_CHECK_ARG(max_n >= 0 && (max_n == 0 || (keys && home)), "bgl_key_home: null pointer");
    if (max_n == 0) return BGL_OK;
    key_home_kernel<<<grid_for(max_n, 256), 256, 0, as_stream(stream)>>>(keys, n_dev, max_n, num_shards, home);
    return launch_status("key_home_kernel");
}

}  // extern "C"
