// K2: sorted distinct node set + relabel (np.unique / return_inverse of
// gnnio/sampler.py:115,157).
//
// Direct-address design: one bit per node ID (n/8 bytes: 0.3 MB at the
// products shape, 13.9 MB at papers100M -- L2-resident on B200). Marking is
// an atomicOr per key; a single decoupled look-back pass over the bitmap
// words yields each word's rank base and emits the set bits in ascending ID
// order, so the output is sorted without a sort. rank(v) = word_rank[v/32] +
// popc(word & below(v)). Reset touches only the words of the emitted IDs.
#include "common.cuh"
#include "scan.cuh"

namespace bgl {

constexpr int kUThreads = 256;
constexpr int kUWordsPerThread = 2;   // small tiles: ~150 CTAs at the products shape
constexpr int kUTileWords = kUThreads * kUWordsPerThread;

struct UniqueWs {
    uint32_t* bitmap;      // [nwords]
    uint32_t* word_rank;   // [nwords]
    void* scan;
    int64_t nwords;
    int64_t max_tiles;
};

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static UniqueWs carve_unique(void* ws, int64_t num_nodes) {
    UniqueWs u;
    u.nwords = ceil_div(num_nodes > 0 ? num_nodes : 1, 32);
    u.nwords = ceil_div(u.nwords, kUWordsPerThread) * kUWordsPerThread;   // whole uint2 loads
    char* p = reinterpret_cast<char*>(ws);
    u.bitmap = reinterpret_cast<uint32_t*>(p);
    p += al256(u.nwords * 4);
    u.word_rank = reinterpret_cast<uint32_t*>(p);
    p += al256(u.nwords * 4);
    u.max_tiles = ceil_div(u.nwords, kUTileWords);
    u.scan = p;
    return u;
}

struct Segs {
    int64_t off[8];
    int64_t max[8];
    int64_t start[9];    // prefix of max: flat index space
    const int64_t* cnt;  // device [nseg]
    int nseg;
};

static int make_segs(Segs& s, int32_t nseg, const int64_t* seg_off, const int64_t* seg_cnt_dev,
                     const int64_t* seg_max) {
    BGL_CHECK_ARG(nseg >= 1 && nseg <= 8, "nseg must be in [1, 8]");
    BGL_CHECK_ARG(seg_off && seg_cnt_dev && seg_max, "segment arrays must be non-null");
    s.nseg = nseg;
    s.cnt = seg_cnt_dev;
    s.start[0] = 0;
    for (int i = 0; i < nseg; ++i) {
        s.off[i] = seg_off[i];
        s.max[i] = seg_max[i];
        s.start[i + 1] = s.start[i] + seg_max[i];
    }
    return BGL_OK;
}

// flat index -> (segment, element) ; returns false when beyond the valid count
__device__ __forceinline__ bool seg_locate(const Segs& s, int64_t g, int64_t* pos) {
    int sg = 0;
#pragma unroll 1
    while (sg + 1 < s.nseg && g >= s.start[sg + 1]) ++sg;
    int64_t e = g - s.start[sg];
    if (e >= s.cnt[sg]) return false;
    *pos = s.off[sg] + e;
    return true;
}

__global__ void mark_kernel(const int32_t* __restrict__ keys, Segs s, uint32_t* __restrict__ bitmap) {
    const int64_t total = s.start[s.nseg];
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos;
        if (!seg_locate(s, g, &pos)) continue;
        uint32_t v = (uint32_t)keys[pos];
        atomicOr(bitmap + (v >> 5), 1u << (v & 31));   // RED: no dependent load
    }
}

__global__ void __launch_bounds__(kUThreads)
emit_kernel(const uint32_t* __restrict__ bitmap, int64_t nwords, ScanState ss,
            uint32_t* __restrict__ word_rank, int32_t* __restrict__ uniq, int64_t* __restrict__ num_uniq) {
    __shared__ int64_t s_red[kUThreads / 32 + 1];
    __shared__ int64_t s_agg[1], s_pre[1], s_slot;
    const int64_t ntiles = ceil_div(nwords, kUTileWords);
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int64_t w0 = tile * kUTileWords + (int64_t)threadIdx.x * kUWordsPerThread;
    uint32_t w[kUWordsPerThread];
    if (w0 < nwords) {
        const uint2 a = *reinterpret_cast<const uint2*>(bitmap + w0);
        w[0] = a.x;
        w[1] = a.y;
    } else {
#pragma unroll
        for (int j = 0; j < kUWordsPerThread; ++j) w[j] = 0;
    }
    int64_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kUWordsPerThread; ++j) cnt += __popc(w[j]);
    int64_t total;
    int64_t ex = block_excl_scan(cnt, s_red, &total);
    if (threadIdx.x == 0) s_agg[0] = total;
    __syncthreads();
    lookback<1>(ss, tile, s_agg, s_pre);
    int64_t r = s_pre[0] + ex;
#pragma unroll
    for (int j = 0; j < kUWordsPerThread; ++j) {
        uint32_t x = w[j];
        if (x) {
            word_rank[w0 + j] = (uint32_t)r;
            const int32_t base = (int32_t)((w0 + j) << 5);
            while (x) {
                int b = __ffs(x) - 1;
                uniq[r++] = base + b;
                x &= x - 1;
            }
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *num_uniq = s_pre[0] + total;
}

__global__ void relabel_kernel(const int32_t* __restrict__ keys, Segs s, const uint32_t* __restrict__ bitmap,
                               const uint32_t* __restrict__ word_rank, int32_t* __restrict__ local) {
    const int64_t total = s.start[s.nseg];
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos;
        if (!seg_locate(s, g, &pos)) continue;
        uint32_t v = (uint32_t)keys[pos];
        uint32_t wd = bitmap[v >> 5];
        local[pos] = (int32_t)(word_rank[v >> 5] + __popc(wd & ((1u << (v & 31)) - 1u)));
    }
}

__global__ void reset_kernel(uint32_t* __restrict__ bitmap, const int32_t* __restrict__ uniq,
                             const int64_t* __restrict__ num_uniq) {
    const int64_t n = *num_uniq;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bitmap[(uint32_t)uniq[i] >> 5] = 0u;
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_unique_workspace(int64_t num_nodes) {
    UniqueWs u = carve_unique(nullptr, num_nodes);
    return al256(u.nwords * 4) * 2 + scan_state_bytes(1, u.max_tiles) + 256;
}

int bgl_unique_workspace_init(void* workspace, int64_t num_nodes, void* stream) {
    BGL_CHECK_ARG(workspace, "bgl_unique_workspace_init: null workspace");
    return cuda_status(cudaMemsetAsync(workspace, 0, bgl_unique_workspace(num_nodes), as_stream(stream)),
                       "unique workspace memset");
}

int bgl_unique_sorted(const int32_t* keys, int32_t nseg, const int64_t* seg_off, const int64_t* seg_cnt_dev,
                      const int64_t* seg_max, int64_t num_nodes, void* workspace, int32_t* uniq_out,
                      int64_t* num_uniq_dev, void* stream) {
    BGL_CHECK_ARG(num_nodes >= 1 && num_nodes < (1ll << 31), "num_nodes must be in [1, 2^31)");
    BGL_CHECK_ARG(workspace && uniq_out && num_uniq_dev, "bgl_unique_sorted: null pointer");
    Segs s;
    BGL_TRY(make_segs(s, nseg, seg_off, seg_cnt_dev, seg_max));
    cudaStream_t st = as_stream(stream);
    UniqueWs u = carve_unique(workspace, num_nodes);
    const int64_t total = s.start[nseg];
    if (total > 0) {
        mark_kernel<<<grid_for(total, 256), 256, 0, st>>>(keys, s, u.bitmap);
        BGL_TRY(launch_status("mark_kernel"));
    }
    BGL_TRY(reset_scan_state(u.scan, 1, u.max_tiles, st));
    ScanState ss = make_scan_state(u.scan, 1, u.max_tiles);
    emit_kernel<<<(unsigned)u.max_tiles, kUThreads, 0, st>>>(u.bitmap, u.nwords, ss, u.word_rank, uniq_out,
                                                               num_uniq_dev);
    return launch_status("emit_kernel");
}

int bgl_relabel(const int32_t* keys, int32_t nseg, const int64_t* seg_off, const int64_t* seg_cnt_dev,
                const int64_t* seg_max, int64_t num_nodes, const void* workspace, int32_t* local, void* stream) {
    BGL_CHECK_ARG(workspace && local, "bgl_relabel: null pointer");
    Segs s;
    BGL_TRY(make_segs(s, nseg, seg_off, seg_cnt_dev, seg_max));
    UniqueWs u = carve_unique(const_cast<void*>(workspace), num_nodes);
    const int64_t total = s.start[nseg];
    if (total == 0) return BGL_OK;
    relabel_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(keys, s, u.bitmap, u.word_rank, local);
    return launch_status("relabel_kernel");
}

int bgl_unique_reset(void* workspace, int64_t num_nodes, const int32_t* uniq, const int64_t* num_uniq_dev,
                     int64_t max_uniq, void* stream) {
    BGL_CHECK_ARG(workspace && uniq && num_uniq_dev, "bgl_unique_reset: null pointer");
    if (max_uniq <= 0) return BGL_OK;
    UniqueWs u = carve_unique(workspace, num_nodes);
    reset_kernel<<<grid_for(max_uniq, 256), 256, 0, as_stream(stream)>>>(u.bitmap, uniq, num_uniq_dev);
    return launch_status("reset_kernel");
}

}  // extern "C"
