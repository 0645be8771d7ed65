// K1: one hop of uniform without-replacement neighbour sampling, bit-exact
// with gnnio.sampler._sample_hop (sampler.py:65-94) under PCG64 replay.
//
// Restatement: parent q owns draws
//   u[D + pre_q + t], t in [0, deg_q),  pre_q = sum_{q'<q} deg_q'
// of the batch stream and emits col[off_q + t] for the k = min(fanout, deg)
// smallest (u, t) pairs in ascending order (np.lexsort is stable, so equal
// draws keep adjacency order). u = m * 2^-53 with m the 53-bit integer, so
// comparing (m, t) integer pairs is exact and needs no fp64.
//
// Kernels per hop:
//   hop_scan     decoupled look-back prefix of deg (draw offsets) and k
//                (output offsets) over the parents; writes the chained draw
//                base of the next hop and the output count.
//   sample_warp  k <= 32: one warp walks a contiguous run of parents; lanes
//                hold PCG64 states for 32 consecutive draws and keep a running
//                top-32 of (m, t) keys as a bitonic-sorted warp register
//                list; the state is handed from one parent to the next with a
//                lane rotation (no per-parent jump-ahead).
//   sample_block k > 32 (fanout > 32): one CTA per parent, chunked bitonic
//                sort in shared memory (KCAP <= 4096).
// Only the k selected neighbours are read from col: the draws need deg, not
// the neighbour IDs, so col traffic is k * 4 B per parent, not deg * 4 B.
#include "common.cuh"
#include "pcg64.cuh"
#include "scan.cuh"

namespace bgl {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

struct HopWorkspace {
    int64_t* deg_prefix;   // [max_parents]
    int64_t* k_prefix;     // [max_parents]
    void* scan;            // scan state for 2 values
    int64_t max_tiles;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static HopWorkspace carve_hop_ws(void* ws, int64_t max_parents) {
    HopWorkspace w;
    char* p = reinterpret_cast<char*>(ws);
    int64_t m = max_parents > 0 ? max_parents : 1;
    w.deg_prefix = reinterpret_cast<int64_t*>(p);
    p += align256(m * 8);
    w.k_prefix = reinterpret_cast<int64_t*>(p);
    p += align256(m * 8);
    w.max_tiles = ceil_div(m, kScanTile);
    w.scan = p;
    return w;
}

__global__ void __launch_bounds__(kScanThreads)
hop_scan_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ parents,
                const int64_t* __restrict__ num_parents_dev, int32_t fanout, ScanState ss,
                int64_t* __restrict__ deg_prefix, int64_t* __restrict__ k_prefix,
                int64_t* __restrict__ draw_base, int64_t* __restrict__ num_out) {
    __shared__ int64_t s_deg[kScanTile];
    __shared__ int32_t s_k[kScanTile];
    __shared__ int64_t s_red[kScanThreads / 32 + 1];
    __shared__ int64_t s_agg[2], s_pre[2], s_slot;

    const int64_t n = *num_parents_dev;
    const int64_t ntiles = n > 0 ? ceil_div(n, kScanTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int64_t base = tile * kScanTile;

    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
        int64_t q = base + i;
        int64_t d = 0;
        if (q < n) {
            int64_t p = parents[q];
            d = indptr[p + 1] - indptr[p];
        }
        s_deg[i] = d;
        s_k[i] = (int32_t)(d < fanout ? d : fanout);
    }
    __syncthreads();
    int64_t my_d = 0, my_k = 0;
    const int first = threadIdx.x * kScanItems;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        my_d += s_deg[first + j];
        my_k += s_k[first + j];
    }
    int64_t tot_d, tot_k;
    int64_t ex_d = block_excl_scan(my_d, s_red, &tot_d);
    int64_t ex_k = block_excl_scan(my_k, s_red, &tot_k);
    if (threadIdx.x == 0) {
        s_agg[0] = tot_d;
        s_agg[1] = tot_k;
    }
    __syncthreads();
    lookback<2>(ss, tile, s_agg, s_pre);
    const int64_t pd = s_pre[0], pk = s_pre[1];
    // write blocked results back to smem, then coalesced stores
    int64_t rd = ex_d, rk = ex_k;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t d = s_deg[first + j];
        int64_t k = s_k[first + j];
        s_deg[first + j] = rd;
        s_k[first + j] = (int32_t)rk;
        rd += d;
        rk += k;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
        int64_t q = base + i;
        if (q < n) {
            deg_prefix[q] = pd + s_deg[i];
            k_prefix[q] = pk + s_k[i];
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        draw_base[1] = draw_base[0] + pd + tot_d;
        *num_out = pk + tot_k;
    }
}

// ---------------------------------------------------------------- warp top-k
struct Key {
    uint64_t m;
    uint32_t t;
};

__device__ __forceinline__ bool key_lt(const Key& a, const Key& b) {
    return a.m < b.m || (a.m == b.m && a.t < b.t);
}

__device__ __forceinline__ Key shfl_key(const Key& k, int src) {
    Key r;
    r.m = __shfl_sync(0xffffffffu, k.m, src);
    r.t = __shfl_sync(0xffffffffu, k.t, src);
    return r;
}

__device__ __forceinline__ Key shfl_xor_key(const Key& k, int mask) {
    Key r;
    r.m = __shfl_xor_sync(0xffffffffu, k.m, mask);
    r.t = __shfl_xor_sync(0xffffffffu, k.t, mask);
    return r;
}

// compare-exchange with the partner lane^j; lower lane keeps the min when asc.
__device__ __forceinline__ Key cmpx(const Key& x, int j, bool asc) {
    Key o = shfl_xor_key(x, j);
    bool lower = (lane_id() & j) == 0;
    bool take_min = (lower == asc);
    bool o_lt = key_lt(o, x);
    return (take_min == o_lt) ? o : x;
}

__device__ __forceinline__ Key warp_bitonic_sort(Key x) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) x = cmpx(x, j, (lane & k) == 0);
    }
    return x;
}

__device__ __forceinline__ Key warp_bitonic_merge(Key x) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) x = cmpx(x, j, true);
    return x;
}

constexpr int kWarpsPerBlock = 8;

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
sample_warp_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                   const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                   int32_t fanout, const uint64_t* __restrict__ table,
                   const int64_t* __restrict__ draw_base, const int64_t* __restrict__ deg_prefix,
                   const int64_t* __restrict__ k_prefix, int32_t* __restrict__ out_ids,
                   int32_t* __restrict__ out_pidx, int32_t run) {
    const int64_t n = *num_parents_dev;
    const int lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const PcgTable T{table};
    const U128 A32 = T.A(5), C32 = T.C(5);
    const int64_t D0 = draw_base[0];
    const Key INF{~0ull, ~0u};

    for (int64_t q0 = warp * run; q0 < n; q0 += nwarps * run) {
        const int64_t q1 = min(q0 + run, n);
        bool have = false;
        U128 s{0, 0};
        for (int64_t q = q0; q < q1; ++q) {
            const int32_t p = parents[q];
            const int64_t off = indptr[p];
            const int64_t deg = indptr[p + 1] - off;
            if (deg == 0) continue;                  // consumes no draws (sampler.py:77-79)
            const int k = (int)(deg < fanout ? deg : fanout);
            if (k > 32) {                            // sample_block_kernel's parent
                have = false;
                continue;
            }
            if (!have) {
                s = T.at((uint64_t)(D0 + deg_prefix[q] + lane + 1));
                have = true;
            }
            Key best = INF;
            Key kth = INF;   // current k-th smallest (threshold)
            const int64_t nc = (deg + 31) >> 5;
            for (int64_t c = 0; c < nc; ++c) {
                if (c > 0) s = affine(A32, C32, s);
                const int64_t t = (c << 5) + lane;
                Key cand = INF;
                if (t < deg) {
                    cand.m = draw_of_state(s);
                    cand.t = (uint32_t)t;
                }
                const bool better = key_lt(cand, kth);
                if (!__any_sync(0xffffffffu, better)) continue;
                if (!better) cand = INF;
                cand = warp_bitonic_sort(cand);
                Key rev = shfl_key(cand, 31 - lane);
                if (key_lt(rev, best)) best = rev;
                best = warp_bitonic_merge(best);
                kth = shfl_key(best, k - 1);
            }
            // hand the stream to the next parent: it starts at draw deg (relative)
            {
                const int64_t x = deg + lane;           // wanted relative draw
                const int src = (int)(x & 31);
                U128 r;
                r.hi = __shfl_sync(0xffffffffu, s.hi, src);
                r.lo = __shfl_sync(0xffffffffu, s.lo, src);
                if (x >= (nc << 5)) r = affine(A32, C32, r);
                s = r;
            }
            if (lane < k) {
                const int64_t o = k_prefix[q] + lane;
                out_ids[o] = indices[off + best.t];
                out_pidx[o] = (int32_t)q;
            }
        }
    }
}

// ---------------------------------------------------------------- block top-k
constexpr int kBlockThreads = 256;

__device__ __forceinline__ void smem_bitonic_sort(uint64_t* m, uint32_t* t, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool asc = (i & k) == 0;
                    uint64_t mi = m[i], mj = m[ixj];
                    uint32_t ti = t[i], tj = t[ixj];
                    bool j_lt_i = mj < mi || (mj == mi && tj < ti);
                    if (j_lt_i == asc) {
                        m[i] = mj; m[ixj] = mi;
                        t[i] = tj; t[ixj] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kBlockThreads)
sample_block_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                    const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                    int32_t fanout, int kcap, const uint64_t* __restrict__ table,
                    const int64_t* __restrict__ draw_base, const int64_t* __restrict__ deg_prefix,
                    const int64_t* __restrict__ k_prefix, int32_t* __restrict__ out_ids,
                    int32_t* __restrict__ out_pidx) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* m = reinterpret_cast<uint64_t*>(smem);
    uint32_t* tt = reinterpret_cast<uint32_t*>(smem + sizeof(uint64_t) * 2 * kcap);
    const int64_t n = *num_parents_dev;
    const PcgTable T{table};
    const U128 A256 = T.A(8), C256 = T.C(8);
    const int64_t D0 = draw_base[0];
    for (int64_t q = blockIdx.x; q < n; q += gridDim.x) {
        const int32_t p = parents[q];
        const int64_t off = indptr[p];
        const int64_t deg = indptr[p + 1] - off;
        const int64_t k = deg < fanout ? deg : fanout;
        if (k <= 32) continue;
        for (int i = threadIdx.x; i < kcap; i += blockDim.x) {
            m[i] = ~0ull;
            tt[i] = ~0u;
        }
        const int64_t dq = D0 + deg_prefix[q];
        for (int64_t base = 0; base < deg; base += kcap) {
            U128 s = T.at((uint64_t)(dq + base + threadIdx.x + 1));
            for (int i = threadIdx.x; i < kcap; i += blockDim.x) {
                if (i != (int)threadIdx.x) s = affine(A256, C256, s);
                int64_t t = base + i;
                if (t < deg) {
                    m[kcap + i] = draw_of_state(s);
                    tt[kcap + i] = (uint32_t)t;
                } else {
                    m[kcap + i] = ~0ull;
                    tt[kcap + i] = ~0u;
                }
            }
            __syncthreads();
            smem_bitonic_sort(m, tt, 2 * kcap);
        }
        const int64_t o = k_prefix[q];
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            out_ids[o + i] = indices[off + tt[i]];
            out_pidx[o + i] = (int32_t)q;
        }
        __syncthreads();
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_sample_hop_workspace(int64_t max_parents) {
    int64_t m = max_parents > 0 ? max_parents : 1;
    return align256(m * 8) * 2 + scan_state_bytes(2, ceil_div(m, kScanTile)) + 256;
}

int bgl_sample_hop(const int64_t* indptr, const int32_t* indices, const int32_t* parents,
                   const int64_t* num_parents_dev, int64_t max_parents, int32_t fanout,
                   const uint64_t* table, int64_t* draw_base, int32_t* out_ids,
                   int32_t* out_parent_idx, int64_t* num_out_dev, void* workspace, void* stream) {
    BGL_CHECK_ARG(fanout >= 1, "fanouts must be positive");
    BGL_CHECK_ARG(max_parents >= 0, "bgl_sample_hop: max_parents < 0");
    BGL_CHECK_ARG(indptr && table && draw_base && num_parents_dev && num_out_dev && workspace,
                  "bgl_sample_hop: null pointer");
    cudaStream_t st = as_stream(stream);
    HopWorkspace w = carve_hop_ws(workspace, max_parents);
    BGL_TRY(reset_scan_state(w.scan, 2, w.max_tiles, st));
    ScanState ss = make_scan_state(w.scan, 2, w.max_tiles);
    hop_scan_kernel<<<(unsigned)w.max_tiles, kScanThreads, 0, st>>>(
        indptr, parents, num_parents_dev, fanout, ss, w.deg_prefix, w.k_prefix, draw_base, num_out_dev);
    BGL_TRY(launch_status("hop_scan_kernel"));
    if (max_parents == 0) return BGL_OK;
    // contiguous runs of parents per warp; ~4 runs per resident warp
    const int64_t resident_warps = (int64_t)kNumSMs * 48;
    int64_t run = ceil_div(max_parents, resident_warps * 4);
    if (run < 1) run = 1;
    if (run > 64) run = 64;
    int64_t warps = ceil_div(max_parents, run);
    unsigned blocks = (unsigned)ceil_div(warps, kWarpsPerBlock);
    sample_warp_kernel<<<blocks, kWarpsPerBlock * 32, 0, st>>>(
        indptr, indices, parents, num_parents_dev, fanout, table, draw_base, w.deg_prefix, w.k_prefix,
        out_ids, out_parent_idx, (int32_t)run);
    BGL_TRY(launch_status("sample_warp_kernel"));
    if (fanout > 32) {
        int kcap = 64;
        while (kcap < fanout && kcap < 4096) kcap <<= 1;
        size_t smem = (size_t)2 * kcap * (sizeof(uint64_t) + sizeof(uint32_t));
        if (smem > 48 * 1024)
            BGL_TRY(cuda_status(cudaFuncSetAttribute(sample_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem), "cudaFuncSetAttribute(sample_block)"));
        unsigned grid = grid_for(max_parents, 1, 16);
        sample_block_kernel<<<grid, kBlockThreads, smem, st>>>(
            indptr, indices, parents, num_parents_dev, fanout, kcap, table, draw_base, w.deg_prefix,
            w.k_prefix, out_ids, out_parent_idx);
        BGL_TRY(launch_status("sample_block_kernel"));
    }
    return BGL_OK;
}

}  // extern "C"
