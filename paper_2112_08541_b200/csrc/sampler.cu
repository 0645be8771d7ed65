// K1: one hop of uniform without-replacement neighbour sampling, bit-exact
// with gnnio.sampler._sample_hop (sampler.py:65-94) under PCG64 replay.
//
// Restatement: parent q owns draws
//   u[D + pre_q + t], t in [0, deg_q),  pre_q = sum_{q'<q} deg_q'
// of the batch stream and emits col[off_q + t] for the k = min(fanout, deg)
// smallest (u, t) pairs in ascending order (np.lexsort is stable, so equal
// draws keep adjacency order). u = m * 2^-53 with m the 53-bit integer, so
// comparing (m, t) integer pairs is exact and needs no fp64; for deg <= 2048
// the pair packs into one 64-bit key (m << 11 | t).
//
// Kernels per hop:
//   sample_fused light parents: a warp claims a run of parents (atomic
//                ticket), resolves the run's draw and output offsets with a
//                warp-level decoupled look-back over runs (prefix of deg and
//                of k = min(fanout, deg); the last run writes the chained draw
//                base of the next hop and the output count), lists the heavy
//                parents (deg > 2048 or k > 32), then walks its parents: lanes
//                hold PCG64 states for 32 consecutive draws and keep a running
//                top-k as a warp-distributed sorted list; a chunk of 32 draws is
//                merged by bitonic sort+merge when many lanes beat the current
//                k-th key, else by per-candidate insertion. The stream is handed
//                from one parent to the next with a lane rotation (one
//                jump-ahead per run, not per parent).
//   sample_heavy one CTA per heavy parent: k <= 32 -> 8 warps each keep a
//                top-k over a strided share of the chunks, merged in smem;
//                k > 32 -> chunked bitonic sort in smem (KCAP <= 4096).
// Only the k selected neighbours are read from col: the draws need deg, not
// the neighbour IDs, so col traffic is k * 4 B per parent, not deg * 4 B.
// Optionally every output is also marked in the dedup bitmap (fused K2 mark).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "pcg64.cuh"
#include "scan.cuh"

#include <cub/block/block_radix_sort.cuh>


namespace bgl {

constexpr int64_t kNarrowMaxDeg = 2048;   // t fits 11 bits next to the 53-bit draw
constexpr int kRun = 32;                  // parents per look-back run of the fused kernel

struct HopWorkspace {
    int64_t* deg_prefix;   // [max_parents]
    int64_t* k_prefix;     // [max_parents]
    int32_t* heavy;        // [max_parents] heavy parent positions (unordered)
    int64_t* heavy_count;  // [1]
    void* scan;            // scan state for 2 values
    int64_t max_tiles;
    int32_t* split_ctr;    // [3] split queue: pushed, claimed, runs that have decided (after heavy_count)
    int32_t* split_ready;  // [max_tiles] entry published
    int64_t* split_ent;    // [max_tiles] run << 8 | first parent of the split-off part
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
    w.heavy = reinterpret_cast<int32_t*>(p);
    p += align256(m * 4);
    w.max_tiles = m;                          // look-back runs of the fused kernel (run length >= 1)
    w.scan = p;
    p += align256(scan_state_bytes(2, w.max_tiles));
    w.heavy_count = reinterpret_cast<int64_t*>(p);   // zeroed with the scan state (contiguous)
    w.split_ctr = reinterpret_cast<int32_t*>(p + 64);
    p += 256;
    w.split_ready = reinterpret_cast<int32_t*>(p);   // zeroed too
    p += align256(m * 4);
    w.split_ent = reinterpret_cast<int64_t*>(p);
    return w;
}

// Slice-path workspace, after the HopWorkspace: [prep scan state (4 values) |
// heavy count | HopMeta] (one memset per hop), then the light-parent arrays.
static int64_t prep_tiles(int64_t m) { return ceil_div(m > 0 ? m : 1, 2048); }
// [deg prefix | k prefix | heavy list | scan state | counters (256) | split ready | split entries];
// scan state and counters are zeroed per hop, the split-ready flags when the hop splits
static size_t hop_reset_bytes(int64_t m) { return align256(scan_state_bytes(2, m)) + 256 + align256(m * 4); }
static size_t hop_ws_bytes(int64_t m) { return align256(m * 8) * 2 + align256(m * 4) + hop_reset_bytes(m) + align256(m * 8); }
static size_t slice_reset_bytes(int64_t m) { return align256(scan_state_bytes(5, prep_tiles(m))) + 256; }
static size_t light_list_bytes(int64_t m) { return align256(m * 4) * 3 + align256(m * 8) * 4; }
static size_t slice_ws_bytes(int64_t m) {
    // prep state | wide list | slice map | lane list | perm | tile bases | tile counts
    return slice_reset_bytes(m) + 2 * light_list_bytes(m) + align256((8 * m + 2) * 4) + align256(m * 4) +
           2 * align256(prep_tiles(m) * 4);
}

// fire-and-forget (RED.OR): no dependent load of the word before the atomic
__device__ __forceinline__ void mark_bit(uint32_t* bitmap, int32_t v) {
    atomicOr(bitmap + (v >> 5), 1u << (v & 31));
}

// ---------------------------------------------------------------- key types
// Narrow: 64-bit (m << 11 | t), deg <= 2048. Wide: (m, t) pair.
struct WideKey {
    uint64_t m;
    uint32_t t;
};

__device__ __forceinline__ bool key_lt(uint64_t a, uint64_t b) { return a < b; }
__device__ __forceinline__ bool key_lt(const WideKey& a, const WideKey& b) {
    return a.m < b.m || (a.m == b.m && a.t < b.t);
}
__device__ __forceinline__ uint64_t shfl(uint64_t k, int src) { return __shfl_sync(0xffffffffu, k, src); }
__device__ __forceinline__ WideKey shfl(const WideKey& k, int src) {
    return WideKey{__shfl_sync(0xffffffffu, k.m, src), __shfl_sync(0xffffffffu, k.t, src)};
}
__device__ __forceinline__ uint64_t shfl_xor(uint64_t k, int m) { return __shfl_xor_sync(0xffffffffu, k, m); }
__device__ __forceinline__ WideKey shfl_xor(const WideKey& k, int m) {
    return WideKey{__shfl_xor_sync(0xffffffffu, k.m, m), __shfl_xor_sync(0xffffffffu, k.t, m)};
}
__device__ __forceinline__ uint64_t shfl_up(uint64_t k, int d) { return __shfl_up_sync(0xffffffffu, k, d); }
__device__ __forceinline__ WideKey shfl_up(const WideKey& k, int d) {
    return WideKey{__shfl_up_sync(0xffffffffu, k.m, d), __shfl_up_sync(0xffffffffu, k.t, d)};
}
template <typename K> __device__ __forceinline__ K key_inf();
template <> __device__ __forceinline__ uint64_t key_inf<uint64_t>() { return ~0ull; }
template <> __device__ __forceinline__ WideKey key_inf<WideKey>() { return WideKey{~0ull, ~0u}; }
__device__ __forceinline__ uint64_t make_key(uint64_t m, uint32_t t, uint64_t*) { return (m << 11) | t; }
__device__ __forceinline__ WideKey make_key(uint64_t m, uint32_t t, WideKey*) { return WideKey{m, t}; }
__device__ __forceinline__ uint32_t key_t(uint64_t k) { return (uint32_t)(k & 2047u); }
__device__ __forceinline__ uint32_t key_t(const WideKey& k) { return k.t; }

// compare-exchange with lane^j; the lower lane keeps the min when asc
template <typename K>
__device__ __forceinline__ K cmpx(const K& x, int j, bool asc) {
    K o = shfl_xor(x, j);
    bool lower = (lane_id() & j) == 0;
    return ((lower == asc) == key_lt(o, x)) ? o : x;
}

template <typename K>
__device__ __forceinline__ K warp_bitonic_sort(K x) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) x = cmpx(x, j, (lane & k) == 0);
    }
    return x;
}

template <typename K>
__device__ __forceinline__ K warp_bitonic_merge(K x) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) x = cmpx(x, j, true);
    return x;
}

// best: ascending warp list; merge a sorted candidate list (32 smallest kept)
template <typename K>
__device__ __forceinline__ K merge_sorted(const K& best, const K& sorted_cand) {
    K rev = shfl(sorted_cand, 31 - lane_id());
    K x = key_lt(rev, best) ? rev : best;
    return warp_bitonic_merge(x);
}

constexpr int kInsertMax = 6;   // <= this many passing lanes: insert one by one

// Fold one chunk of candidates (one per lane, INF when invalid) into `best`.
template <typename K>
__device__ __forceinline__ void fold_chunk(K& best, K& kth, K cand, int k) {
    const bool pass = key_lt(cand, kth);
    unsigned mask = __ballot_sync(0xffffffffu, pass);
    if (!mask) return;
    if (__popc(mask) > kInsertMax) {
        if (!pass) cand = key_inf<K>();
        best = merge_sorted(best, warp_bitonic_sort(cand));
    } else {
        const int lane = lane_id();
        while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            const K c = shfl(cand, src);
            const int pos = __popc(__ballot_sync(0xffffffffu, key_lt(best, c)));
            const K up = shfl_up(best, 1);
            if (lane == pos) best = c;
            else if (lane > pos) best = up;
        }
    }
    kth = shfl(best, k - 1);
}

constexpr int kWarpsPerBlock = 8;

// ---------------------------------------------------------------- fused scan + sample
// Warp-level decoupled look-back over runs of `run` (<= kRun) parents: a warp
// claims run r (atomic ticket, so every predecessor is already resident),
// publishes the run's degree and k sums, resolves its exclusive prefix from
// its predecessors, then samples the run. No separate scan pass: only heavy
// parents get their offsets written out (for sample_heavy_kernel).
__device__ __forceinline__ int64_t warp_lookback1(uint64_t* status, int64_t r, int64_t agg) {
    const int lane = lane_id();
    int64_t acc = 0;
    if (r > 0) {
        int64_t j = r - 1;
        while (true) {
            const int64_t idx = j - lane;
            uint64_t w = kFlagInc;
            if (idx >= 0) {
                do { w = ld_status(status + idx); } while ((w >> 62) == 0);
            }
            const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
            const int stop = inc ? __ffs(inc) - 1 : 31;
            acc += warp_sum_i64(lane <= stop ? (int64_t)(w & kValMask) : 0);
            if (inc) break;
            j -= 32;
        }
    }
    if (lane == 0)
        atomicExch((unsigned long long*)(status + r), (unsigned long long)(kFlagInc | ((uint64_t)(acc + agg) & kValMask)));
    return acc;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
sample_fused_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                    const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                    int32_t fanout, const uint64_t* __restrict__ table, int64_t* __restrict__ draw_base,
                    ScanState ss, int64_t* __restrict__ deg_prefix, int64_t* __restrict__ k_prefix,
                    int32_t* __restrict__ heavy, int64_t* __restrict__ heavy_count,
                    int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx, int64_t* __restrict__ num_out,
                    uint32_t* __restrict__ bitmap, int32_t run, int64_t heavy_deg) {
    const int64_t n = *num_parents_dev;
    const int64_t nruns = n > 0 ? ceil_div(n, run) : 1;
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const PcgTable T{table};
    const U128 A32 = T.A(5), C32 = T.C(5);
    const int64_t D0 = draw_base[0];
    const uint64_t INF = ~0ull;
    while (true) {
        int64_t r = 0;
        if (lane == 0) r = (int64_t)atomicAdd(ss.ticket, 1u);
        r = __shfl_sync(0xffffffffu, r, 0);
        if (r >= nruns) break;
        const int64_t q = r * run + lane;
        const bool valid = lane < run && q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        // publish the run's aggregates first (successors never wait on a scan)
        const int64_t incl_d = warp_incl_scan(deg);
        const int64_t incl_k = warp_incl_scan(k);
        const int64_t agg_d = __shfl_sync(0xffffffffu, incl_d, 31);
        const int64_t agg_k = __shfl_sync(0xffffffffu, incl_k, 31);
        if (lane == 0) {
            const uint64_t f = r == 0 ? kFlagInc : kFlagAgg;
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(f | ((uint64_t)agg_d & kValMask)));
            atomicExch((unsigned long long*)(ss.status + ss.max_tiles + r),
                       (unsigned long long)(f | ((uint64_t)agg_k & kValMask)));
        }
        const int64_t pre_d = warp_lookback1(ss.status, r, agg_d);
        const int64_t pre_k = warp_lookback1(ss.status + ss.max_tiles, r, agg_k);
        const int64_t ex_d = pre_d + incl_d - deg;   // draws before this parent (relative to D0)
        const int64_t ex_k = pre_k + incl_k - k;     // outputs before this parent
        const bool hv = valid && (k > 32 || deg > heavy_deg);
        const unsigned hm = __ballot_sync(0xffffffffu, hv);
        if (hm) {
            int64_t slot = 0;
            if (lane == 0) slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, (unsigned long long)__popc(hm));
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (hv) {
                heavy[slot + __popc(hm & lt)] = (int32_t)q;
                deg_prefix[q] = ex_d;
                k_prefix[q] = ex_k;
            }
        }
        if (r == nruns - 1 && lane == 31) {
            draw_base[1] = D0 + pre_d + incl_d;
            *num_out = pre_k + incl_k;
        }
        // sample the run's light parents in order, handing the stream along
        bool have = false;
        U128 s{0, 0};
        const int cnt = (int)((n - r * run) < run ? (n - r * run) : run);
        for (int i = 0; i < cnt; ++i) {
            const int64_t dg = __shfl_sync(0xffffffffu, deg, i);
            if (dg == 0) continue;                    // consumes no draws (sampler.py:77-79)
            const int ki = (int)__shfl_sync(0xffffffffu, k, i);
            if (ki > 32 || dg > heavy_deg) {          // heavy: sample_heavy_kernel
                have = false;
                continue;
            }
            if (!have) {
                s = T.at((uint64_t)(D0 + __shfl_sync(0xffffffffu, ex_d, i) + lane + 1));
                have = true;
            }
            uint64_t best = INF, kth = INF;
            const int64_t nc = (dg + 31) >> 5;
            for (int64_t c = 0; c < nc; ++c) {
                if (c > 0) s = affine(A32, C32, s);
                const int64_t t = (c << 5) + lane;
                const uint64_t cand = t < dg ? make_key(draw_of_state(s), (uint32_t)t, (uint64_t*)nullptr) : INF;
                if (c == 0) {
                    // first chunk: the sorted chunk is the list (no merge with an empty list)
                    best = warp_bitonic_sort(cand);
                    kth = shfl(best, ki - 1);
                } else {
                    fold_chunk(best, kth, cand, ki);
                }
            }
            {
                const int64_t x = dg + lane;
                const int src = (int)(x & 31);
                U128 rr;
                rr.hi = __shfl_sync(0xffffffffu, s.hi, src);
                rr.lo = __shfl_sync(0xffffffffu, s.lo, src);
                if (x >= (nc << 5)) rr = affine(A32, C32, rr);
                s = rr;
            }
            const int64_t oi = __shfl_sync(0xffffffffu, ex_k, i);
            const int64_t offi = __shfl_sync(0xffffffffu, off, i);
            if (lane < ki) {
                const int32_t v = indices[offi + key_t(best)];
                if (out_ids) out_ids[oi + lane] = v;
                if (out_pidx) out_pidx[oi + lane] = (int32_t)(r * run + i);
                if (bitmap) mark_bit(bitmap, v);
            }
        }
    }
}

// ---------------------------------------------------------------- threshold-candidate sampling
// Same look-back prologue and lane-aligned per-parent stream walk as
// sample_fused_kernel, but without a running top-k: a draw is a candidate when
// m < T(k, deg), a per-parent threshold that keeps ~mu = k + 2 sqrt(k) + 1
// of the parent's deg draws. Candidates are appended to a per-warp smem list;
// after the parent's last chunk each candidate's rank is counted by broadcast
// comparisons and the k smallest are written at their rank. Exact: with
// L >= k candidates every non-candidate has m >= T > every candidate's m, so
// the k smallest (m, t) overall are the k smallest candidates. L < k (rare)
// repeats the parent's pass from its first draw with a doubled threshold;
// L > 64 (rarer still) sends it to sample_heavy_kernel.
constexpr int kCandCap = 64;

__device__ __forceinline__ uint64_t cand_threshold(int64_t k, int64_t deg, float ma, float mb) {
    if (deg <= k) return 1ull << 53;
    const double mu = (double)k + (double)ma * sqrt((double)k) + (double)mb;
    if (mu >= (double)deg) return 1ull << 53;
    return (uint64_t)(mu / (double)deg * 9007199254740992.0);
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
sample_cand_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                   const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                   int32_t fanout, const uint64_t* __restrict__ table, int64_t* __restrict__ draw_base,
                   ScanState ss, int64_t* __restrict__ deg_prefix, int64_t* __restrict__ k_prefix,
                   int32_t* __restrict__ heavy, int64_t* __restrict__ heavy_count,
                   int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx, int64_t* __restrict__ num_out,
                   uint32_t* __restrict__ bitmap, int32_t run, int64_t heavy_deg, float ma, float mb) {
    __shared__ uint64_t s_cand[kWarpsPerBlock][kCandCap];
    uint64_t* cand = s_cand[warp_id()];
    const int64_t n = *num_parents_dev;
    const int64_t nruns = n > 0 ? ceil_div(n, run) : 1;
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned FULL = 0xffffffffu;
    const PcgTable T{table};
    const U128 A32 = T.A(5), C32 = T.C(5);
    const int64_t D0 = draw_base[0];
    while (true) {
        int64_t r = 0;
        if (lane == 0) r = (int64_t)atomicAdd(ss.ticket, 1u);
        r = __shfl_sync(FULL, r, 0);
        if (r >= nruns) break;
        const int64_t q = r * run + lane;
        const bool valid = lane < run && q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        const int64_t incl_d = warp_incl_scan(deg);
        const int64_t incl_k = warp_incl_scan(k);
        const int64_t agg_d = __shfl_sync(FULL, incl_d, 31);
        const int64_t agg_k = __shfl_sync(FULL, incl_k, 31);
        if (lane == 0) {
            const uint64_t f = r == 0 ? kFlagInc : kFlagAgg;
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(f | ((uint64_t)agg_d & kValMask)));
            atomicExch((unsigned long long*)(ss.status + ss.max_tiles + r),
                       (unsigned long long)(f | ((uint64_t)agg_k & kValMask)));
        }
        const int64_t pre_d = warp_lookback1(ss.status, r, agg_d);
        const int64_t pre_k = warp_lookback1(ss.status + ss.max_tiles, r, agg_k);
        const int64_t ex_d = pre_d + incl_d - deg;
        const int64_t ex_k = pre_k + incl_k - k;
        const bool hv = valid && (k > 32 || deg > heavy_deg);
        const unsigned hm = __ballot_sync(FULL, hv);
        if (hm) {
            int64_t slot = 0;
            if (lane == 0) slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, (unsigned long long)__popc(hm));
            slot = __shfl_sync(FULL, slot, 0);
            if (hv) {
                heavy[slot + __popc(hm & lt)] = (int32_t)q;
                deg_prefix[q] = ex_d;
                k_prefix[q] = ex_k;
            }
        }
        if (r == nruns - 1 && lane == 31) {
            draw_base[1] = D0 + pre_d + incl_d;
            *num_out = pre_k + incl_k;
        }
        const uint64_t Tm = (valid && !hv) ? cand_threshold(k, deg, ma, mb) : 0;
        bool have = false;
        U128 s{0, 0};
        const int cnt = (int)((n - r * run) < run ? (n - r * run) : run);
        for (int i = 0; i < cnt; ++i) {
            const int64_t dg = __shfl_sync(FULL, deg, i);
            if (dg == 0) continue;                    // consumes no draws (sampler.py:77-79)
            if ((hm >> i) & 1u) {                     // heavy: sample_heavy_kernel
                have = false;
                continue;
            }
            const int ki = (int)__shfl_sync(FULL, k, i);
            const uint64_t tm = __shfl_sync(FULL, Tm, i);
            if (!have) {
                s = T.at((uint64_t)(D0 + __shfl_sync(FULL, ex_d, i) + lane + 1));
                have = true;
            }
            const U128 s_first = s;                       // state of the parent's first draw
            const int nc = (int)((dg + 31) >> 5);
            int L = 0;
            U128 sn;
            uint64_t tcur = tm;
            while (true) {
                L = 0;
                s = s_first;
                for (int c = 0; c < nc; ++c) {
                    const int t = (c << 5) + lane;
                    const uint64_t m = draw_of_state(s);
                    sn = affine(A32, C32, s);            // next chunk (the last one feeds the hand-off)
                    const bool pass = t < dg && m < tcur;
                    const unsigned bm = __ballot_sync(FULL, pass);
                    if (bm) {
                        const int pos = L + __popc(bm & lt);
                        if (pass && pos < kCandCap) cand[pos] = (m << 11) | (uint64_t)t;
                        L += __popc(bm);
                    }
                    if (c + 1 < nc) s = sn;
                }
                // rare: fewer than k candidates -> the same pass with a doubled threshold
                if (L >= ki || tcur >= (1ull << 53)) break;
                tcur = tcur > (1ull << 52) ? (1ull << 53) : tcur * 2;
                __syncwarp();
            }
            {   // hand the stream to the next parent: lane l gets draw (dg + l) of this parent's stream
                const int x = (int)(dg & 31) + lane;                   // offset into chunk nc-1 (if <32) else chunk nc
                const int src = x & 31;
                const bool nxt = ((int64_t)((nc - 1) << 5) + x) >= ((int64_t)nc << 5);
                const uint64_t ahi = __shfl_sync(FULL, s.hi, src), alo = __shfl_sync(FULL, s.lo, src);
                const uint64_t bhi = __shfl_sync(FULL, sn.hi, src), blo = __shfl_sync(FULL, sn.lo, src);
                // dg not a multiple of 32: lanes with dg%32 + lane < 32 stay in chunk nc-1
                const bool use_next = (dg & 31) == 0 ? true : nxt;
                s.hi = use_next ? bhi : ahi;
                s.lo = use_next ? blo : alo;
            }
            __syncwarp();
            const int64_t oi = __shfl_sync(FULL, ex_k, i);
            const int64_t gq = r * run + i;
            if (L > kCandCap) {                       // rarer still (a doubled threshold kept > 64): CTA kernel
                const int64_t dq = __shfl_sync(FULL, ex_d, i);
                if (lane == 0) {
                    const int64_t slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, 1ull);
                    heavy[slot] = (int32_t)gq;
                    deg_prefix[gq] = dq;
                    k_prefix[gq] = oi;
                }
                __syncwarp();
                continue;
            }
            const int64_t offi = __shfl_sync(FULL, off, i);
            const uint64_t c0 = lane < L ? cand[lane] : ~0ull;
            int r0 = 0;
            if (L <= 32) {
#pragma unroll 4
                for (int j = 0; j < L; ++j) r0 += cand[j] < c0;
            } else {
                const uint64_t c1 = lane + 32 < L ? cand[32 + lane] : ~0ull;
                int r1 = 0;
#pragma unroll 4
                for (int j = 0; j < L; ++j) {
                    const uint64_t kj = cand[j];
                    r0 += kj < c0;
                    r1 += kj < c1;
                }
                if (lane + 32 < L && r1 < ki) {
                    const int32_t v = indices[offi + (int64_t)(c1 & 2047u)];
                    if (out_ids) out_ids[oi + r1] = v;
                    if (out_pidx) out_pidx[oi + r1] = (int32_t)gq;
                    if (bitmap) mark_bit(bitmap, v);
                }
            }
            if (lane < L && r0 < ki) {
                const int32_t v = indices[offi + (int64_t)(c0 & 2047u)];
                if (out_ids) out_ids[oi + r0] = v;
                if (out_pidx) out_pidx[oi + r0] = (int32_t)gq;
                if (bitmap) mark_bit(bitmap, v);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- segmented threshold walk
// The draws of a run's parents are consecutive in the batch stream, so the
// warp walks the run's light draws as ONE sequence (lane l takes walk position
// W + l, chunk after chunk) instead of parent by parent: no per-parent stream
// hand-off, no half-empty last chunk per parent. Heavy and degree-0 parents
// have walk length 0; a lane whose next draw lies past a heavy parent's draws
// jumps its PCG64 state over them (gap[j] = heavy draws before parent j). A
// draw of parent j is a candidate when m < T_j (as in sample_cand_kernel);
// candidates are appended in walk order, so each parent's candidates are one
// contiguous range of the warp's list and a candidate's rank is counted over
// its own range only. A parent with fewer than k candidates (or whose range
// overflowed the list) is redone exactly with a warp top-k over all its draws.
constexpr int kSegCap = 512;

// Diagnostics (tools/seg_timeline.py, bgl_debug_seg_trace): when set, lane 0
// of every run appends a 16-word record {n, r, smid, Wtot, t_claim, t_walk,
// t_post, t_end, t_loaded, t_prefix, 0...} (globaltimer ns; t_loaded once
// the run's degrees are in registers, t_prefix once both look-backs are
// done) -- the per-run timeline behind DESIGN.md's sampler notes.
__device__ unsigned long long* g_seg_trace = nullptr;
constexpr int kSegTraceWords = 16;
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// globaltimer read after `dep` is available (the asm consumes it)
__device__ __forceinline__ uint64_t gtimer_after(int64_t dep) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "l"(dep));
    return t;
}
__device__ __noinline__ void seg_trace_record(unsigned long long* trace, int64_t n, int64_t r, int32_t Wtot,
                                              const uint64_t* ts) {
    const uint64_t t_claim = ts[0], t_loaded = ts[1], t_prefix = ts[2], t_walk = ts[3], t_post = ts[4];
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    const unsigned long long slot = atomicAdd(trace, 1ull);
    unsigned long long* rec = trace + kSegTraceWords + kSegTraceWords * slot;
    rec[0] = (unsigned long long)n;
    rec[1] = (unsigned long long)r;
    rec[2] = sm;
    rec[3] = (unsigned long long)Wtot;
    rec[4] = t_claim;
    rec[5] = t_walk;
    rec[6] = t_post;
    rec[7] = gtimer();
    rec[8] = t_loaded;
    rec[9] = t_prefix;
}

struct SegWarp {
    uint64_t cand[kSegCap];
    uint32_t thr[33];    // high-word thresholds; [32]: sentinel 0 (lanes past the run's draws never pass)
    int64_t gap[33];
    int32_t wst[33];
    int32_t wend[33];    // [32]: sentinel INT_MAX (ends the parent search)
    int32_t cst[33];     // seg_post: each parent's candidate range start; [32] = list length
    uint8_t cj[kSegCap];
    uint64_t ts[6];      // diagnostics: claim, loaded, prefix, walk, post (lane 0; kept out of registers)
};

// The lane's parent bound / threshold / walk start stay in registers and are
// reloaded only when the lane crosses into the next parent.
__device__ __forceinline__ void seg_take(SegWarp& sw, int w, int& j, int& nb, uint32_t& th, int& ws) {
    if (w >= nb) {
        do {
            ++j;
            nb = sw.wend[j];
        } while (w >= nb);
        th = sw.thr[j];
        ws = sw.wst[j];
    }
}

// High word of a candidate threshold: out < (thh << 32). Rounding T << 11 up
// to a multiple of 2^32 keeps the candidate set a threshold set (every
// non-candidate's m is strictly above every candidate's), so the selection
// stays exact and the walk compares one 32-bit word per draw.
__device__ __forceinline__ uint32_t thr_hi(uint64_t tm /* T, <= 2^53 */) {
    if (tm >= (1ull << 53)) return 0xffffffffu;   // every draw but out_hi == 2^32 - 1 (the largest m)
    const uint64_t t = tm << 11;
    const uint64_t h = (t >> 32) + ((t & 0xffffffffull) != 0);
    return h > 0xffffffffull ? 0xffffffffu : (uint32_t)h;
}

// Walk the run's light draws in chunks of 32; returns the candidate count.
// Per chunk: the 128-bit affine step (affine_cc), the high word of XSL-RR,
// one 32-bit compare, a ballot and a branch-free append (every lane forms its
// key, passing lanes store it: faster than a branch around the append, whose
// body runs in ~97% of chunks anyway).
// The state of walk position w (parent j) is s0 advanced by d_run + gap_j + w + 1.
template <bool kGaps>
__device__ __forceinline__ int seg_walk(SegWarp& sw, const PcgTable T, U128 A32, U128 C32, U128 s0, int64_t d_run,
                                        int32_t Wtot, int lane, unsigned lt, int cap) {
    int j = 0;
    while (lane >= sw.wend[j]) ++j;
    int nb = sw.wend[j], ws = sw.wst[j];
    uint32_t th = sw.thr[j];
    int64_t g = kGaps ? sw.gap[j] : 0;
    U128 s = T.adv(s0, (uint64_t)(d_run + lane + g + 1));
    int L = 0;
    const int wlim = Wtot + lane;
    for (int w = lane; w < wlim; w += 32) {
        if (w >= nb) {
            seg_take(sw, w, j, nb, th, ws);
            if (kGaps) {
                const int64_t gj = sw.gap[j];
                if (gj != g && w < Wtot) {          // heavy parents' draws lie between
                    s = T.adv(s, (uint64_t)(gj - g));
                    g = gj;
                }
            }
        }
        const uint32_t hh = (uint32_t)(s.hi >> 32);
        const uint32_t xl = (uint32_t)s.lo ^ (uint32_t)s.hi, xh = (uint32_t)(s.lo >> 32) ^ hh;
        const uint32_t rot = hh >> 26;
        const uint32_t a = (rot & 32u) ? xl : xh, b = (rot & 32u) ? xh : xl;
        const uint32_t out_hi = __funnelshift_r(a, b, rot);
        const bool pass = out_hi < th;
        const unsigned bm = __ballot_sync(0xffffffffu, pass);
        // every lane forms its key, passing lanes store it
        const int pos = L + __popc(bm & lt);
        const uint32_t out_lo = __funnelshift_r(b, a, rot);
        const uint64_t key = ((uint64_t)out_hi << 32) | (uint64_t)((out_lo & ~2047u) | (uint32_t)(w - ws));
        if (pass && pos < cap) {
            sw.cand[pos] = key;
            sw.cj[pos] = (uint8_t)j;
        }
        L += __popc(bm);
        s = affine_cc(A32, C32, s);
    }
    return L;
}

// Ranking + output of one run/group after its walk (lane i = parent i):
// each parent's candidates are one range of the (parent-ordered) list; the
// k smallest are written at their rank. Parents with fewer than k candidates
// (or whose range was cut by the list's end) take an exact warp top-k over
// all their draws (first draw's state: s0 advanced by dpos + 1).
__device__ __forceinline__ void seg_post(SegWarp& sw, int L, int cap, int lane, int k, int64_t off, int64_t ex_k,
                                         bool light, int64_t deg, U128 s0, uint64_t dpos, int32_t pid,
                                         const PcgTable T, U128 A32, U128 C32,
                                         const int32_t* __restrict__ indices, int32_t* __restrict__ out_ids,
                                         int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap) {
    const unsigned FULL = 0xffffffffu;
    const int Ls = L < cap ? L : cap;
    int lo = 0, hi = Ls;                    // first index with cj >= lane
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int)sw.cj[mid] < lane) lo = mid + 1; else hi = mid;
    }
    const int c_st = lo;
    const int c_end = __shfl_down_sync(FULL, c_st, 1);
    const int c_own = lane < 31 ? c_end - c_st : Ls - c_st;
    // a range touching the list's end is incomplete when the list overflowed
    const bool cut = L > cap && c_st + c_own >= Ls;
    sw.cst[lane] = c_st;
    if (lane == 0) sw.cst[32] = Ls;
    const bool fb = light && (c_own < k || cut);
    __syncwarp();
    // rank each candidate over its parent's range, write the k smallest at their rank
    for (int b0 = 0; b0 < Ls; b0 += 32) {
        const int i = b0 + lane;
        const bool has = i < Ls;
        const uint64_t key = has ? sw.cand[i] : ~0ull;
        const int j = has ? (int)sw.cj[i] : 0;
        const int kj = __shfl_sync(FULL, k, j);
        const int64_t offj = __shfl_sync(FULL, off, j);
        const int64_t oij = __shfl_sync(FULL, ex_k, j);
        const bool fbj = __shfl_sync(FULL, (int)fb, j) != 0;
        const int32_t pj = __shfl_sync(FULL, pid, j);
        if (has && !fbj) {
            const int st = sw.cst[j], e = sw.cst[j + 1];
            int rk = 0;
            for (int x = st; x < e; ++x) rk += sw.cand[x] < key;
            if (rk < kj) {
                const int32_t v = indices[offj + (int64_t)(key & 2047u)];
                if (out_ids) out_ids[oij + rk] = v;
                if (out_pidx) out_pidx[oij + rk] = pj;
                if (bitmap) mark_bit(bitmap, v);
            }
        }
    }
    // fallback: exact warp top-k over all of the parent's draws
    unsigned fm = __ballot_sync(FULL, fb);
    while (fm) {
        const int i = __ffs(fm) - 1;
        fm &= fm - 1;
        const int64_t dg = __shfl_sync(FULL, deg, i);
        const int ki = __shfl_sync(FULL, k, i);
        U128 s = T.adv(s0, __shfl_sync(FULL, dpos, i) + (uint64_t)lane + 1);
        uint64_t best = ~0ull, kth = ~0ull;
        const int nc = (int)((dg + 31) >> 5);
        for (int c = 0; c < nc; ++c) {
            if (c > 0) s = affine(A32, C32, s);
            const int t = (c << 5) + lane;
            const uint64_t cand = t < dg ? ((draw_of_state(s) << 11) | (uint64_t)t) : ~0ull;
            if (c == 0) {
                best = warp_bitonic_sort(cand);
                kth = shfl(best, ki - 1);
            } else {
                fold_chunk(best, kth, cand, ki);
            }
        }
        const int64_t oi = __shfl_sync(FULL, ex_k, i);
        const int64_t offi = __shfl_sync(FULL, off, i);
        const int32_t pi = __shfl_sync(FULL, pid, i);
        if (lane < ki) {
            const int32_t v = indices[offi + key_t(best)];
            if (out_ids) out_ids[oi + lane] = v;
            if (out_pidx) out_pidx[oi + lane] = pi;
            if (bitmap) mark_bit(bitmap, v);
        }
    }
    __syncwarp();
}

// One part of a run (lane i = parent i of the part; invalid lanes take no
// part): walk layout of its light parents, the walk from the part's first
// draw (D0 + ex_d of lane 0), ranking/output and fallbacks.
__device__ __forceinline__ void seg_part(SegWarp& sw, bool valid, int64_t off, int64_t deg, int64_t k, int64_t ex_d,
                                         int64_t ex_k, bool hv, int32_t pid, int64_t D0, const PcgTable T, U128 A32,
                                         U128 C32, int lane, unsigned lt, int cap, float ma, float mb,
                                         const int32_t* __restrict__ indices, int32_t* __restrict__ out_ids,
                                         int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap,
                                         bool trace, int32_t& Wtot_out) {
    const unsigned FULL = 0xffffffffu;
    const int64_t ex0 = __shfl_sync(FULL, ex_d, 0);
    const bool light = valid && !hv && deg > 0;
    const int32_t ldeg = light ? (int32_t)deg : 0;
    const int32_t incl_l = warp_incl_scan(ldeg);
    const int32_t Wtot = __shfl_sync(FULL, incl_l, 31);
    sw.wst[lane] = incl_l - ldeg;
    sw.wend[lane] = incl_l;
    sw.gap[lane] = (ex_d - ex0) - (int64_t)(incl_l - ldeg);
    // T = 2^53 ("every draw") -> 2^32 - 1, which drops only draws with
    // out_hi = 2^32 - 1: the largest m, so either k others remain or the
    // parent takes the exact fallback (fewer than k candidates)
    sw.thr[lane] = light ? thr_hi(cand_threshold(k, deg, ma, mb)) : 0u;
    if (lane == 0) {
        sw.wend[32] = 0x7fffffff;
        sw.thr[32] = 0;
        sw.gap[32] = 0;
        sw.wst[32] = 0;
    }
    const unsigned hm = __ballot_sync(FULL, valid && hv);
    __syncwarp();
    int L = 0;
    if (trace && lane == 0) sw.ts[3] = gtimer();
    if (Wtot > 0) L = hm ? seg_walk<true>(sw, T, A32, C32, T.state(), D0 + ex0, Wtot, lane, lt, cap)
                         : seg_walk<false>(sw, T, A32, C32, T.state(), D0 + ex0, Wtot, lane, lt, cap);
    __syncwarp();
    if (trace && lane == 0) sw.ts[4] = gtimer();
    seg_post(sw, L, cap, lane, (int)k, off, ex_k, light, deg, T.state(), (uint64_t)(D0 + ex_d), pid, T, A32, C32,
             indices, out_ids, out_pidx, bitmap);
    Wtot_out = Wtot;
}

// WPB warps per CTA, MINB CTAs per SM: (8, 4) = 32 resident warps per SM
// (64 registers); (6, 6) = 36 (56 registers), enough for the largest hop's
// runs to start in one wave (153.6K parents / 32 = 4800 runs vs 4736 / 5328).
// split_min > 0: a run whose light draws reach split_min hands the parents
// past its walk's midpoint to a queue (their offsets in deg_prefix /
// k_prefix); warps that find no run left take them, so the longest runs no
// longer set the kernel's tail alone.
template <int WPB, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB)
sample_seg_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                  const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                  int32_t fanout, const uint64_t* __restrict__ table, int64_t* __restrict__ draw_base,
                  ScanState ss, int64_t* __restrict__ deg_prefix, int64_t* __restrict__ k_prefix,
                  int32_t* __restrict__ heavy, int64_t* __restrict__ heavy_count,
                  int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx, int64_t* __restrict__ num_out,
                  uint32_t* __restrict__ bitmap, int32_t run, int64_t heavy_deg, float ma, float mb, int cap,
                  int32_t split_min, int32_t* __restrict__ split_ctr, int32_t* __restrict__ split_ready,
                  int64_t* __restrict__ split_ent) {
    __shared__ SegWarp s_seg[WPB];
    SegWarp& sw = s_seg[warp_id()];
    const int64_t n = *num_parents_dev;
    const int64_t nruns = n > 0 ? ceil_div(n, run) : 1;
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned FULL = 0xffffffffu;
    const PcgTable T{table};
    const U128 A32 = T.A(5), C32 = T.C(5);
    const int64_t D0 = draw_base[0];
    unsigned long long* trace = g_seg_trace;
    while (true) {
        int64_t r = 0;
        if (lane == 0) r = (int64_t)atomicAdd(ss.ticket, 1u);
        r = __shfl_sync(FULL, r, 0);
        if (r >= nruns) break;
        if (trace && lane == 0) sw.ts[0] = gtimer();
        const int64_t q = r * run + lane;
        const bool valid = lane < run && q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        const int64_t incl_d = warp_incl_scan(deg);
        const int64_t incl_k = warp_incl_scan(k);
        const int64_t agg_d = __shfl_sync(FULL, incl_d, 31);
        const int64_t agg_k = __shfl_sync(FULL, incl_k, 31);
        if (trace && lane == 0) sw.ts[1] = gtimer_after(agg_k);
        if (lane == 0) {
            const uint64_t f = r == 0 ? kFlagInc : kFlagAgg;
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(f | ((uint64_t)agg_d & kValMask)));
            atomicExch((unsigned long long*)(ss.status + ss.max_tiles + r),
                       (unsigned long long)(f | ((uint64_t)agg_k & kValMask)));
        }
        const int64_t pre_d = warp_lookback1(ss.status, r, agg_d);
        const int64_t pre_k = warp_lookback1(ss.status + ss.max_tiles, r, agg_k);
        if (trace && lane == 0) sw.ts[2] = gtimer_after(pre_d + pre_k);
        const int64_t ex_d = pre_d + incl_d - deg;
        const int64_t ex_k = pre_k + incl_k - k;
        const bool hv = valid && (k > 32 || deg > heavy_deg);
        const unsigned hm = __ballot_sync(FULL, hv);
        if (hm) {
            int64_t slot = 0;
            if (lane == 0) slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, (unsigned long long)__popc(hm));
            slot = __shfl_sync(FULL, slot, 0);
            if (hv) {
                heavy[slot + __popc(hm & lt)] = (int32_t)q;
                deg_prefix[q] = ex_d;
                k_prefix[q] = ex_k;
            }
        }
        if (r == nruns - 1 && lane == 31) {
            draw_base[1] = D0 + pre_d + incl_d;
            *num_out = pre_k + incl_k;
        }
        int jend = 32;
        if (split_min > 0) {
            const bool light = valid && !hv && deg > 0;
            const int32_t incl_l = warp_incl_scan(light ? (int32_t)deg : 0);
            const int32_t Wt = __shfl_sync(FULL, incl_l, 31);
            if (Wt >= split_min) {
                // part A: parents up to the one crossing the walk's midpoint; part B: the rest
                const unsigned cross = __ballot_sync(FULL, valid && 2 * incl_l >= Wt);
                const int j1 = cross ? __ffs(cross) : 32;
                const int cnt = (int)(n - r * run < run ? n - r * run : run);
                const int32_t before = j1 > 0 && j1 < 32 ? __shfl_sync(FULL, incl_l, j1 - 1) : Wt;
                if (j1 < cnt && Wt - before > 0) {
                    if (valid && lane >= j1) {
                        deg_prefix[q] = ex_d;
                        k_prefix[q] = ex_k;
                    }
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) {
                        const int slot = atomicAdd(split_ctr + 0, 1);
                        split_ent[slot] = (r << 8) | j1;
                        __threadfence();
                        atomicExch(split_ready + slot, 1);
                    }
                    jend = j1;
                }
            }
            if (lane == 0) {
                __threadfence();
                atomicAdd(split_ctr + 2, 1);
            }
        }
        int32_t Wtot = 0;
        seg_part(sw, valid && lane < jend, off, deg, k, ex_d, ex_k, hv, (int32_t)q, D0, T, A32, C32, lane, lt, cap,
                 ma, mb, indices, out_ids, out_pidx, bitmap, trace != nullptr, Wtot);
        if (trace && lane == 0) seg_trace_record(trace, n, r, Wtot, sw.ts);
    }
    if (split_min <= 0) return;
    // no run left: take split-off parts until every run has decided and the queue is drained
    while (true) {
        int64_t idx = 0;
        if (lane == 0) {
            idx = atomicAdd(split_ctr + 1, 1);
            if (idx >= nruns) {
                idx = -1;   // never valid: at most one part per run
            } else {
                unsigned ns = 64;
                while (!ld_volatile(split_ready + idx)) {
                    if (ld_volatile(split_ctr + 2) >= nruns && ld_volatile(split_ctr + 0) <= idx) {
                        idx = -1;
                        break;
                    }
                    __nanosleep(ns);
                    ns = ns < 1024 ? 2 * ns : ns;
                }
            }
        }
        idx = __shfl_sync(FULL, idx, 0);
        if (idx < 0) break;
        __threadfence();
        const int64_t e = ld_volatile(split_ent + idx);
        const int64_t r = e >> 8;
        const int j1 = (int)(e & 255);
        const int64_t q = r * run + j1 + lane;
        const bool valid = j1 + lane < run && q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        const int64_t ex_d = valid ? ld_volatile(deg_prefix + q) : 0;
        const int64_t ex_k = valid ? ld_volatile(k_prefix + q) : 0;
        const bool hv = valid && (k > 32 || deg > heavy_deg);
        int32_t Wtot = 0;
        seg_part(sw, valid, off, deg, k, ex_d, ex_k, hv, (int32_t)q, D0, T, A32, C32, lane, lt, cap, ma, mb, indices,
                 out_ids, out_pidx, bitmap, false, Wtot);
    }
}

// ---------------------------------------------------------------- prep + slice walk (default)
// Two launches per hop instead of the look-back inside the walk:
//   sample_prep_kernel  one pass over the hop's parents (1024 per CTA tile,
//       decoupled look-back over tiles, the four prefixes resolved by four
//       warps at once): deg/k/light-draw/light-count prefixes; the light
//       parents compacted in order with everything the walk needs (parent
//       index, light-draw start, heavy-draw gap, col offset, output offset,
//       deg|k, threshold); heavy parents listed for sample_heavy_kernel; the
//       slice map sf[s] = first light parent starting at or after light draw
//       s*S; the hop's base PCG64 state; the chained draw base and output
//       count. No per-run look-back is left on the walk's critical path.
//   sample_slice_kernel persistent warps claim slices of ~S light draws
//       (whole parents, atomic ticket), so every warp does about the same
//       number of draws and the tail is one slice, not one 32-parent run;
//       each group of <= 32 parents of a slice is walked with seg_walk (state
//       jumped from the hop's base, <= 7 affine maps) and finished by seg_post.
constexpr int kPrepThreads = 1024;
constexpr int kPrepWarps = kPrepThreads / 32;
constexpr int kPrepPPT = 2;                         // parents per thread
constexpr int kPrepTile = kPrepThreads * kPrepPPT;  // parents per CTA tile
constexpr int kSliceMin = 256;            // smallest slice: bounds the slice map at 8 entries per parent

struct HopMeta {
    uint64_t s0_hi, s0_lo;   // state after D0 steps (the hop's base)
    int64_t nlight;          // light parents
    int64_t ltot;            // light draws
    int64_t nslices;         // slices = ltot / S + 1
    unsigned ticket;         // slice / group claims (zeroed with the prep scan state)
    unsigned ntiles;         // prep tiles of this hop
};

struct LightParents {
    int32_t* q;        // parent position in the hop's input
    int64_t* lp;       // first light draw (prefix over light parents)
    int64_t* gap;      // heavy parents' draws before it (full position = lp + gap)
    int64_t* off;      // col offset (indptr[p])
    int64_t* kpre;     // output offset
    int32_t* dk;       // deg | k << 16 (light: deg <= 2048, k <= 32)
    uint32_t* thr;     // candidate threshold, high word
    int32_t* sf;       // [nslices + 1] slice -> first light parent
    int32_t* perm;     // lane walk: light parents of each prep tile by descending degree
    int32_t* tbase;    // lane walk: [tile] first light index of the tile
    int32_t* tcount;   // lane walk: [tile] light parents in the tile
};

// Parents split four ways: zero-degree (no draws), heavy (deg > 2048 or
// k > 32: sample_heavy_kernel), lane (deg <= dlane: one lane each, the
// tile's lane parents ordered by descending degree) and wide (the rest:
// slices of ~S draws). dlane = 0: every light parent is wide.
constexpr int kPrepVals = 5;   // deg, k, wide draws, wide parents, lane parents

__global__ void __launch_bounds__(kPrepThreads, 1)
sample_prep_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ parents,
                   const int64_t* __restrict__ num_parents_dev, int32_t fanout, const uint64_t* __restrict__ table,
                   int64_t* __restrict__ draw_base, ScanState ss, int64_t* __restrict__ deg_prefix,
                   int64_t* __restrict__ k_prefix, int32_t* __restrict__ heavy, int64_t* __restrict__ heavy_count,
                   LightParents lpar, LightParents lpl, HopMeta* __restrict__ meta, int64_t* __restrict__ num_out,
                   int64_t heavy_deg, float ma, float mb, int32_t S, int32_t dlane) {
    using Sorter = cub::BlockRadixSort<uint16_t, kPrepThreads, kPrepPPT, int16_t>;
    __shared__ typename Sorter::TempStorage s_sort;
    __shared__ int64_t s_tile;
    __shared__ int64_t s_warp[kPrepVals][kPrepWarps];
    __shared__ int64_t s_pre[kPrepVals], s_tot[kPrepVals];
    const int64_t n = *num_parents_dev;
    const int64_t ntiles = n > 0 ? ceil_div(n, kPrepTile) : 1;
    const int64_t tile = claim_tile(ss, &s_tile);
    const int lane = lane_id(), wid = warp_id();
    if (tile >= ntiles) {
        // the first spare CTA (grid = max tiles + 1) computes the hop's base
        // state beside the scan: the <= 16 jump rows loaded at once by 16
        // lanes, then applied in order from registers via shuffles
        if (tile == ntiles && wid == 0) {
            const PcgTable T{table};
            const uint64_t D0 = (uint64_t)draw_base[0];
            const int dig = (int)((D0 >> (4 * (lane & 15))) & 15u);
            U128 A{0, 0}, C{0, 0};
            if (lane < 16 && dig) {
                const uint64_t* r = T.row(lane, dig);
                A = U128{__ldg(r + 0), __ldg(r + 1)};
                C = U128{__ldg(r + 2), __ldg(r + 3)};
            }
            U128 st = T.state();
            for (int i = 0; i < 16; ++i) {
                const int di = __shfl_sync(0xffffffffu, dig, i);
                const U128 Ai{__shfl_sync(0xffffffffu, A.hi, i), __shfl_sync(0xffffffffu, A.lo, i)};
                const U128 Ci{__shfl_sync(0xffffffffu, C.hi, i), __shfl_sync(0xffffffffu, C.lo, i)};
                if (di) st = affine(Ai, Ci, st);
            }
            if (lane == 0) {
                meta->s0_hi = st.hi;
                meta->s0_lo = st.lo;
            }
        }
        return;
    }
    // thread t holds parents 2t, 2t+1 of the tile
    int64_t qv[kPrepPPT], offv[kPrepPPT], degv[kPrepPPT], kv[kPrepPPT];
    int cls[kPrepPPT];   // 0 none, 1 heavy, 2 wide, 3 lane
    int64_t v[kPrepVals] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < kPrepPPT; ++e) {
        const int64_t q = tile * kPrepTile + kPrepPPT * threadIdx.x + e;
        const bool valid = q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        qv[e] = q;
        offv[e] = off;
        degv[e] = deg;
        kv[e] = k;
        cls[e] = !valid || deg == 0 ? 0 : (k > 32 || deg > heavy_deg) ? 1 : deg <= dlane ? 3 : 2;
        v[0] += deg;
        v[1] += k;
        v[2] += cls[e] == 2 ? deg : 0;
        v[3] += cls[e] == 2 ? 1 : 0;
        v[4] += cls[e] == 3 ? 1 : 0;
    }
    int64_t incl[kPrepVals];
#pragma unroll
    for (int c = 0; c < kPrepVals; ++c) {
        incl[c] = warp_incl_scan(v[c]);
        if (lane == 31) s_warp[c][wid] = incl[c];
    }
    __syncthreads();
    if (wid < kPrepVals) {   // warp c: exclusive prefix of the warp totals of value c, tile total
        const int64_t x = s_warp[wid][lane];
        const int64_t xi = warp_incl_scan(x);
        s_warp[wid][lane] = xi - x;
        if (lane == 31) s_tot[wid] = xi;
    }
    __syncthreads();
    if (threadIdx.x < kPrepVals) {
        const uint64_t w = (tile == 0 ? kFlagInc : kFlagAgg) | ((uint64_t)s_tot[threadIdx.x] & kValMask);
        atomicExch((unsigned long long*)&ss.status[threadIdx.x * ss.max_tiles + tile], (unsigned long long)w);
        if (tile == 0) s_pre[threadIdx.x] = 0;
    }
    __syncthreads();   // aggregates published before anyone reads
    if (tile > 0 && wid < kPrepVals) {   // the prefixes at once: every predecessor's aggregate, read directly
        const uint64_t* st = ss.status + wid * ss.max_tiles;
        int64_t acc = 0;
        for (int64_t j = lane; j < tile; j += 32) {
            uint64_t w;
            do { w = ld_status(st + j); } while ((w >> 62) == 0);
            acc += (int64_t)(w & kValMask);
        }
        acc = warp_sum_i64(acc);
        if (lane == 0) s_pre[wid] = acc;
    }
    __syncthreads();
    int64_t ex[kPrepVals];
#pragma unroll
    for (int c = 0; c < kPrepVals; ++c) ex[c] = s_warp[c][wid] + incl[c] - v[c];   // tile-relative
    if (dlane > 0) {   // the tile's lane parents by descending degree
        uint16_t key[kPrepPPT];
        int16_t val[kPrepPPT];
        int64_t r = ex[4];
#pragma unroll
        for (int e = 0; e < kPrepPPT; ++e) {
            key[e] = cls[e] == 3 ? (uint16_t)(kNarrowMaxDeg - degv[e]) : (uint16_t)4095;
            val[e] = (int16_t)r;
            r += cls[e] == 3 ? 1 : 0;
        }
        Sorter(s_sort).Sort(key, val, 0, 12);
        const int64_t lb = s_pre[4], lc = s_tot[4];
#pragma unroll
        for (int e = 0; e < kPrepPPT; ++e) {
            const int64_t pos = (int64_t)kPrepPPT * threadIdx.x + e;
            if (pos < lc) lpl.perm[lb + pos] = (int32_t)(lb + val[e]);
        }
        if (threadIdx.x == 0) {
            lpl.tbase[tile] = (int32_t)lb;
            lpl.tcount[tile] = (int32_t)lc;
        }
    }
    int64_t dpre = s_pre[0] + ex[0], kpre = s_pre[1] + ex[1], wpre = s_pre[2] + ex[2];
    int64_t wi = s_pre[3] + ex[3], ni = s_pre[4] + ex[4];
#pragma unroll
    for (int e = 0; e < kPrepPPT; ++e) {
        const int64_t q = qv[e], deg = degv[e], k = kv[e];
        const bool hv = cls[e] == 1;
        const unsigned hm = __ballot_sync(0xffffffffu, hv);
        if (hm) {
            int64_t slot = 0;
            if (lane == 0) slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, (unsigned long long)__popc(hm));
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (hv) {
                heavy[slot + __popc(hm & ((1u << lane) - 1u))] = (int32_t)q;
                deg_prefix[q] = dpre;
                k_prefix[q] = kpre;
            }
        }
        if (cls[e] >= 2) {
            const bool wide = cls[e] == 2;
            LightParents& L = wide ? lpar : lpl;
            const int64_t i = wide ? wi : ni;
            L.q[i] = (int32_t)q;
            L.lp[i] = wide ? wpre : dpre;
            L.gap[i] = wide ? dpre - wpre : 0;
            L.off[i] = offv[e];
            L.kpre[i] = kpre;
            L.dk[i] = (int32_t)(deg | (k << 16));
            L.thr[i] = thr_hi(cand_threshold(k, deg, ma, mb));
            // slices whose start s*S lies in (wpre, wpre + deg] begin at the next wide parent
            if (wide)
                for (int64_t sl = wpre / S + 1; sl * S <= wpre + deg; ++sl) lpar.sf[sl] = (int32_t)(wi + 1);
        }
        dpre += deg;
        kpre += k;
        wpre += cls[e] == 2 ? deg : 0;
        wi += cls[e] == 2 ? 1 : 0;
        ni += cls[e] == 3 ? 1 : 0;
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const int64_t D0 = draw_base[0];
        const int64_t ltot = s_pre[2] + s_tot[2], nl = s_pre[3] + s_tot[3];
        const int64_t ns = ltot / S + 1;
        draw_base[1] = D0 + s_pre[0] + s_tot[0];
        *num_out = s_pre[1] + s_tot[1];
        meta->nlight = nl;
        meta->ltot = ltot;
        meta->nslices = ns;
        meta->ntiles = (unsigned)ntiles;
        lpar.sf[0] = 0;
        lpar.sf[ns] = (int32_t)nl;
    }
}

// One slice of the wide list: groups of <= `group` parents walked with
// seg_walk (state jumped from the hop's base) and finished by seg_post.
// Per-group values that live across the walk are re-read after it (light
// list / hop meta, L1/L2 hits) instead of being held in registers.
__device__ __forceinline__ void slice_one(SegWarp& sw, int i0, int i1, const LightParents& lpar,
                                          const HopMeta* meta, const PcgTable T, U128 A32, U128 C32,
                                          const int32_t* __restrict__ indices, int32_t* __restrict__ out_ids,
                                          int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap, int group,
                                          int cap, int lane, unsigned lt) {
    const unsigned FULL = 0xffffffffu;
    for (int ib = i0; ib < i1; ib += group) {
        const int ie = ib + group < i1 ? ib + group : i1;
        int L, Wtot;
        {
            const int i = ib + lane;
            const bool valid = lane < ie - ib;
            const int64_t lp = valid ? lpar.lp[i] : 0;
            const int64_t gap = valid ? lpar.gap[i] : 0;
            const int deg = valid ? (lpar.dk[i] & 0xffff) : 0;
            const int64_t LB = __shfl_sync(FULL, lp, 0);
            const int64_t LE = ie < meta->nlight ? lpar.lp[ie] : meta->ltot;   // same address on every lane
            Wtot = (int32_t)(LE - LB);
            sw.wst[lane] = valid ? (int32_t)(lp - LB) : Wtot;
            sw.wend[lane] = valid ? (int32_t)(lp - LB) + deg : Wtot;
            const int64_t G0 = __shfl_sync(FULL, gap, 0);   // gaps relative to the group's first parent
            sw.gap[lane] = valid ? gap - G0 : 0;
            sw.thr[lane] = valid ? lpar.thr[i] : 0u;
            if (lane == 0) {
                sw.wend[32] = 0x7fffffff;
                sw.thr[32] = 0;
                sw.gap[32] = 0;
                sw.wst[32] = 0;
            }
            const bool gaps = G0 != __shfl_sync(FULL, gap, ie - ib - 1);
            const U128 s0{meta->s0_hi, meta->s0_lo};
            __syncwarp();
            L = gaps ? seg_walk<true>(sw, T, A32, C32, s0, LB + G0, Wtot, lane, lt, cap)
                     : seg_walk<false>(sw, T, A32, C32, s0, LB + G0, Wtot, lane, lt, cap);
        }
        __syncwarp();
        const int i = ib + lane;
        const bool valid = lane < ie - ib;
        const int dk = valid ? lpar.dk[i] : 0;
        const int64_t dpos = valid ? lpar.lp[i] + lpar.gap[i] : 0;
        const int64_t off = valid ? lpar.off[i] : 0;
        const int64_t kpre = valid ? lpar.kpre[i] : 0;
        const int32_t q = valid ? lpar.q[i] : 0;
        const U128 s0{meta->s0_hi, meta->s0_lo};
        seg_post(sw, L, cap, lane, dk >> 16, off, kpre, valid, dk & 0xffff, s0, (uint64_t)dpos, q, T, A32, C32,
                 indices, out_ids, out_pidx, bitmap);
    }
}

// ---------------------------------------------------------------- lane walk
// One lane per low-degree parent (deg <= dlane): the lane replays its
// parent's own draws with the 1-step map (no cross-lane hand-off), keeps
// the draws below the parent's threshold in its own shared-memory column
// (high word + position) and selects the k smallest by an in-place
// selection sort over the column: no ballot, no cross-lane compaction, no
// ranking against other lanes' candidates (47 SASS instructions per draw
// against ~69 in the segmented walk). sample_prep_kernel orders each tile's
// lane parents by descending degree, so a warp's lanes walk about as many
// draws each, and dlane bounds the serial chain of one lane. Candidate-set
// exactness as in the segmented walk (out < thh * 2^32 is a threshold
// set). Parents with fewer than k candidates, a full column, or two
// candidates with equal high words (their order needs the low word) take
// the exact CTA kernel (sample_heavy_kernel) through the heavy list.
constexpr int kLaneCap = 32;

struct LaneCols {
    uint32_t hi[kLaneCap][32];
    uint16_t t[kLaneCap][32];
};

__device__ __forceinline__ void lane_one(LaneCols& cl, int g, const LightParents& lpl, const HopMeta* meta,
                                         int ntiles, const PcgTable T, U128 A1, U128 C1,
                                         const int32_t* __restrict__ indices, int64_t* __restrict__ deg_prefix,
                                         int64_t* __restrict__ k_prefix, int32_t* __restrict__ heavy,
                                         int64_t* __restrict__ heavy_count, int32_t* __restrict__ out_ids,
                                         int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap, int capl,
                                         int lane) {
    const int tile = g % ntiles, grp = g / ntiles;
    const int lc = lpl.tcount[tile];
    if (32 * grp >= lc) return;
    const int lb = lpl.tbase[tile];
    const bool valid = 32 * grp + lane < lc;
    const int li = valid ? lpl.perm[lb + 32 * grp + lane] : 0;
    const int dk = valid ? lpl.dk[li] : 0;
    const int deg = dk & 0xffff, k = dk >> 16;
    const uint32_t th = valid ? lpl.thr[li] : 0u;
    const int64_t dpos = valid ? lpl.lp[li] : 0;   // the lane list holds the full draw offset
    U128 s = T.adv(U128{meta->s0_hi, meta->s0_lo}, (uint64_t)dpos + 1);
    int c = 0;
    for (int t = 0; t < deg; ++t) {
        const uint32_t hh = (uint32_t)(s.hi >> 32);
        const uint32_t xl = (uint32_t)s.lo ^ (uint32_t)s.hi, xh = (uint32_t)(s.lo >> 32) ^ hh;
        const uint32_t rot = hh >> 26;
        const uint32_t a = (rot & 32u) ? xl : xh, b = (rot & 32u) ? xh : xl;
        const uint32_t out_hi = __funnelshift_r(a, b, rot);
        if (out_hi < th) {
            if (c < capl) {
                cl.hi[c][lane] = out_hi;
                cl.t[c][lane] = (uint16_t)t;
            }
            ++c;
        }
        s = affine_cc(A1, C1, s);
    }
    // selection sort of the column's k smallest into its first k slots
    bool fb = valid && (c < k || c > capl);
    const int kk = fb ? 0 : k;
    for (int r = 0; r < kk; ++r) {
        uint32_t best = cl.hi[r][lane];
        int bi = r;
        for (int x = r + 1; x < c; ++x) {
            const uint32_t h = cl.hi[x][lane];
            fb |= h == best;
            if (h < best) {
                best = h;
                bi = x;
            }
        }
        const uint16_t tb = cl.t[bi][lane];
        cl.hi[bi][lane] = cl.hi[r][lane];
        cl.t[bi][lane] = cl.t[r][lane];
        cl.hi[r][lane] = best;
        cl.t[r][lane] = tb;
    }
    const int64_t off = valid ? lpl.off[li] : 0;
    const int64_t kpre = valid ? lpl.kpre[li] : 0;
    const int32_t q = valid ? lpl.q[li] : 0;
    if (fb) {   // exact CTA kernel (runs after this one)
        const int64_t slot = (int64_t)atomicAdd((unsigned long long*)heavy_count, 1ull);
        heavy[slot] = q;
        deg_prefix[q] = dpos;
        k_prefix[q] = kpre;
    }
    const int ko = fb ? 0 : kk;
    for (int r0 = 0; r0 < ko; r0 += 4) {   // four column reads in flight before their stores
        int32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (r0 + u < ko) v[u] = indices[off + cl.t[r0 + u][lane]];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (r0 + u < ko) {
                if (out_ids) out_ids[kpre + r0 + u] = v[u];
                if (out_pidx) out_pidx[kpre + r0 + u] = q;
                if (bitmap) mark_bit(bitmap, v[u]);
            }
        }
    }
    __syncwarp();
}

union WalkSmem {
    SegWarp seg;
    LaneCols lane;
};

// Persistent warps over one claim counter: the wide list's slices first
// (the long work starts early), then the lane groups, heaviest first
// (group j of every prep tile before group j + 1 of any).
template <int WPB, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB)
sample_walk_kernel(const int32_t* __restrict__ indices, const uint64_t* __restrict__ table, LightParents lpar,
                   LightParents lpl, HopMeta* __restrict__ meta, int64_t* __restrict__ deg_prefix,
                   int64_t* __restrict__ k_prefix, int32_t* __restrict__ heavy, int64_t* __restrict__ heavy_count,
                   int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap,
                   int group, int cap, int capl, int lanes_on) {
    __shared__ WalkSmem s_walk[WPB];
    WalkSmem& ws = s_walk[warp_id()];
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned FULL = 0xffffffffu;
    const PcgTable T{table};
    const int nslices = (int)meta->nslices;
    const int ntiles = (int)meta->ntiles;
    const int nclaims = nslices + (lanes_on ? ntiles * (kPrepTile / 32) : 0);
    while (true) {
        int g = 0;
        if (lane == 0) g = (int)atomicAdd(&meta->ticket, 1u);
        g = __shfl_sync(FULL, g, 0);
        if (g >= nclaims) break;
        if (g < nslices) {
            slice_one(ws.seg, lpar.sf[g], lpar.sf[g + 1], lpar, meta, T, T.A(5), T.C(5), indices, out_ids, out_pidx,
                      bitmap, group, cap, lane, lt);
        } else {
            lane_one(ws.lane, g - nslices, lpl, meta, ntiles, T, T.A(0), T.C(0), indices, deg_prefix, k_prefix,
                     heavy, heavy_count, out_ids, out_pidx, bitmap, capl, lane);
        }
    }
}

// ---------------------------------------------------------------- heavy parents
constexpr int kHeavyThreads = 256;
constexpr int kHeavyWarps = kHeavyThreads / 32;

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

__global__ void __launch_bounds__(kHeavyThreads)
sample_heavy_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                    const int32_t* __restrict__ parents, const int32_t* __restrict__ heavy,
                    const int64_t* __restrict__ heavy_count, int32_t fanout, int kcap,
                    const uint64_t* __restrict__ table, const int64_t* __restrict__ draw_base,
                    const int64_t* __restrict__ deg_prefix, const int64_t* __restrict__ k_prefix,
                    int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx, uint32_t* __restrict__ bitmap) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* sm = reinterpret_cast<uint64_t*>(smem);
    uint32_t* st = reinterpret_cast<uint32_t*>(smem + sizeof(uint64_t) * 2 * kcap);
    const int64_t nh = *heavy_count;
    const PcgTable T{table};
    const int64_t D0 = draw_base[0];
    const int lane = lane_id(), wid = warp_id();
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t q = heavy[h];
        const int32_t p = parents[q];
        const int64_t off = indptr[p];
        const int64_t deg = indptr[p + 1] - off;
        const int k = (int)(deg < fanout ? deg : fanout);
        const int64_t dq = D0 + deg_prefix[q];
        const int64_t o = k_prefix[q];
        if (k <= 32) {
            // warp w folds chunks w, w+8, ... into its own top-k
            const U128 A256 = T.A(8), C256 = T.C(8);
            WideKey best = key_inf<WideKey>(), kth = best;
            const int64_t nc = (deg + 31) >> 5;
            U128 s{0, 0};
            for (int64_t c = wid; c < nc; c += kHeavyWarps) {
                s = (c == wid) ? T.at((uint64_t)(dq + (c << 5) + lane + 1)) : affine(A256, C256, s);
                const int64_t t = (c << 5) + lane;
                WideKey cand = key_inf<WideKey>();
                if (t < deg) cand = WideKey{draw_of_state(s), (uint32_t)t};
                fold_chunk(best, kth, cand, k);
            }
            uint32_t* st2 = reinterpret_cast<uint32_t*>(smem + sizeof(uint64_t) * kHeavyThreads);
            sm[wid * 32 + lane] = best.m;
            st2[wid * 32 + lane] = best.t;
            __syncthreads();
            if (wid == 0) {
                WideKey acc{sm[lane], st2[lane]};
                for (int w = 1; w < kHeavyWarps; ++w)
                    acc = merge_sorted(acc, WideKey{sm[w * 32 + lane], st2[w * 32 + lane]});
                if (lane < k) {
                    const int32_t v = indices[off + acc.t];
                    if (out_ids) out_ids[o + lane] = v;
                    if (out_pidx) out_pidx[o + lane] = (int32_t)q;
                    if (bitmap) mark_bit(bitmap, v);
                }
            }
            __syncthreads();
            continue;
        }
        // k > 32: chunked bitonic sort of (current top-kcap | next kcap draws)
        const U128 Ab = T.A(8), Cb = T.C(8);   // blockDim == 256 == 2^8
        for (int i = threadIdx.x; i < kcap; i += blockDim.x) {
            sm[i] = ~0ull;
            st[i] = ~0u;
        }
        for (int64_t base = 0; base < deg; base += kcap) {
            U128 s = T.at((uint64_t)(dq + base + threadIdx.x + 1));
            for (int i = threadIdx.x; i < kcap; i += blockDim.x) {
                if (i != (int)threadIdx.x) s = affine(Ab, Cb, s);
                int64_t t = base + i;
                sm[kcap + i] = t < deg ? draw_of_state(s) : ~0ull;
                st[kcap + i] = t < deg ? (uint32_t)t : ~0u;
            }
            __syncthreads();
            smem_bitonic_sort(sm, st, 2 * kcap);
        }
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            const int32_t v = indices[off + st[i]];
            if (out_ids) out_ids[o + i] = v;
            if (out_pidx) out_pidx[o + i] = (int32_t)q;
            if (bitmap) mark_bit(bitmap, v);
        }
        __syncthreads();
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

// Diagnostics only: route the segmented walk's per-run timeline into buf
// (device; buf[0] = record count, records of 8 u64 from buf + 8); NULL = off.
int bgl_debug_seg_trace(void* buf) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
    return cuda_status(cudaMemcpyToSymbol(g_seg_trace, &p, sizeof(p)), "bgl_debug_seg_trace");
}

size_t bgl_sample_hop_workspace(int64_t max_parents) {
    int64_t m = max_parents > 0 ? max_parents : 1;
    return hop_ws_bytes(m) + slice_ws_bytes(m);
}

int bgl_sample_hop(const int64_t* indptr, const int32_t* indices, const int32_t* parents,
                   const int64_t* num_parents_dev, int64_t max_parents, int32_t fanout,
                   const uint64_t* table, int64_t* draw_base, int32_t* out_ids,
                   int32_t* out_parent_idx, int64_t* num_out_dev, void* workspace, void* mark_bitmap,
                   int32_t max_ctas, void* stream) {
    BGL_CHECK_ARG(fanout >= 1, "fanouts must be positive");
    BGL_CHECK_ARG(fanout <= 4096, "fanout > 4096 unsupported (clamp it to the graph's max degree)");
    BGL_CHECK_ARG(max_parents >= 0, "bgl_sample_hop: max_parents < 0");
    BGL_CHECK_ARG(indptr && table && draw_base && num_parents_dev && num_out_dev && workspace,
                  "bgl_sample_hop: null pointer");
    cudaStream_t st = as_stream(stream);
    HopWorkspace w = carve_hop_ws(workspace, max_parents);
    uint32_t* bm = reinterpret_cast<uint32_t*>(mark_bitmap);
    // fused scan + sample over runs of `run` parents: short runs when the hop is
    // small (enough warps for hop 1), up to kRun (one per lane) when it is large
    // ~32 runs per SM (one per resident warp): longer runs amortise the
    // look-back and the run's PCG64 jump (C2 HBM sweep with sample_seg: 96 ->
    // 4405, 64 -> 4586, 48 -> 4857, 32 -> 4975, 16 -> 4958, 8 -> 4837 b/s)
    static const int64_t runs_per_sm = [] {
        const char* e = getenv("BGL_RUNS_PER_SM");
        return (int64_t)(e ? atoi(e) : 32);
    }();
    const int64_t want_runs = (int64_t)kNumSMs * runs_per_sm;
    int64_t run = ceil_div(std::max<int64_t>(max_parents, 1), want_runs);
    run = std::min<int64_t>(std::max<int64_t>(run, 1), kRun);
    // fanout <= 32: segmented threshold walk (default), BGL_SAMPLER=cand the
    // per-parent threshold kernel, =fused the running top-k kernel (A/B)
    static const int mode_env = [] {
        const char* e = getenv("BGL_SAMPLER");
        if (e && std::string(e) == "fused") return 0;
        if (e && std::string(e) == "cand") return 1;
        if (e && std::string(e) == "slice") return 3;
        if (e && std::string(e) == "hybrid") return 4;
        return 2;
    }();
    const int mode = fanout <= 32 ? mode_env : 0;
    if (mode >= 3) run = kRun;                 // a slice's parents are walked 32 at a time
    else   // scan state + counters are contiguous: one memset (the split-ready flags only when splitting)
        BGL_TRY(cuda_status(cudaMemsetAsync(w.scan, 0, align256(scan_state_bytes(2, w.max_tiles)) + 256, st),
                            "hop workspace reset"));
    // candidate threshold keeps ~k + 2 sqrt(k) + 1 draws per parent (a sweep of
    // the margin at C2: (1, 1) 4027, (1.5, 1) 4079, (2, 1) 4102, (2.5, 2) 4046,
    // (3, 3) 4032 b/s with HBM features -- a few % either way; the segmented
    // walk: (1, 0.5) 4578, (1, 1) 4702, (1.5, 1) 4932, (2, 1) 4987, (2.5, 1)
    // 4975, (3, 2) 4961)
    const float mar[2] = {2.0f, 1.0f};
    // candidate list length per warp (BGL_SEG_CAP < 512: tests force overflow)
    static const int seg_cap = [] {
        const char* e = getenv("BGL_SEG_CAP");
        const int c = e ? atoi(e) : kSegCap;
        return c < 1 ? 1 : (c > kSegCap ? kSegCap : c);
    }();
    if (mode >= 2 && seg_cap == kSegCap) {   // a run's expected candidates stay well inside the list
        const double mu = fanout + mar[0] * std::sqrt((double)fanout) + mar[1];
        const int64_t rmax = std::max<int64_t>(1, (int64_t)(kSegCap / (1.5 * mu)));
        run = std::min<int64_t>(run, rmax);
    }
    const int64_t runs = std::max<int64_t>(1, ceil_div(max_parents, run));
    // parents above this degree go to the 8-warp CTA kernel (lower thresholds
    // for the small hops were measured slower: the CTA kernel runs after it)
    const int64_t heavy_deg = kNarrowMaxDeg;
    ScanState ss = make_scan_state(w.scan, 2, w.max_tiles);
    // BGL_SEG_OCC=8x4 (default) | 6x6: warps per CTA x CTAs per SM of the segmented walk
    static const int seg_wpb = [] {
        const char* e = getenv("BGL_SEG_OCC");
        return (e && std::string(e) == "6x6") ? 6 : 8;
    }();
    const int wpb = mode == 2 ? seg_wpb : kWarpsPerBlock;
    unsigned blocks = (unsigned)ceil_div(runs, wpb);
    const unsigned cap_blocks = (unsigned)kNumSMs * 8;
    if (blocks > cap_blocks) blocks = cap_blocks;               // runs are claimed dynamically
    if (max_ctas > 0 && blocks > (unsigned)max_ctas) blocks = (unsigned)max_ctas;
    if (mode >= 3) {
        // wide parents: slices of ~S light draws, ~1.5 per resident warp at
        // the expected hop size (max_parents x BGL_SLICE_DEG, default 128
        // draws per parent; BGL_SLICE_DRAWS overrides), never below kSliceMin;
        // lane parents (mode 4, k <= 10): deg <= BGL_LANE_DEG (default 64)
        static const int64_t slice_env = [] {
            const char* e = getenv("BGL_SLICE_DRAWS");
            return (int64_t)(e ? atoll(e) : 0);
        }();
        static const int64_t deg_hint = [] {
            const char* e = getenv("BGL_SLICE_DEG");
            return (int64_t)(e ? atoll(e) : 128);
        }();
        static const int lane_deg = [] {
            const char* e = getenv("BGL_LANE_DEG");
            return e ? std::max(0, std::min(atoi(e), (int)kNarrowMaxDeg)) : 64;
        }();
        // column length per lane (BGL_LANE_CAP < kLaneCap: tests force full columns)
        static const int lane_cap = [] {
            const char* e = getenv("BGL_LANE_CAP");
            return e ? std::max(1, std::min(atoi(e), kLaneCap)) : kLaneCap;
        }();
        const int dlane = (mode == 4 && fanout <= 10) ? lane_deg : 0;
        int64_t S = slice_env;
        if (S <= 0) {   // ~1.5 slices per resident warp (32 per SM)
            const int64_t want = (int64_t)kNumSMs * 48;
            S = kSliceMin;
            while (S < 8192 && 2 * S * want <= max_parents * deg_hint) S *= 2;
        }
        S = std::max<int64_t>(S, kSliceMin);
        const int64_t m = std::max<int64_t>(max_parents, 1);
        char* base = reinterpret_cast<char*>(workspace) + hop_ws_bytes(m);
        const int64_t ptiles = prep_tiles(m);
        BGL_TRY(cuda_status(cudaMemsetAsync(base, 0, slice_reset_bytes(m), st), "walk workspace reset"));
        ScanState ps = make_scan_state(base, kPrepVals, ptiles);
        char* r = base + align256(scan_state_bytes(kPrepVals, ptiles));
        int64_t* hcount = reinterpret_cast<int64_t*>(r);
        HopMeta* meta = reinterpret_cast<HopMeta*>(r + 64);
        char* a = base + slice_reset_bytes(m);
        auto carve_list = [&](LightParents& L) {
            L.q = reinterpret_cast<int32_t*>(a); a += align256(m * 4);
            L.dk = reinterpret_cast<int32_t*>(a); a += align256(m * 4);
            L.thr = reinterpret_cast<uint32_t*>(a); a += align256(m * 4);
            L.lp = reinterpret_cast<int64_t*>(a); a += align256(m * 8);
            L.gap = reinterpret_cast<int64_t*>(a); a += align256(m * 8);
            L.off = reinterpret_cast<int64_t*>(a); a += align256(m * 8);
            L.kpre = reinterpret_cast<int64_t*>(a); a += align256(m * 8);
            L.sf = L.perm = L.tbase = L.tcount = nullptr;
        };
        LightParents wl, ll;
        carve_list(wl);
        wl.sf = reinterpret_cast<int32_t*>(a); a += align256((8 * m + 2) * 4);
        carve_list(ll);
        ll.perm = reinterpret_cast<int32_t*>(a); a += align256(m * 4);
        ll.tbase = reinterpret_cast<int32_t*>(a); a += align256(ptiles * 4);
        ll.tcount = reinterpret_cast<int32_t*>(a);
        sample_prep_kernel<<<(unsigned)ptiles + 1, kPrepThreads, 0, st>>>(
            indptr, parents, num_parents_dev, fanout, table, draw_base, ps, w.deg_prefix, w.k_prefix, w.heavy, hcount,
            wl, ll, meta, num_out_dev, heavy_deg, mar[0], mar[1], (int32_t)S, dlane);
        BGL_TRY(launch_status("sample_prep_kernel"));
        unsigned sblocks = (unsigned)kNumSMs * 4;
        if (max_ctas > 0 && sblocks > (unsigned)max_ctas) sblocks = (unsigned)max_ctas;
        sample_walk_kernel<8, 4><<<sblocks, 8 * 32, 0, st>>>(indices, table, wl, ll, meta, w.deg_prefix, w.k_prefix,
                                                             w.heavy, hcount, out_ids, out_parent_idx, bm,
                                                             (int32_t)run, seg_cap, lane_cap, dlane > 0 ? 1 : 0);
        BGL_TRY(launch_status("sample_walk_kernel"));
        w.heavy_count = hcount;
    } else if (mode == 2) {
        // BGL_SEG_SPLIT=D: runs of >= 16 parents whose light draws reach D hand
        // their second half to warps that find no run left (C2 hop 3 warm,
        // graph replays: 112.9 -> 105.9 us at D = 3072; 2048: 106.2, 4096:
        // 109.2, 6144: 114.6). Off by default: the pipelined C2 HBM line is
        // unchanged (5225 vs 5215) and hop 3 under ncu's serialised, cold-cache
        // replay takes 63.5 M instead of 56 M instructions and 105-113 us.
        static const int32_t split_env = [] {
            const char* e = getenv("BGL_SEG_SPLIT");
            return (int32_t)(e ? atoi(e) : 0);
        }();
        const int32_t split_min = run >= 16 ? split_env : 0;
        if (split_min > 0)
            BGL_TRY(cuda_status(cudaMemsetAsync(w.split_ready, 0, (size_t)w.max_tiles * 4, st), "split flags reset"));
        auto kern = wpb == 6 ? sample_seg_kernel<6, 6> : sample_seg_kernel<8, 4>;
        kern<<<blocks, wpb * 32, 0, st>>>(
            indptr, indices, parents, num_parents_dev, fanout, table, draw_base, ss, w.deg_prefix, w.k_prefix,
            w.heavy, w.heavy_count, out_ids, out_parent_idx, num_out_dev, bm, (int32_t)run, heavy_deg, mar[0], mar[1],
            seg_cap, split_min, w.split_ctr, w.split_ready, w.split_ent);
        BGL_TRY(launch_status("sample_seg_kernel"));
    } else if (mode == 1) {
        sample_cand_kernel<<<blocks, kWarpsPerBlock * 32, 0, st>>>(
            indptr, indices, parents, num_parents_dev, fanout, table, draw_base, ss, w.deg_prefix, w.k_prefix,
            w.heavy, w.heavy_count, out_ids, out_parent_idx, num_out_dev, bm, (int32_t)run, heavy_deg, mar[0], mar[1]);
        BGL_TRY(launch_status("sample_cand_kernel"));
    } else {
        sample_fused_kernel<<<blocks, kWarpsPerBlock * 32, 0, st>>>(
            indptr, indices, parents, num_parents_dev, fanout, table, draw_base, ss, w.deg_prefix, w.k_prefix,
            w.heavy, w.heavy_count, out_ids, out_parent_idx, num_out_dev, bm, (int32_t)run, heavy_deg);
        BGL_TRY(launch_status("sample_fused_kernel"));
    }
    if (max_parents == 0) return BGL_OK;
    int kcap = 32;
    if (fanout > 32) {
        kcap = 64;
        while (kcap < fanout) kcap <<= 1;
    }
    size_t smem = (size_t)2 * kcap * (sizeof(uint64_t) + sizeof(uint32_t));
    if (smem < (size_t)kHeavyWarps * 32 * 12) smem = (size_t)kHeavyWarps * 32 * 12;
    if (smem > 48 * 1024)
        BGL_TRY(cuda_status(cudaFuncSetAttribute(sample_heavy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem), "cudaFuncSetAttribute(sample_heavy)"));
    unsigned hblocks = (unsigned)kNumSMs * 4;
    if (max_ctas > 0 && hblocks > (unsigned)max_ctas) hblocks = (unsigned)max_ctas;
    sample_heavy_kernel<<<hblocks, kHeavyThreads, smem, st>>>(
        indptr, indices, parents, w.heavy, w.heavy_count, fanout, kcap, table, draw_base, w.deg_prefix,
        w.k_prefix, out_ids, out_parent_idx, bm);
    return launch_status("sample_heavy_kernel");
}

}  // extern "C"
