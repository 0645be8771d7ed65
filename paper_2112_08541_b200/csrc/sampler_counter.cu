// K1 (counter-RNG mode): one hop of uniform without-replacement neighbour
// sampling with a counter-based RNG -- the north_star's "warp-per-seed CSR
// uniform-fanout sampler with a counter-based RNG". NOT bit-exact with the
// reference's numpy stream (that is bgl_sample_hop's PCG64 replay); validated
// by neighbour-validity and fanout-distribution checks, and bit for bit
// against its own CPU restatement (oracle/counter_sampler.py).
//
// Per parent q (lane per parent, 32 parents per warp run): k = min(fanout,
// deg); deg <= k -> every neighbour in adjacency order; else Floyd's
// algorithm -- for j = deg-k .. deg-1: r = uniform[0, j]; r = j if r was
// already chosen; emit col[off + r] -- a uniform k-subset from k draws, not
// deg draws (the replay kernel must make deg draws to reproduce numpy).
// Draws: Philox4x32-10, key = hash of the batch's stream state (row 0 of the
// PCG64 table, i.e. of (seed, batch_seed)), counter = (q, hop, step / 4, 0);
// bounded draws by Lemire's multiply with rejection. Output offsets: warp
// scan of k + decoupled look-back over runs (no separate pass); every output
// is marked in the dedup bitmap.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "pcg64.cuh"
#include "scan.cuh"

namespace bgl {

__host__ __device__ __forceinline__ void philox_round(uint32_t* c, const uint32_t* k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(M0, c[0]), hi1 = __umulhi(M1, c[2]);
#else
    const uint32_t hi0 = (uint32_t)(((uint64_t)M0 * c[0]) >> 32), hi1 = (uint32_t)(((uint64_t)M1 * c[2]) >> 32);
#endif
    const uint32_t lo0 = M0 * c[0], lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
}

// Philox4x32-10 (Salmon et al., SC'11)
__host__ __device__ __forceinline__ void philox4x32(uint32_t* c, uint32_t k0, uint32_t k1) {
    uint32_t k[2] = {k0, k1};
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(c, k);
        if (r < 9) {
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
    }
}

struct PhiloxStream {
    uint32_t k0, k1, q, hop, blk, used;
    uint32_t buf[4];
    __device__ __forceinline__ uint32_t next() {
        if (used == 4) {
            buf[0] = q;
            buf[1] = hop;
            buf[2] = blk++;
            buf[3] = 0;
            philox4x32(buf, k0, k1);
            used = 0;
        }
        return buf[used++];
    }
    // uniform in [0, bound) (Lemire, rejection)
    __device__ __forceinline__ uint32_t bounded(uint32_t bound) {
        uint64_t m = (uint64_t)next() * bound;
        uint32_t lo = (uint32_t)m;
        if (lo < bound) {
            const uint32_t thr = (0u - bound) % bound;
            while (lo < thr) {
                m = (uint64_t)next() * bound;
                lo = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

constexpr int kCWarps = 8;
constexpr int kCMaxK = 32;

__global__ void __launch_bounds__(kCWarps * 32)
sample_counter_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                      const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                      int32_t fanout, const uint64_t* __restrict__ table, int32_t hop, ScanState ss,
                      int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx,
                      int64_t* __restrict__ num_out, uint32_t* __restrict__ bitmap) {
    __shared__ int32_t s_chosen[kCWarps][kCMaxK][32];
    int32_t (*chosen)[32] = s_chosen[warp_id()];
    const int64_t n = *num_parents_dev;
    const int64_t nruns = n > 0 ? ceil_div(n, 32) : 1;
    const int lane = lane_id();
    // key of the batch's stream: its PCG64 (state, inc) from SeedSequence
    const uint64_t a = __ldg(table + 0) ^ __ldg(table + 2), b = __ldg(table + 1) ^ __ldg(table + 3);
    const uint32_t k0 = (uint32_t)(a ^ (a >> 32)) ^ (uint32_t)b, k1 = (uint32_t)(b >> 32) ^ (uint32_t)(a >> 17);
    while (true) {
        int64_t r = 0;
        if (lane == 0) r = (int64_t)atomicAdd(ss.ticket, 1u);
        r = __shfl_sync(0xffffffffu, r, 0);
        if (r >= nruns) break;
        const int64_t q = r * 32 + lane;
        const bool valid = q < n;
        const int32_t p = valid ? parents[q] : 0;
        const int64_t off = valid ? indptr[p] : 0;
        const int64_t deg = valid ? indptr[p + 1] - off : 0;
        const int64_t k = deg < fanout ? deg : fanout;
        const int64_t incl = warp_incl_scan(k);
        const int64_t agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) {
            const uint64_t f = r == 0 ? kFlagInc : kFlagAgg;
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(f | ((uint64_t)agg & kValMask)));
        }
        // look-back over runs for the exclusive output offset
        int64_t pre = 0;
        if (r > 0) {
            int64_t j = r - 1;
            while (true) {
                const int64_t idx = j - lane;
                uint64_t w = kFlagInc;
                if (idx >= 0) {
                    do { w = ld_status(ss.status + idx); } while ((w >> 62) == 0);
                }
                const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                const int stop = inc ? __ffs(inc) - 1 : 31;
                pre += warp_sum_i64(lane <= stop ? (int64_t)(w & kValMask) : 0);
                if (inc) break;
                j -= 32;
            }
        }
        if (lane == 0)
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(kFlagInc | ((uint64_t)(pre + agg) & kValMask)));
        if (r == nruns - 1 && lane == 31) *num_out = pre + incl;
        const int64_t o = pre + incl - k;
        if (!valid || k == 0) continue;
        if (deg <= k) {                               // every neighbour, adjacency order
#pragma unroll 4
            for (int64_t t = 0; t < k; ++t) {
                const int32_t v = indices[off + t];
                if (out_ids) out_ids[o + t] = v;
                if (out_pidx) out_pidx[o + t] = (int32_t)q;
                if (bitmap) atomicOr(bitmap + (v >> 5), 1u << (v & 31));   // fire-and-forget (RED)
            }
            continue;
        }
        // phase 1: Floyd's selection (RNG + smem membership only, no global memory)
        PhiloxStream rs{k0, k1, (uint32_t)q, (uint32_t)hop, 0u, 4u, {0, 0, 0, 0}};
        for (int i = 0; i < (int)k; ++i) {            // j = deg - k + i
            const uint32_t j = (uint32_t)(deg - k + i);
            uint32_t x = rs.bounded(j + 1);
            for (int e = 0; e < i; ++e)
                if ((uint32_t)chosen[e][lane] == x) {
                    x = j;
                    break;
                }
            chosen[i][lane] = (int32_t)x;
        }
        // phase 2: k independent gathers + stores
#pragma unroll 4
        for (int i = 0; i < (int)k; ++i) {
            const int32_t v = indices[off + chosen[i][lane]];
            if (out_ids) out_ids[o + i] = v;
            if (out_pidx) out_pidx[o + i] = (int32_t)q;
            if (bitmap) atomicOr(bitmap + (v >> 5), 1u << (v & 31));
        }
    }
}

// Sub-warp per seed: G lanes (G = next power of two >= fanout) sample one
// parent, R = 32 / G parents per warp run. m = min(k, deg - k) slots draw in
// parallel, one Philox4x32-10 call per lane and round (counter (q, hop |
// round << 8, slot, 0)); a slot keeps its draw unless a slot that is already
// kept holds the same value or a lower slot drew it in the same round
// (__match_any_sync). The rule only compares values, so the kept m-set is
// invariant under relabelling the neighbours: a uniform m-subset. k <= deg/2:
// the m = k kept indices are the sample (slot order); k > deg/2: they are the
// deg - k EXCLUDED indices and the rest is emitted in adjacency order.
template <int G>
__global__ void __launch_bounds__(kCWarps * 32)
sample_counter_group_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* __restrict__ parents, const int64_t* __restrict__ num_parents_dev,
                            int32_t fanout, const uint64_t* __restrict__ table, int32_t hop, ScanState ss,
                            int32_t* __restrict__ out_ids, int32_t* __restrict__ out_pidx,
                            int64_t* __restrict__ num_out, uint32_t* __restrict__ bitmap) {
    constexpr int R = 32 / G;
    const unsigned FULL = 0xffffffffu;
    const int64_t n = *num_parents_dev;
    const int64_t nruns = n > 0 ? ceil_div(n, R) : 1;
    const int lane = lane_id();
    const int g = lane / G, sub = lane % G;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (g * G));
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t a = __ldg(table + 0) ^ __ldg(table + 2), b = __ldg(table + 1) ^ __ldg(table + 3);
    const uint32_t k0 = (uint32_t)(a ^ (a >> 32)) ^ (uint32_t)b, k1 = (uint32_t)(b >> 32) ^ (uint32_t)(a >> 17);
    while (true) {
        int64_t r = 0;
        if (lane == 0) r = (int64_t)atomicAdd(ss.ticket, 1u);
        r = __shfl_sync(FULL, r, 0);
        if (r >= nruns) break;
        // prologue: lanes < R own the run's parents (degree, k, output offset)
        const int64_t qp = r * R + lane;
        const bool vp = lane < R && qp < n;
        const int32_t pp = vp ? parents[qp] : 0;
        const int64_t offp = vp ? indptr[pp] : 0;
        const int64_t degp = vp ? indptr[pp + 1] - offp : 0;
        const int64_t kp = degp < fanout ? degp : fanout;
        const int64_t incl = warp_incl_scan(kp);
        const int64_t agg = __shfl_sync(FULL, incl, 31);
        if (lane == 0) {
            const uint64_t f = r == 0 ? kFlagInc : kFlagAgg;
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(f | ((uint64_t)agg & kValMask)));
        }
        int64_t pre = 0;
        if (r > 0) {
            int64_t j = r - 1;
            while (true) {
                const int64_t idx = j - lane;
                uint64_t w = kFlagInc;
                if (idx >= 0) {
                    do { w = ld_status(ss.status + idx); } while ((w >> 62) == 0);
                }
                const unsigned inc = __ballot_sync(FULL, (w >> 62) == 2);
                const int stop = inc ? __ffs(inc) - 1 : 31;
                pre += warp_sum_i64(lane <= stop ? (int64_t)(w & kValMask) : 0);
                if (inc) break;
                j -= 32;
            }
        }
        if (lane == 0)
            atomicExch((unsigned long long*)(ss.status + r), (unsigned long long)(kFlagInc | ((uint64_t)(pre + agg) & kValMask)));
        if (r == nruns - 1 && lane == 31) *num_out = pre + incl;
        // group g takes parent g of the run
        const int64_t q = r * R + g;
        const bool valid = q < n;
        const int64_t deg = __shfl_sync(FULL, degp, g);
        const int64_t k = __shfl_sync(FULL, kp, g);
        const int64_t off = __shfl_sync(FULL, offp, g);
        const int64_t o = pre + __shfl_sync(FULL, incl, g) - k;
        const bool all = valid && deg <= k;
        const bool excl = valid && !all && 2 * k > deg;
        const int m = valid && !all ? (int)(excl ? deg - k : k) : 0;
        const bool slot = sub < m;
        uint32_t x = 0;
        bool kept = false;
        for (uint32_t rho = 0;; ++rho) {
            const bool need = slot && !kept;
            if (!__any_sync(FULL, need)) break;
            uint32_t v = 0xFFFFFFFFu - (uint32_t)lane;          // unique sentinel for idle lanes
            bool drew = false;
            if (need) {
                uint32_t c[4] = {(uint32_t)q, (uint32_t)hop | (rho << 8), (uint32_t)sub, 0u};
                philox4x32(c, k0, k1);
                const uint32_t bound = (uint32_t)deg;
                const uint32_t thr = (0u - bound) % bound;
#pragma unroll
                for (int u = 0; u < 4 && !drew; ++u) {
                    const uint64_t mm = (uint64_t)c[u] * bound;
                    if ((uint32_t)mm >= thr) {
                        v = (uint32_t)(mm >> 32);
                        drew = true;
                    }
                }
            } else if (kept) {
                v = x;
            }
            const unsigned keptm = __ballot_sync(FULL, kept);
            const unsigned drewm = __ballot_sync(FULL, drew);
            const unsigned peers = __match_any_sync(FULL, v) & gmask;
            if (drew) {
                const bool lose = (peers & keptm) || (peers & drewm & lt);
                if (!lose) {
                    x = v;
                    kept = true;
                }
            }
        }
        if (!valid || k == 0) continue;
        if (all) {
            for (int t = sub; t < (int)k; t += G) {
                const int32_t vv = indices[off + t];
                if (out_ids) out_ids[o + t] = vv;
                if (out_pidx) out_pidx[o + t] = (int32_t)q;
                if (bitmap) atomicOr(bitmap + (vv >> 5), 1u << (vv & 31));
            }
        } else if (!excl) {
            if (slot) {
                const int32_t vv = indices[off + x];
                if (out_ids) out_ids[o + sub] = vv;
                if (out_pidx) out_pidx[o + sub] = (int32_t)q;
                if (bitmap) atomicOr(bitmap + (vv >> 5), 1u << (vv & 31));
            }
        } else {
            // emit [0, deg) minus the m excluded indices, adjacency order (deg < 2k <= 2G)
            int base = 0;
            for (int t0 = 0; t0 < (int)deg; t0 += G) {
                const int t = t0 + sub;
                bool ex = false;
                for (int e = 0; e < m; ++e) ex |= (__shfl_sync(gmask, x, (g * G) + e, 32) == (uint32_t)t);
                const bool emit = t < (int)deg && !ex;
                const unsigned em = __ballot_sync(gmask, emit) & gmask;
                if (emit) {
                    const int pos = base + __popc(em & lt);
                    const int32_t vv = indices[off + t];
                    if (out_ids) out_ids[o + pos] = vv;
                    if (out_pidx) out_pidx[o + pos] = (int32_t)q;
                    if (bitmap) atomicOr(bitmap + (vv >> 5), 1u << (vv & 31));
                }
                base += __popc(em);
            }
        }
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

void bgl_philox4x32(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    philox4x32(c, key[0], key[1]);
    for (int i = 0; i < 4; ++i) out[i] = c[i];
}

size_t bgl_sample_hop_counter_workspace(int64_t max_parents) {
    return scan_state_bytes(1, std::max<int64_t>(1, max_parents)) + 256;   // runs of >= 1 parent
}

int bgl_sample_hop_counter(const int64_t* indptr, const int32_t* indices, const int32_t* parents,
                           const int64_t* num_parents_dev, int64_t max_parents, int32_t fanout,
                           const uint64_t* table, int32_t hop, int32_t* out_ids, int32_t* out_parent_idx,
                           int64_t* num_out_dev, void* workspace, void* mark_bitmap, void* stream) {
    BGL_CHECK_ARG(fanout >= 1 && fanout <= kCMaxK, "counter-RNG sampler: fanout must be in [1, 32]");
    BGL_CHECK_ARG(max_parents >= 0 && hop >= 0, "bgl_sample_hop_counter: bad arguments");
    BGL_CHECK_ARG(indptr && table && num_parents_dev && num_out_dev && workspace,
                  "bgl_sample_hop_counter: null pointer");
    cudaStream_t st = as_stream(stream);
    const int64_t runs = std::max<int64_t>(1, ceil_div(max_parents, 32));
    BGL_TRY(reset_scan_state(workspace, 1, runs, st));
    unsigned blocks = (unsigned)ceil_div(runs, kCWarps);
    const unsigned cap = (unsigned)kNumSMs * 8;
    if (blocks > cap) blocks = cap;
    int G = 1;
    while (G < fanout) G <<= 1;
    const int64_t R = 32 / G;
    const int64_t gruns = std::max<int64_t>(1, ceil_div(max_parents, R));
    // hop 0 (the batch's seeds: few parents, latency-bound) runs sub-warp per
    // seed; the wide later hops lane per parent (measured at C2: hop 0 13 vs
    // 24 us, hop 2 73.6 vs 40 us). The rule is part of the stream definition.
    if (hop == 0) {
        BGL_TRY(reset_scan_state(workspace, 1, gruns, st));
        unsigned gb = (unsigned)ceil_div(gruns, kCWarps);
        if (gb > (unsigned)kNumSMs * 16) gb = (unsigned)kNumSMs * 16;
        ScanState gs = make_scan_state(workspace, 1, gruns);
        uint32_t* bm = (uint32_t*)mark_bitmap;
        switch (G) {
            case 1: sample_counter_group_kernel<1><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
            case 2: sample_counter_group_kernel<2><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
            case 4: sample_counter_group_kernel<4><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
            case 8: sample_counter_group_kernel<8><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
            case 16: sample_counter_group_kernel<16><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
            default: sample_counter_group_kernel<32><<<gb, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table, hop, gs, out_ids, out_parent_idx, num_out_dev, bm); break;
        }
        return launch_status("sample_counter_group_kernel");
    }
    sample_counter_kernel<<<blocks, kCWarps * 32, 0, st>>>(indptr, indices, parents, num_parents_dev, fanout, table,
                                                            hop, make_scan_state(workspace, 1, runs), out_ids,
                                                            out_parent_idx, num_out_dev, (uint32_t*)mark_bitmap);
    return launch_status("sample_counter_kernel");
}

}  // extern "C"
