// K7/K8: proximity-aware ordering on the device, bit-exact with
// gnnio.ordering.generate_bfs_sequences (ordering.py:57-116) and the
// round-robin of form_batches over randomly shifted sequences
// (ordering.py:119-151, 192-196).
//
// One BFS level:
//   bfs_emit   frontier members that are in the shard and not yet emitted are
//              appended to the sequence in frontier order (stable compaction,
//              ordering.py:94-98); the same look-back pass computes the
//              prefix of frontier degrees = the global position key base
//              g(i, j) = sum_{i'<i} deg(front[i']) + j of every candidate.
//   bfs_mark   candidates = adjacency of the frontier in frontier order; the
//              first occurrence of every unvisited neighbour is the smallest
//              key: atomicMin(best[u], g) (ordering.py:100-111).
//   bfs_next   keep candidate (i, j) iff best[u] == g(i, j); stable
//              compaction in key order -> next frontier; mark visited and
//              reset best[u] (ordering.py:111-112).
// The host keeps the numpy rng (one draw per restart, ordering.py:89-90) and
// `bfs_select` turns the draw r into the r-th pending shard member.
#include <algorithm>

#include "common.cuh"
#include "scan.cuh"

namespace bgl {

constexpr uint8_t kInShard = 1, kEmitted = 2, kVisited = 4;
constexpr int kBThreads = 256;
constexpr int kBItems = 8;
constexpr int kBTile = kBThreads * kBItems;
constexpr int kNextTile = kBThreads;   // frontier nodes per bfs_next tile
constexpr unsigned long long kInf = 0x7fffffffffffffffull;

struct BfsWs {
    int64_t* pre_deg;   // [n]
    void* scan_emit;    // 2 values, tiles of kBTile
    void* scan_next;    // 1 value, tiles of kNextTile
    void* scan_sel;     // 1 value, tiles of kBTile
    int64_t t_emit, t_next, t_sel;
    int64_t* scalars;   // [0] = number of candidates (sum deg of frontier)
};

static size_t al256b(size_t x) { return (x + 255) & ~(size_t)255; }

static BfsWs carve_bfs(void* ws, int64_t n) {
    BfsWs w;
    n = n > 0 ? n : 1;
    w.t_emit = ceil_div(n, kBTile);
    w.t_next = ceil_div(n, kNextTile);
    w.t_sel = ceil_div(n, kBTile);
    char* p = reinterpret_cast<char*>(ws);
    w.pre_deg = reinterpret_cast<int64_t*>(p);
    p += al256b(n * 8);
    w.scan_emit = p;
    p += al256b(scan_state_bytes(2, w.t_emit));
    w.scan_next = p;
    p += al256b(scan_state_bytes(1, w.t_next));
    w.scan_sel = p;
    p += al256b(scan_state_bytes(1, w.t_sel));
    w.scalars = reinterpret_cast<int64_t*>(p);
    return w;
}

__global__ void __launch_bounds__(kBThreads)
bfs_emit_kernel(const int64_t* __restrict__ indptr, uint8_t* __restrict__ flags, const int32_t* __restrict__ front,
                const int64_t* __restrict__ n_front_dev, ScanState ss, int64_t* __restrict__ pre_deg,
                int32_t* __restrict__ seq_out, int64_t* __restrict__ seq_len, int64_t* __restrict__ remaining,
                int64_t* __restrict__ n_cand) {
    __shared__ int32_t s_v[kBTile];
    __shared__ int64_t s_deg[kBTile];
    __shared__ int64_t s_red[kBThreads / 32 + 1];
    __shared__ int64_t s_agg[2], s_pre[2], s_slot;
    const int64_t n = *n_front_dev;
    // read before publishing anything: the last tile rewrites *seq_len only
    // after every tile has published (look-back chain), hence after this read
    const int64_t sl = *seq_len;
    const int64_t ntiles = n > 0 ? ceil_div(n, kBTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int64_t base = tile * kBTile;
    for (int i = threadIdx.x; i < kBTile; i += kBThreads) {
        int64_t q = base + i;
        int32_t v = -1;
        int64_t d = 0;
        if (q < n) {
            v = front[q];
            d = indptr[v + 1] - indptr[v];
            uint8_t f = flags[v];
            if (!((f & kInShard) && !(f & kEmitted))) v = -1 - v;   // keep id, mark "not emitted"
        }
        s_v[i] = v;
        s_deg[i] = d;
    }
    __syncthreads();
    const int first = threadIdx.x * kBItems;
    int64_t my_e = 0, my_d = 0;
#pragma unroll
    for (int j = 0; j < kBItems; ++j) {
        my_e += (s_v[first + j] >= 0);
        my_d += s_deg[first + j];
    }
    int64_t tot_e, tot_d;
    int64_t ex_e = block_excl_scan(my_e, s_red, &tot_e);
    int64_t ex_d = block_excl_scan(my_d, s_red, &tot_d);
    if (threadIdx.x == 0) {
        s_agg[0] = tot_e;
        s_agg[1] = tot_d;
    }
    __syncthreads();
    lookback<2>(ss, tile, s_agg, s_pre);
    int64_t re = s_pre[0] + ex_e, rd = s_pre[1] + ex_d;
#pragma unroll
    for (int j = 0; j < kBItems; ++j) {
        int64_t q = base + first + j;
        if (q < n) {
            int32_t v = s_v[first + j];
            pre_deg[q] = rd;
            rd += s_deg[first + j];
            if (v >= 0) {
                seq_out[sl + re] = v;
                flags[v] |= kEmitted;
                ++re;
            }
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        *seq_len = sl + s_pre[0] + tot_e;
        *remaining -= s_pre[0] + tot_e;
        *n_cand = s_pre[1] + tot_d;
    }
}

__global__ void bfs_mark_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                const uint8_t* __restrict__ flags, const int32_t* __restrict__ front,
                                const int64_t* __restrict__ n_front_dev, const int64_t* __restrict__ pre_deg,
                                const int64_t* __restrict__ remaining, unsigned long long* __restrict__ best) {
    if (*remaining <= 0) return;
    const int64_t n = *n_front_dev;
    const int lane = lane_id();
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t v = front[i];
        const int64_t off = indptr[v];
        const int64_t deg = indptr[v + 1] - off;
        const int64_t g0 = pre_deg[i];
        for (int64_t j = lane; j < deg; j += 32) {
            const int32_t u = indices[off + j];
            if (!(flags[u] & kVisited)) atomicMin(best + u, (unsigned long long)(g0 + j));
        }
    }
}

__global__ void __launch_bounds__(kBThreads)
bfs_next_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                uint8_t* __restrict__ flags, const int32_t* __restrict__ front, const int64_t* __restrict__ n_front_dev,
                const int64_t* __restrict__ pre_deg, const int64_t* __restrict__ remaining,
                unsigned long long* __restrict__ best, ScanState ss, int32_t* __restrict__ next,
                int64_t* __restrict__ n_next) {
    __shared__ int64_t s_cnt[kNextTile];
    __shared__ int64_t s_red[kBThreads / 32 + 1];
    __shared__ int64_t s_agg[1], s_pre[1], s_slot;
    const int64_t n = (*remaining > 0) ? *n_front_dev : 0;
    const int64_t ntiles = n > 0 ? ceil_div(n, kNextTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int lane = lane_id(), wid = warp_id();
    const unsigned lt = (1u << lane) - 1u;
    const int per_warp = kNextTile / (kBThreads / 32);
    // pass 1: kept count per frontier node
    for (int k = 0; k < per_warp; ++k) {
        const int li = wid * per_warp + k;
        const int64_t i = tile * kNextTile + li;
        int64_t cnt = 0;
        if (i < n) {
            const int32_t v = front[i];
            const int64_t off = indptr[v];
            const int64_t deg = indptr[v + 1] - off;
            const int64_t g0 = pre_deg[i];
            for (int64_t j0 = 0; j0 < deg; j0 += 32) {
                const int64_t j = j0 + lane;
                bool keep = false;
                if (j < deg) keep = ld_volatile(best + indices[off + j]) == (unsigned long long)(g0 + j);
                cnt += __popc(__ballot_sync(0xffffffffu, keep));
            }
        }
        if (lane == 0) s_cnt[li] = cnt;
    }
    __syncthreads();
    int64_t tot;
    int64_t ex = block_excl_scan(s_cnt[threadIdx.x], s_red, &tot);
    __syncthreads();
    s_cnt[threadIdx.x] = ex;
    if (threadIdx.x == 0) s_agg[0] = tot;
    __syncthreads();
    lookback<1>(ss, tile, s_agg, s_pre);
    // pass 2: write in key order, mark visited, reset best
    for (int k = 0; k < per_warp; ++k) {
        const int li = wid * per_warp + k;
        const int64_t i = tile * kNextTile + li;
        if (i >= n) break;
        const int32_t v = front[i];
        const int64_t off = indptr[v];
        const int64_t deg = indptr[v + 1] - off;
        const int64_t g0 = pre_deg[i];
        int64_t pos = s_pre[0] + s_cnt[li];
        for (int64_t j0 = 0; j0 < deg; j0 += 32) {
            const int64_t j = j0 + lane;
            int32_t u = -1;
            bool keep = false;
            if (j < deg) {
                u = indices[off + j];
                keep = ld_volatile(best + u) == (unsigned long long)(g0 + j);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                next[pos + __popc(m & lt)] = u;
                flags[u] |= kVisited;
                best[u] = kInf;
            }
            pos += __popc(m);
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *n_next = s_pre[0] + tot;
}

__global__ void __launch_bounds__(kBThreads)
bfs_select_kernel(const int32_t* __restrict__ shard, int64_t len, uint8_t* __restrict__ flags, int64_t r,
                  ScanState ss, int32_t* __restrict__ front, int64_t* __restrict__ n_front) {
    __shared__ int64_t s_red[kBThreads / 32 + 1];
    __shared__ int64_t s_agg[1], s_pre[1], s_slot;
    const int64_t ntiles = len > 0 ? ceil_div(len, kBTile) : 1;
    const int64_t tile = claim_tile(ss, &s_slot);
    if (tile >= ntiles) return;
    const int64_t q0 = tile * kBTile + (int64_t)threadIdx.x * kBItems;
    int64_t cnt = 0;
    for (int j = 0; j < kBItems; ++j) {
        int64_t q = q0 + j;
        if (q < len) cnt += !(flags[shard[q]] & kEmitted);
    }
    int64_t tot;
    int64_t ex = block_excl_scan(cnt, s_red, &tot);
    if (threadIdx.x == 0) s_agg[0] = tot;
    __syncthreads();
    lookback<1>(ss, tile, s_agg, s_pre);
    int64_t rank = s_pre[0] + ex;
    for (int j = 0; j < kBItems; ++j) {
        int64_t q = q0 + j;
        if (q < len) {
            int32_t v = shard[q];
            if (!(flags[v] & kEmitted)) {
                if (rank == r) {
                    front[0] = v;
                    flags[v] |= kVisited;
                    *n_front = 1;
                }
                ++rank;
            }
        }
    }
}

__global__ void interleave_kernel(const int32_t* __restrict__ seqs, const int64_t* __restrict__ seq_off,
                                  const int64_t* __restrict__ shift, int32_t S, int64_t total,
                                  int32_t* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int i = 0;
        while (i + 1 < S && e >= seq_off[i + 1]) ++i;
        const int64_t r = e - seq_off[i];
        int64_t pos = 0;
        for (int j = 0; j < S; ++j) {
            const int64_t L = seq_off[j + 1] - seq_off[j];
            pos += L < r ? L : r;
            if (j < i && L > r) ++pos;
        }
        const int64_t Li = seq_off[i + 1] - seq_off[i];
        out[pos] = seqs[seq_off[i] + (r + shift[i]) % Li];
    }
}

}  // namespace bgl

using namespace bgl;

extern "C" {

size_t bgl_bfs_workspace(int64_t num_nodes) {
    int64_t n = num_nodes > 0 ? num_nodes : 1;
    return al256b(n * 8) + al256b(scan_state_bytes(2, ceil_div(n, kBTile))) +
           al256b(scan_state_bytes(1, ceil_div(n, kNextTile))) + al256b(scan_state_bytes(1, ceil_div(n, kBTile))) +
           256;
}

int bgl_bfs_level(const int64_t* indptr, const int32_t* indices, int64_t num_nodes, uint8_t* flags,
                  const int32_t* frontier, const int64_t* n_front_dev, int64_t max_front, int32_t* seq_out,
                  int64_t* seq_len_dev, int32_t* next_front, int64_t* n_next_dev, int64_t max_next, int64_t* best,
                  void* workspace, int64_t* remaining_dev, void* stream) {
    BGL_CHECK_ARG(indptr && indices && flags && frontier && n_front_dev && seq_out && seq_len_dev && next_front &&
                      n_next_dev && best && workspace && remaining_dev,
                  "bgl_bfs_level: null pointer");
    BGL_CHECK_ARG(max_front >= 0 && max_front <= num_nodes && max_next <= num_nodes, "frontier larger than graph");
    cudaStream_t st = as_stream(stream);
    BfsWs w = carve_bfs(workspace, num_nodes);
    const int64_t tf = std::max<int64_t>(1, ceil_div(max_front, kBTile));
    BGL_TRY(reset_scan_state(w.scan_emit, 2, w.t_emit, st));
    bfs_emit_kernel<<<(unsigned)tf, kBThreads, 0, st>>>(indptr, flags, frontier, n_front_dev,
                                                        make_scan_state(w.scan_emit, 2, w.t_emit), w.pre_deg, seq_out,
                                                        seq_len_dev, remaining_dev, w.scalars);
    BGL_TRY(launch_status("bfs_emit_kernel"));
    if (max_front > 0) {
        bfs_mark_kernel<<<grid_for(max_front * 32, 256, 16), 256, 0, st>>>(
            indptr, indices, flags, frontier, n_front_dev, w.pre_deg, remaining_dev, (unsigned long long*)best);
        BGL_TRY(launch_status("bfs_mark_kernel"));
    }
    const int64_t tn = std::max<int64_t>(1, ceil_div(max_front, kNextTile));
    BGL_TRY(reset_scan_state(w.scan_next, 1, w.t_next, st));
    bfs_next_kernel<<<(unsigned)tn, kBThreads, 0, st>>>(indptr, indices, flags, frontier, n_front_dev, w.pre_deg,
                                                        remaining_dev, (unsigned long long*)best,
                                                        make_scan_state(w.scan_next, 1, w.t_next), next_front,
                                                        n_next_dev);
    return launch_status("bfs_next_kernel");
}

int bgl_select_pending(const int32_t* shard, int64_t len, const uint8_t* flags, int64_t r, int32_t* frontier_out,
                       int64_t* n_front_dev, void* workspace, int64_t num_nodes, void* stream) {
    BGL_CHECK_ARG(shard && flags && frontier_out && n_front_dev && workspace, "bgl_select_pending: null pointer");
    BGL_CHECK_ARG(r >= 0 && r < len, "pending index out of range");
    cudaStream_t st = as_stream(stream);
    BfsWs w = carve_bfs(workspace, num_nodes);
    BGL_TRY(reset_scan_state(w.scan_sel, 1, w.t_sel, st));
    bfs_select_kernel<<<(unsigned)std::max<int64_t>(1, ceil_div(len, kBTile)), kBThreads, 0, st>>>(
        shard, len, const_cast<uint8_t*>(flags), r, make_scan_state(w.scan_sel, 1, w.t_sel), frontier_out,
        n_front_dev);
    return launch_status("bfs_select_kernel");
}

int bgl_interleave(const int32_t* seq_concat, const int64_t* seq_off, const int64_t* shift, int32_t S, int64_t total,
                   int32_t* out, void* stream) {
    BGL_CHECK_ARG(S >= 1, "need at least one sequence");
    BGL_CHECK_ARG(seq_concat && seq_off && shift && out, "bgl_interleave: null pointer");
    if (total <= 0) return BGL_OK;
    interleave_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(seq_concat, seq_off, shift, S, total, out);
    return launch_status("interleave_kernel");
}

}  // extern "C"
