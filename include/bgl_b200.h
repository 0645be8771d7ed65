/*
 * bgl_b200.h -- C ABI of the B200-native BGL per-mini-batch preprocessing path.
 *
 * Drop-in boundary. The reference (`gnnio`, /root/reference/pkg/src/gnnio) is a
 * pure-Python package, so its "FFI" for this path is the set of Python module
 * functions it exports; each entry point below replaces the arithmetic of one
 * of them and cites the reference interface (file:line) it stands in for. The
 * Python host layer `paper_2112_08541_b200/{sampler,cachesim,ordering,
 * features}.py` keeps the reference signatures and calls these through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - All functions return an int status (BGL_OK = 0) and never throw; the
 *     message of the last failure on the calling thread is bgl_last_error().
 *   - Pointers are device pointers unless the name says host. Node IDs are
 *     int32 (n < 2^31), CSR offsets int64. Sizes named `max_*` are host-known
 *     upper bounds used for launch geometry; the true counts live on the
 *     device (`*_dev` scalars) so a whole mini-batch runs without a host sync
 *     and can be captured in a CUDA graph.
 *   - `stream` is a cudaStream_t passed as void*. No function allocates device
 *     memory except bgl_cache_create; workspaces are caller-owned.
 *   - Handles are not thread-safe; order every call by stream.
 */
#ifndef BGL_B200_H
#define BGL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    BGL_OK = 0,
    BGL_EINVAL = 1,      /* bad argument (ValueError on the Python side) */
    BGL_ECUDA = 2,       /* CUDA runtime / launch failure */
    BGL_ENOMEM = 3,      /* device allocation failed */
    BGL_EUNSUPPORTED = 4 /* shape outside what the kernels implement */
};

const char* bgl_last_error(void);
int bgl_abi_version(void);

/* ---------------------------------------------------------------- host memory */
/* Device-usable alias of a pinned host buffer (zero-copy miss path). */
int bgl_host_device_pointer(void* host_ptr, void** dev_ptr);
/* Page-lock + map an existing host buffer (cudaHostRegister Mapped|Portable). */
int bgl_host_register(void* host_ptr, size_t bytes);
int bgl_host_unregister(void* host_ptr);

/* ---------------------------------------------------------------- PCG64 replay
 * Replaces the numpy stream `np.random.default_rng((cfg.seed, batch_seed))`
 * drawn by `Generator.random` in gnnio/sampler.py:61-62,90.
 * states: uint64[nb][4] = (state_hi, state_lo, inc_hi, inc_lo) taken from
 *         numpy's bit_generator.state (the host keeps SeedSequence).
 * tables: uint64[nb][BGL_PCG_TABLE_ROWS][4]; row 0 = the state, row
 *         1 + 15*i + (j-1) = (A_hi, A_lo, C_hi, C_lo) of the affine map
 *         advancing the LCG by j * 16^i steps (i < 16, 1 <= j <= 15). */
#define BGL_PCG_TABLE_ROWS 241
int bgl_pcg64_tables(const uint64_t* states, int64_t nb, uint64_t* tables, void* stream);
/* 53-bit integers m of draws [first, first+n) of the stream of `table`
 * (Generator.random() == m * 2^-53). Parity/diagnostics only. */
int bgl_pcg64_draws(const uint64_t* table, int64_t first, int64_t n, uint64_t* out, void* stream);

/* ---------------------------------------------------------------- sampler
 * One hop of uniform without-replacement neighbour sampling, bit-exact with
 * gnnio.sampler._sample_hop (sampler.py:65-94): parent q owns draws
 * [draw_base[0] + sum_{q'<q} deg(q'), ... + deg(q)) of the batch stream and
 * emits col[off_q + t] for the min(fanout, deg) smallest (draw, t), ascending,
 * grouped by parent in parent order. Writes draw_base[1] = draw_base[0] +
 * sum deg (the chain across hops, sampler.py:110-114) and *num_out_dev.
 * fanout <= 4096 (clamp it to the graph's max degree: k = min(fanout, deg)).
 * out_ids / out_parent_idx may be NULL (nothing stored: a last hop whose
 * frontier is only needed as marks in the dedup bitmap).
 * mark_bitmap (may be NULL): the dedup workspace of bgl_unique_sorted; every
 * output is also marked there (fused K2 mark), so the later
 * bgl_unique_sorted call only needs the seed segment. max_ctas > 0 caps the
 * CTAs of the sampling kernels (grid-stride loops cover the rest), leaving
 * SMs to a concurrently running gather; 0 = fill the GPU. */
size_t bgl_sample_hop_workspace(int64_t max_parents);
/* Diagnostics (tools/seg_timeline.py): buf (device, zeroed by the caller)
 * receives one {num_parents, run, smid, walk draws, t_claim, t_walk, t_post,
 * t_end} record (8 u64, globaltimer ns) per run of the segmented walk,
 * buf[0] = record count; NULL turns it off. */
int bgl_debug_seg_trace(void* buf);
int bgl_sample_hop(const int64_t* indptr, const int32_t* indices,
                   const int32_t* parents, const int64_t* num_parents_dev, int64_t max_parents,
                   int32_t fanout, const uint64_t* table, int64_t* draw_base,
                   int32_t* out_ids, int32_t* out_parent_idx, int64_t* num_out_dev,
                   void* workspace, void* mark_bitmap, int32_t max_ctas, void* stream);

/* Counter-RNG mode (not bit-exact with the reference's numpy stream): per
 * parent a uniform min(fanout, deg)-subset of its neighbours from
 * Philox4x32-10 draws keyed by the batch's stream state (row 0 of `table`) --
 * k draws per parent instead of deg. hop 0: sub-warp per seed, parallel
 * rejection rounds (counter (q, hop | round << 8, slot, 0)); later hops: lane
 * per parent, Floyd's algorithm (counter (q, hop, block, 0)); see
 * oracle/counter_sampler.py. Same outputs/layout as bgl_sample_hop (grouped
 * by parent in parent order).
 * fanout <= 32. workspace: bgl_sample_hop_counter_workspace(max_parents). */
size_t bgl_sample_hop_counter_workspace(int64_t max_parents);
/* Host-side Philox4x32-10 of the kernel (diagnostics / known-answer tests). */
void bgl_philox4x32(const uint32_t* ctr, const uint32_t* key, uint32_t* out);
int bgl_sample_hop_counter(const int64_t* indptr, const int32_t* indices, const int32_t* parents,
                           const int64_t* num_parents_dev, int64_t max_parents, int32_t fanout,
                           const uint64_t* table, int32_t hop, int32_t* out_ids, int32_t* out_parent_idx,
                           int64_t* num_out_dev, void* workspace, void* mark_bitmap, void* stream);

/* Partition accounting of simulate_epoch (sampler.py:139-153).
 * request_load[part_of[p]] += 1 for every parent; local_remote[0] += #parents
 * with part_of[p] == origins[q]; local_remote[1] += the rest. origins NULL:
 * only the load histogram (seed load, sampler.py:139). */
int bgl_comm_account(const int32_t* parents, const int64_t* num_dev, int64_t max_n,
                     const int32_t* origins, const int32_t* part_of, int32_t k,
                     int64_t* load, int64_t* local_remote, void* stream);
/* out[i] = src[idx[i]] for i < *num_dev (origin propagation, sampler.py:153). */
int bgl_take_i32(const int32_t* src, const int32_t* idx, const int64_t* num_dev, int64_t max_n,
                 int32_t* out, void* stream);

/* ---------------------------------------------------------------- dedup / relabel
 * Sorted distinct node set of a batch (np.unique, sampler.py:115,157) and the
 * relabel map rank-in-sorted-set. Direct-address bitmap over the node-ID space
 * (the paper's "contiguous 1D array as a hashmap") scanned with
 * a decoupled look-back prefix: output is sorted without a sort.
 * Keys come in up to 8 segments (seeds, hop 1, hop 2, ...): segment s is
 * keys + seg_off[s] with *seg_cnt_dev[s] valid entries (max seg_max[s]).
 * The workspace must be zeroed once (bgl_unique_workspace_init) and is left
 * clean by bgl_unique_reset. */
size_t bgl_unique_workspace(int64_t num_nodes);
int bgl_unique_workspace_init(void* workspace, int64_t num_nodes, void* stream);
int bgl_unique_sorted(const int32_t* keys, int32_t nseg, const int64_t* seg_off,
                      const int64_t* seg_cnt_dev, const int64_t* seg_max,
                      int64_t num_nodes, void* workspace,
                      int32_t* uniq_out, int64_t* num_uniq_dev, void* stream);
/* local[i] = rank of keys[i] in the sorted set (np.unique return_inverse);
 * same segment layout for keys and local. Call before bgl_unique_reset. */
int bgl_relabel(const int32_t* keys, int32_t nseg, const int64_t* seg_off,
                const int64_t* seg_cnt_dev, const int64_t* seg_max,
                int64_t num_nodes, const void* workspace, int32_t* local, void* stream);
int bgl_unique_reset(void* workspace, int64_t num_nodes, const int32_t* uniq,
                     const int64_t* num_uniq_dev, int64_t max_uniq, void* stream);

/* Sparse int64 node IDs (IDs not dense in [0, 2^31)): np.unique(keys,
 * return_inverse=True) with a GPU open-addressing hash table (linear probing,
 * 64-bit atomicCAS claim) + an LSD radix sort of the distinct keys. Replaces
 * the same np.unique (gnnio/sampler.py:115,157) where gnnio's dict-based FIFO
 * (cachesim.py:81-107, simulate :275-363) accepts any int64 node ID.
 * keys: int64[n], every key in [0, 2^key_bits) (key_bits 0 = 64; keys must be
 * >= 0). Writes the ascending distinct keys to uniq_out[0..U) (may be NULL),
 * U to *num_uniq_dev and rank_out[i] = rank of keys[i] (may be NULL). */
size_t bgl_hash_unique_workspace(int64_t max_n);
int bgl_hash_unique(const int64_t* keys, int64_t n, int32_t key_bits, void* workspace,
                    int64_t* uniq_out, int64_t* num_uniq_dev, int32_t* rank_out, void* stream);
/* home[i] = keys[i] % num_shards (cachesim.py:320) for i < *n_dev (n_dev may be
 * NULL: max_n keys). */
int bgl_key_home(const int64_t* keys, const int64_t* n_dev, int64_t max_n, int32_t num_shards,
                 uint8_t* home, void* stream);

/* ---------------------------------------------------------------- FIFO cache
 * BGL's dynamic FIFO feature cache (gnnio.cachesim FifoLevel, cachesim.py:
 * 81-107, engine cachesim.py:190-203, simulate cachesim.py:275-363).
 * `num_shards` device rings of `shard_capacity` slots (node v lives on shard
 * v % num_shards), one shared host ring of `host_capacity` slots, a direct-
 * address index per level, and optionally `row_bytes` of feature storage per
 * device slot. Batch protocol: lookup -> (gather) -> insert. */
typedef struct bgl_cache* bgl_cache_t;
int bgl_cache_create(int64_t num_nodes, int32_t num_shards, int64_t shard_capacity,
                     int64_t host_capacity, int64_t row_bytes, bgl_cache_t* out);
int bgl_cache_destroy(bgl_cache_t cache);
/* Grow the node-ID space of the index (IDs >= old num_nodes become valid). */
int bgl_cache_reserve_nodes(bgl_cache_t cache, int64_t num_nodes, void* stream);
int bgl_cache_reset(bgl_cache_t cache, void* stream);
/* Size the per-batch scratch for batches of up to max_batch distinct IDs
 * (allocates; call outside CUDA-graph capture). */
int bgl_cache_reserve_batch(bgl_cache_t cache, int64_t max_batch);
/* Multi-GPU: this single-shard handle is shard `shard_index` of
 * `num_global_shards` (node v lives on GPU v % num_global_shards,
 * cachesim.py:319-320); lookups code a hit D when worker == shard_index,
 * else P. Single-process handles keep the default (0 of num_shards). */
int bgl_cache_set_shard(bgl_cache_t cache, int32_t shard_index, int32_t num_global_shards);
/* Sparse node IDs: the cache runs on dense ranks (bgl_hash_unique) and the
 * shard of rank r is home_of[r] (= the sparse ID % num_shards) instead of
 * r % num_shards. home_of is caller-owned device memory that must outlive its
 * use; NULL restores v % num_shards. */
int bgl_cache_set_home_map(bgl_cache_t cache, const uint8_t* home_of);
/* Rename every resident rank v to old_to_new[v] (NULL: keep) and rebuild the
 * indices for a node space of new_num_nodes (the key set grew: ranks move). */
int bgl_cache_remap(bgl_cache_t cache, const int32_t* old_to_new, int64_t new_num_nodes, void* stream);
/* LRU / LFU levels (gnnio LruLevel cachesim.py:110-133, LfuLevel :136-175),
 * set once on a fresh handle without feature rows: policy 1 = LRU, 2 = LFU
 * (0 = FIFO, the default). The batch's lookup is bgl_cache_lookup (codes
 * required); bgl_cache_update_ordered then applies the batch to every level
 * in closed form (ordered.cu): LRU hits move to the recency end in the
 * order of their last hit, LFU hits add to the frequency; inserts of the
 * ascending miss lists evict per the policy. counters[5..7] += insertions,
 * evictions, metadata updates (cachesim.py:346-361). */
int bgl_cache_set_policy(bgl_cache_t cache, int32_t policy);
int bgl_cache_update_ordered(bgl_cache_t cache, const int32_t* ids, const int64_t* n_dev, int64_t max_n,
                             const uint8_t* codes, const int32_t* sorted_ids, int64_t* counters, void* stream);
/* Host copy of one level (level == num_shards: the host level): its residents
 * in eviction order (LRU: least recent first; LFU: insertion-tick order),
 * their LFU freq / tick (may be NULL), the level's tick counter and metadata
 * updates (may be NULL). list_host holds the level's capacity. */
int bgl_cache_export_ordered(bgl_cache_t cache, int32_t level, int64_t* list_host, int64_t* len_host,
                             int64_t* freq_host, int64_t* tick_host, int64_t* level_tick_host, int64_t* md_host);
/* Device pointers of the ring feature rows ([num_shards*shard_capacity][row_bytes]). */
void* bgl_cache_rows(bgl_cache_t cache);
/* Classify every query against the pre-batch state (cachesim.py:318-339):
 * codes[i] in {0:D own, 1:P peer, 2:H host, 3:M miss} (may be NULL);
 * src_row[i] = global ring row (shard*cap + slot) for D/P, -1 otherwise (may
 * be NULL); counters[0..4] += queries, own, peer, host, miss.
 * Then builds the ascending, duplicate-free insert lists from `sorted_ids`
 * (= ids itself when the batch is already sorted and unique; else the sorted
 * distinct set of ids, e.g. from bgl_unique_sorted). */
int bgl_cache_lookup(bgl_cache_t cache, const int32_t* ids, const int64_t* n_dev, int64_t max_n,
                     int32_t worker, const int32_t* sorted_ids, const int64_t* n_sorted_dev,
                     int64_t max_sorted, uint8_t* codes, int64_t* src_row, int64_t* counters,
                     void* stream);
/* The single-shard fused lookup (d == 1, ids sorted and distinct, as
 * bgl_cache_lookup with sorted_ids == ids) that also writes the ascending
 * batch positions of every device miss (H and M: rows that must come from the
 * feature store) into caller-owned miss_pos[0..*miss_count) -- the compacted
 * list bgl_gather_list consumes. */
int bgl_cache_lookup_misses(bgl_cache_t cache, const int32_t* ids, const int64_t* n_dev, int64_t max_n,
                            int32_t worker, uint8_t* codes, int64_t* src_row, int64_t* counters,
                            int32_t* miss_pos, int64_t* miss_count, void* stream);
/* Insert-after-batch (cachesim.py:341-344): device-missed into their home
 * ring, full misses into the host ring, ascending; counters[5..6] +=
 * insertions, evictions. When batch_rows != NULL, row i of the batch output
 * (aligned with sorted_ids) is copied into the slot its node lands in. */
int bgl_cache_insert(bgl_cache_t cache, const int32_t* sorted_ids, int64_t max_sorted,
                     const void* batch_rows, int64_t* counters, void* stream);
/* The same insert split in two for software pipelining: bgl_cache_insert_plan
 * updates rings, indices, tails and counters now and records every device-
 * level survivor as plan[y][r] = (batch position, slot) (int32 pairs, stride
 * bgl_cache_plan_stride) with plan_count[y] survivors; bgl_cache_copy_rows
 * later copies the survivors' rows (once the misses have arrived and the
 * batch's hits have been read). */
int64_t bgl_cache_plan_stride(bgl_cache_t cache, int64_t max_sorted);
int bgl_cache_insert_plan(bgl_cache_t cache, const int32_t* sorted_ids, int64_t max_sorted,
                          int32_t* plan, int64_t* plan_count, int64_t* counters, void* stream);
int bgl_cache_copy_rows(bgl_cache_t cache, const int32_t* plan, const int64_t* plan_count,
                        int64_t max_sorted, const void* batch_rows, void* stream);
/* bgl_cache_copy_rows with the batch rows addressed through row_index: the
 * survivor at batch position p is copied from batch_rows + row_index[p] *
 * row_bytes (multi-GPU: the rows already pushed into the worker's output,
 * read back over peer memory, row_index = the bucket's batch positions). */
int bgl_cache_copy_rows_indexed(bgl_cache_t cache, const int32_t* plan, const int64_t* plan_count,
                                int64_t max_sorted, const void* batch_rows, const int32_t* row_index,
                                void* stream);
/* Synchronous export of the ring contents (int64, -1 = empty) and tails, in
 * the layout of FifoLevel.slots / .tail (cachesim.py:87-89). Any pointer may
 * be NULL. dev_slots: [num_shards][shard_capacity]; dev_tails: [num_shards]. */
int bgl_cache_export(bgl_cache_t cache, int64_t* dev_slots_host, int64_t* dev_tails_host,
                     int64_t* host_slots_host, int64_t* host_tail_host);
/* Synchronous copy of the per-level operation counters the reference keeps on
 * every level (_Level.insertions / .evictions, cachesim.py:45-49; FifoLevel
 * increments them at cachesim.py:100,104): out_host[2 * y] = insertions,
 * out_host[2 * y + 1] = evictions of level y (y < num_shards: device rings,
 * y == num_shards: the host level). Cumulative since create / reset. */
int bgl_cache_level_stats(bgl_cache_t cache, int64_t* out_host);

/* ---------------------------------------------------------------- static-degree policy
 * gnnio.cachesim.warm_static (cachesim.py:206-224): per shard the capacity
 * highest-degree nodes (ties to the lower ID), then the host level from the
 * rest; lookups then run through bgl_cache_lookup and nothing is inserted.
 * hist: int64 [num_shards][max_degree+1] (degrees clamped), nodes flagged in
 * `exclude` (may be NULL) skipped. select flags: mode 0 -> deg == thresh[v % d]
 * (tie candidates), mode 1 -> deg > thresh[v % d] or tie_sel[v]. compact:
 * ascending IDs of the flagged nodes. warm: rings/indices filled with the
 * chosen nodes (dev_nodes concatenated shard by shard, dev_counts_host per
 * shard, host array). */
int bgl_degree_histogram(const int64_t* indptr, int64_t num_nodes, int32_t num_shards, int64_t max_degree,
                         const uint8_t* exclude, int64_t* hist, void* stream);
int bgl_select_flags(const int64_t* indptr, int64_t num_nodes, int32_t num_shards, const int64_t* thresh,
                     const uint8_t* exclude, const uint8_t* tie_sel, int32_t mode, uint8_t* flags,
                     void* stream);
size_t bgl_compact_workspace(int64_t num_nodes);
int bgl_compact_flags(const uint8_t* flags, int64_t num_nodes, int32_t* out_ids, int64_t* count_dev,
                      void* workspace, void* stream);
int bgl_cache_warm(bgl_cache_t cache, const int32_t* dev_nodes, const int64_t* dev_counts_host,
                   const int32_t* host_nodes, int64_t n_host, void* stream);

/* ---------------------------------------------------------------- feature gather
 * Net-new (the reference only counts bytes, cachesim.py:261-272):
 * out[i] = src_row[i] >= 0 ? ring_rows[src_row[i]] : table[ids[i]], 128-bit
 * vectorised. `table` may be a device pointer (HBM-resident features) or the
 * device alias of pinned host memory (zero-copy miss path). src_row NULL:
 * plain gather out[i] = table[ids[i]]. row_bytes % 4 == 0. mode: 0 = every row,
 * 1 = only hits (src_row >= 0), 2 = only misses (src_row < 0). ctas > 0:
 * launch exactly ctas CTAs of eight warps (the host-link miss path needs only
 * ~150 warps in flight, the rest of the GPU stays free for the sampler);
 * 0 = fill the GPU (HBM rows). */
int bgl_gather_rows(const int32_t* ids, const int64_t* src_row, const int64_t* n_dev, int64_t max_n,
                    const void* ring_rows, const void* table, int64_t row_bytes, void* out,
                    int32_t mode, int32_t ctas, void* stream);
/* Compacted gather: out[pos[j]] = table[ids[pos[j]]] for j < *count_dev
 * (pos from bgl_cache_lookup_misses). rows_in_flight (0 = 4, or 2/4/8) rows
 * per warp are loaded before any is stored; ctas > 0 launches exactly that
 * many 8-warp CTAs. push_out/push_pos (both or neither): every row is also
 * stored at push_out + push_pos[pos[j]] * row_bytes (home-push, peer memory);
 * with a push, `out` may be NULL. */
int bgl_gather_list(const int32_t* pos, const int64_t* count_dev, int64_t max_n, const int32_t* ids,
                    const void* table, int64_t row_bytes, void* out, void* push_out, const int32_t* push_pos,
                    int32_t rows_in_flight, int32_t ctas, void* stream);
/* bgl_gather_list for the miss path, span-aware: runs of consecutive node IDs
 * in the compacted list (consecutive output rows too) are copied with one TMA
 * bulk copy each (host/HBM -> shared -> out), single rows with 16-B loads.
 * row_bytes % 16 == 0; ctas > 0 launches exactly that many 8-warp CTAs. */
int bgl_gather_spans(const int32_t* pos, const int64_t* count_dev, int64_t max_n, const int32_t* ids,
                     const void* table, int64_t row_bytes, void* out, int32_t ctas, void* stream);
/* Fill rows of the deterministic synthetic feature table (oracle/features_oracle.py). */
int bgl_synthetic_features(int64_t first_node, int64_t num_nodes, int32_t dim, uint64_t seed,
                           float* out, void* stream);

/* ---------------------------------------------------------------- graph generator
 * Bit-exact native gnnio.graph.generate_power_law (graph.py:218-297), host
 * code: pcg_state = (state_hi, state_lo, inc_hi, inc_lo, has_uint32,
 * uinteger) of np.random.default_rng(seed).bit_generator.state, m =
 * max(1, round(avg_degree / 2)), num_train = floor(train_fraction * n).
 * edges_out: int32 [max_edges][2] host buffer (>= bgl_power_law_edge_bound)
 * receives the edges in generation order (self-loops and duplicates
 * included, as the reference's list); train_mask_out: uint8 [n]. The CSR is
 * csr_from_edges of the list (graph.py:88-107). */
int64_t bgl_power_law_edge_bound(int64_t n, int64_t m, int32_t num_labels);
int bgl_power_law_generate(int64_t n, int64_t m, int32_t num_labels, double cross_fraction, int64_t num_train,
                           const uint64_t* pcg_state, int32_t* edges_out, int64_t max_edges,
                           int64_t* num_edges_out, uint8_t* train_mask_out);

/* ---------------------------------------------------------------- ordering
 * Level-synchronous BFS of gnnio.ordering.generate_bfs_sequences
 * (ordering.py:57-116) and the closed-form round-robin of form_batches over
 * rotated sequences (ordering.py:119-151). The host keeps the numpy rng (one
 * draw per restart, ordering.py:89-90) and reads two scalars per level.
 * flags: uint8[n], bit0 = in shard, bit1 = emitted, bit2 = visited.
 * best:  int64[n] scratch, INT64_MAX on entry and left so on exit. */
size_t bgl_bfs_workspace(int64_t num_nodes);
/* One level: frontier members in the shard and not yet emitted are appended
 * to seq_out at *seq_len_dev in frontier order (*remaining_dev decremented);
 * unless *remaining_dev reached 0, the next frontier = first occurrence of
 * every unvisited neighbour in (frontier position, adjacency offset) order is
 * written to next_front / *n_next_dev and marked visited. */
int bgl_bfs_level(const int64_t* indptr, const int32_t* indices, int64_t num_nodes,
                  uint8_t* flags, const int32_t* frontier, const int64_t* n_front_dev,
                  int64_t max_front, int32_t* seq_out, int64_t* seq_len_dev,
                  int32_t* next_front, int64_t* n_next_dev, int64_t max_next,
                  int64_t* best, void* workspace, int64_t* remaining_dev, void* stream);
/* Restart root: frontier_out[0] = the r-th shard member (shard ascending) not
 * yet emitted, marked visited; *n_front_dev = 1 (ordering.py:89-92). */
int bgl_select_pending(const int32_t* shard, int64_t len, const uint8_t* flags, int64_t r,
                       int32_t* frontier_out, int64_t* n_front_dev, void* workspace,
                       int64_t num_nodes, void* stream);
/* out[pos(i, r)] = seq_i[(r + shift[i]) % L_i] with pos(i, r) = sum_j min(L_j, r)
 * + #{j < i : L_j > r}: the round-robin of form_batches over np.roll(seq_i,
 * -shift[i]). seq_off: device int64[S+1]; shift: device int64[S]. */
int bgl_interleave(const int32_t* seq_concat, const int64_t* seq_off, const int64_t* shift,
                   int32_t S, int64_t total, int32_t* out, void* stream);

/* Shuffling error of a schedule (gnnio.ordering.shuffling_error,
 * ordering.py:157-186): tv_out[i] = 0.5 * sum_c |cnt_i[c]/len_i - cnt[c]/total|
 * in fp64 for the batches order[batch_off[i] .. batch_off[i+1]) (device
 * int64[num_batches+1]); labels[v] in [0, num_classes), else *bad_label_dev
 * = 1. workspace: bgl_shuffling_workspace(num_classes) bytes. */
size_t bgl_shuffling_workspace(int32_t num_classes);
int bgl_shuffling_tv(const int32_t* labels, const int32_t* order, int64_t total, const int64_t* batch_off,
                     int64_t num_batches, int32_t num_classes, void* workspace, double* tv_out,
                     int32_t* bad_label_dev, void* stream);

/* ---------------------------------------------------------------- multi-GPU exchange
 * Node-ID sharding of the cache across GPUs (home of v = v % H,
 * cachesim.py:319-320). Stable split of a sorted batch into H ascending
 * buckets (out_ids, home-major), out_pos[i] = position of out_ids[i] in the
 * batch, counts_dev[h] = bucket sizes. Then the homes' rows come back and
 * bgl_scatter_rows puts row i at out[pos[i]]. */
size_t bgl_partition_workspace(int64_t max_n, int32_t num_homes);
int bgl_partition_by_home(const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t num_homes,
                          int32_t* out_ids, int32_t* out_pos, int64_t* counts_dev, void* workspace,
                          void* stream);
/* The partition with the ID exchange fused in (no collective for the data):
 * bucket h (ascending IDs of home h) and its batch positions are stored
 * straight into home h's receive area over peer memory -- peer_ids[h] /
 * peer_pos[h] are DEVICE arrays of H pointers (this rank's slot in every
 * home's IPC-mapped receive buffers), *peer_cnt[h] receives the bucket size.
 * counts_dev: local int64 [H]. The kernel ends with a system-scope fence; the
 * caller crosses a barrier before the homes read. */
int bgl_partition_push(const int32_t* ids, const int64_t* n_dev, int64_t max_n, int32_t num_homes,
                       int32_t* const* peer_ids, int32_t* const* peer_pos, int64_t* const* peer_cnt,
                       int64_t* counts_dev, void* workspace, void* stream);
int bgl_scatter_rows(const int32_t* pos, const int64_t* n_dev, int64_t max_n, const void* rows,
                     int64_t row_bytes, void* out, void* stream);
/* Ordered compaction: pos_out[0..*count_out) = the positions i < *n_dev with
 * codes[i] >= min_code, ascending (the worker's device-missed rows: outcome
 * codes H = 2 / M = 3 pushed back by the homes, cachesim.py:330-339 codes). */
size_t bgl_compact_codes_workspace(int64_t max_n);
int bgl_compact_codes(const uint8_t* codes, const int64_t* n_dev, int64_t max_n, int32_t min_code,
                      int32_t* pos_out, int64_t* count_out, void* workspace, void* stream);
/* Home-push gather (the row exchange fused into the gather): rows as in
 * bgl_gather_rows go to the local `out` (kept for the ring insert) AND to
 * push_out + push_pos[i] * row_bytes -- the worker GPU's output buffer,
 * mapped into this process with bgl_ipc_open_handle, written over NVLink.
 * `out` may be NULL (rows only pushed). */
int bgl_gather_rows_push(const int32_t* ids, const int64_t* src_row, const int64_t* n_dev, int64_t max_n,
                         const void* ring_rows, const void* table, int64_t row_bytes, void* out,
                         void* push_out, const int32_t* push_pos, int32_t mode, int32_t ctas,
                         void* stream);
/* Shared host level in the multi-GPU engine (the reference's single host
 * level, cachesim.py:202, lookups :330-334, inserts :343-344), owned by one
 * GPU. bgl_push_pairs: dst_ids[i] = ids[pos[i]], dst_pos[i] = pos[i] for
 * i < *n_dev and *dst_cnt = *n_dev (the worker's ascending device-missed IDs
 * into the owner's receive area; dst may be peer memory; system fence).
 * bgl_host_level_codes: dst_codes[pos[i]] = hl_codes[i] == D ? H : M (the
 * owner's single-level FIFO standing in for the host level: its hits are host
 * hits). bgl_host_level_account: counters[3] += hl[1], counters[4] -= hl[1],
 * counters[5..6] += hl[5..6], then hl = 0. */
int bgl_push_pairs(const int32_t* ids, const int32_t* pos, const int64_t* n_dev, int64_t max_n, int32_t* dst_ids,
                   int32_t* dst_pos, int64_t* dst_cnt, void* stream);
int bgl_host_level_codes(const uint8_t* hl_codes, const int32_t* pos, const int64_t* n_dev, int64_t max_n,
                         uint8_t* dst_codes, void* stream);
int bgl_host_level_account(int64_t* hl_counters, int64_t* counters, void* stream);
/* CUDA IPC of device buffers between the per-GPU processes (64-byte handles).
 * The handle names the whole allocation; *offset_out is dev_ptr's offset in
 * it (add it to the pointer bgl_ipc_open_handle returns). */
int bgl_ipc_get_handle(void* dev_ptr, void* handle_out, int64_t* offset_out);
int bgl_ipc_open_handle(const void* handle, void** dev_ptr_out);
int bgl_ipc_close(void* dev_ptr);

/* ---------------------------------------------------------------- pipeline staging
 * Step staging for the CUDA-graph-captured pipeline (no reference
 * counterpart: the reference loops batches in Python, sampler.py:136).
 * i = (*batch_counter * batch_stride + batch_offset) % num_batches (multi-GPU:
 * stride = number of GPUs, offset = rank); seeds_out = order[i*b, min((i+1)*b,
 * total)), *seed_count_out = its length, table_out = tables[i] (BGL_PCG_TABLE_ROWS x 4),
 * *batch_index_out = i (may be NULL); then *batch_counter += 1.
 * fed_count_dev != NULL (host-fed mode): `order` holds only this batch's
 * seeds (copied from the host), *fed_count_dev of them. */
int bgl_stage_batch(const int32_t* order, int64_t total, int64_t batch_size, int64_t num_batches,
                    const uint64_t* tables, int64_t* batch_counter, int32_t* seeds_out,
                    int64_t* seed_count_out, uint64_t* table_out, int64_t* batch_index_out,
                    const int64_t* fed_count_dev, int64_t batch_stride, int64_t batch_offset, void* stream);
/* Append one batch's sorted distinct IDs to a device-resident trace without
 * a host round trip (simulate_epoch, sampler.py:157): dst[off[b] ..
 * off[b] + n) = src[0 .. n), off[b + 1] = off[b] + n, with n = *n_dev and
 * `off` a device int64 array (off[0] = 0) -- the AccessTrace rows of an epoch
 * are copied to the host once at its end. */
int bgl_trace_append(const int32_t* src, const int64_t* n_dev, int64_t max_n, int32_t* dst, int64_t* off,
                     int64_t batch, void* stream);
/* Sync-free result hand-off: host_ids[0..n) = ids[0..*n_dev) and host_meta =
 * {n, counters[0..8)} written straight into mapped pinned host memory
 * (device aliases from bgl_host_device_pointer). counters may be NULL. */
int bgl_d2h_result(const int32_t* ids, const int64_t* n_dev, int64_t max_n, const int64_t* counters,
                   int32_t* host_ids, int64_t* host_meta, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BGL_B200_H */
