/* CPU restatement of gnnio.graph.generate_power_law + csr_from_edges in C.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/ and by
 * bench.py's reference arm (`--impl reference`) to build the reference's own
 * graph on the host without the product library or a GPU -- the reference
 * takes ~10 minutes of pure Python for the ogbn-products shape, this takes
 * seconds. It restates, step for step, the same arithmetic as the Python
 * restatement in oracle/graph_oracle.py (which is pinned to graphs produced
 * by the reference itself, tests/golden/graphgen.npz):
 *
 *   graph.py:251-274  per community, preferential attachment over the
 *                     repeated-endpoint list; the chosen targets of a node are
 *                     a CPython 3.12 `set`, iterated in slot order
 *   graph.py:276-291  cross-community edges + one bridge per ring step
 *   graph.py:293-295  the training set Generator.choice(n, k, replace=False)
 *   graph.py:88-107   csr_from_edges: drop self-loops, symmetrise, sort,
 *                     deduplicate (np.unique of src * n + dst)
 *
 * numpy's Generator(PCG64) primitives (numpy/random/src/pcg64, distributions.c):
 *   next64  = XSL-RR output of the 128-bit LCG step
 *   next32  = low half of next64 first, the high half buffered
 *   random  = (next64 >> 11) * 2^-53
 *   bounded = Lemire's 32-bit bounded draw with rejection
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
    u128 s, inc;
    int has32;
    uint32_t u32;
} gen_t;

static const u128 MULT = (((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull;

static uint64_t next64(gen_t* g) {
    g->s = g->s * MULT + g->inc;
    uint64_t hi = (uint64_t)(g->s >> 64), lo = (uint64_t)g->s;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t next32(gen_t* g) {
    if (g->has32) {
        g->has32 = 0;
        return g->u32;
    }
    uint64_t v = next64(g);
    g->has32 = 1;
    g->u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

static double random01(gen_t* g) { return (double)(next64(g) >> 11) * (1.0 / 9007199254740992.0); }

/* uniform integer in [0, rng], rng < 2^32 */
static uint32_t bounded(gen_t* g, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFull) return next32(g);
    uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
        while (left < thr) {
            m = (uint64_t)next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

/* CPython 3.12 set of non-negative ints (hash == value): 9 linear probes,
 * then perturbed probing; resized to the smallest power of two > 4 * used
 * (2 * used past 50000) once fill * 5 >= mask * 3. Iteration = slot order. */
typedef struct {
    int64_t* t;
    int64_t* spare;
    size_t cap, mask;
    int64_t fill;
} pyset_t;

static void set_init(pyset_t* s) {
    s->cap = 1024;
    s->t = (int64_t*)malloc(s->cap * sizeof(int64_t));
    s->spare = NULL;
    s->mask = 7;
    s->fill = 0;
    for (size_t i = 0; i < 8; ++i) s->t[i] = -1;
}

static void set_clear(pyset_t* s) {
    s->mask = 7;
    s->fill = 0;
    for (size_t i = 0; i < 8; ++i) s->t[i] = -1;
}

static void insert_clean(int64_t* t, size_t mask, int64_t key) {
    size_t perturb = (size_t)key, i = (size_t)key & mask;
    for (;;) {
        if (t[i] < 0) {
            t[i] = key;
            return;
        }
        if (i + 9 <= mask)
            for (size_t j = 1; j <= 9; ++j)
                if (t[i + j] < 0) {
                    t[i + j] = key;
                    return;
                }
        perturb >>= 5;
        i = (i * 5 + 1 + perturb) & mask;
    }
}

static void set_resize(pyset_t* s, int64_t minused) {
    size_t size = 8;
    while (size <= (size_t)minused) size <<= 1;
    int64_t* nt = (int64_t*)malloc(size * sizeof(int64_t));
    for (size_t i = 0; i < size; ++i) nt[i] = -1;
    for (size_t i = 0; i <= s->mask; ++i)
        if (s->t[i] >= 0) insert_clean(nt, size - 1, s->t[i]);
    free(s->t);
    s->t = nt;
    s->cap = size;
    s->mask = size - 1;
}

static void set_add(pyset_t* s, int64_t key) {
    size_t mask = s->mask, i = (size_t)key & mask, perturb = (size_t)key;
    for (;;) {
        int probes = (i + 9 <= mask) ? 9 : 0;
        size_t e = i;
        for (;;) {
            if (s->t[e] < 0) {
                s->t[e] = key;
                s->fill++;
                if ((size_t)s->fill * 5 >= mask * 3) set_resize(s, s->fill > 50000 ? s->fill * 2 : s->fill * 4);
                return;
            }
            if (s->t[e] == key) return;
            if (probes-- == 0) break;
            ++e;
        }
        perturb >>= 5;
        i = (i * 5 + 1 + perturb) & mask;
    }
}

int64_t ref_power_law_edge_bound(int64_t n, int64_t m, int32_t num_labels) {
    if (n < 2 || m < 1 || num_labels < 1) return 0;
    int64_t total = 0;
    for (int32_t c = 0; c < num_labels; ++c) {
        int64_t size = (int64_t)(c + 1) * n / num_labels - (int64_t)c * n / num_labels;
        int64_t a = m < size - 1 ? m : size - 1;
        if (a > 0) total += a * (a + 1) / 2 + (size - 1 - a) * m;
    }
    return total + n + num_labels;
}

/* state = {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger} of
 * np.random.default_rng(seed).bit_generator.state. Returns 0, or -1 when a
 * path this restatement does not cover is hit (endpoint list >= 2^32). */
int ref_power_law_generate(int64_t n, int64_t m, int32_t num_labels, double cross_fraction, int64_t num_train,
                           const uint64_t* state, int32_t* edges, int64_t* num_edges, uint8_t* train_mask) {
    gen_t g;
    g.s = ((u128)state[0] << 64) | state[1];
    g.inc = ((u128)state[2] << 64) | state[3];
    g.has32 = (int)state[4];
    g.u32 = (uint32_t)state[5];
    int64_t* bounds = (int64_t*)malloc((size_t)(num_labels + 1) * sizeof(int64_t));
    for (int32_t i = 0; i <= num_labels; ++i) bounds[i] = (int64_t)i * n / num_labels;
    int64_t E = 0, maxsize = 0;
    for (int32_t c = 0; c < num_labels; ++c)
        if (bounds[c + 1] - bounds[c] > maxsize) maxsize = bounds[c + 1] - bounds[c];
    int32_t* endpoints = (int32_t*)malloc((size_t)(2 * m * maxsize + 1) * sizeof(int32_t));
    pyset_t chosen;
    set_init(&chosen);
    for (int32_t c = 0; c < num_labels; ++c) { /* graph.py:256-274 */
        int64_t base = bounds[c], size = bounds[c + 1] - bounds[c], ne = 0;
        for (int64_t t = 1; t < size; ++t) {
            int64_t node = base + t, k = m < t ? m : t;
            set_clear(&chosen);
            while (chosen.fill < k) {
                int64_t cand;
                if (ne > 0 && random01(&g) < 0.9) {
                    if ((uint64_t)ne > 0xFFFFFFFFull) return -1;
                    cand = endpoints[bounded(&g, (uint64_t)ne - 1)];
                } else {
                    cand = base + bounded(&g, (uint64_t)t - 1);
                }
                set_add(&chosen, cand);
            }
            for (size_t i = 0; i <= chosen.mask; ++i) {
                int64_t tgt = chosen.t[i];
                if (tgt < 0) continue;
                edges[2 * E] = (int32_t)node;
                edges[2 * E + 1] = (int32_t)tgt;
                ++E;
                endpoints[ne++] = (int32_t)node;
                endpoints[ne++] = (int32_t)tgt;
            }
        }
    }
    free(endpoints);
    free(chosen.t);
    if (num_labels > 1 && cross_fraction > 0) { /* graph.py:276-291 */
        double* u = (double*)malloc((size_t)n * sizeof(double));
        for (int64_t v = 0; v < n; ++v) u[v] = random01(&g);
        int32_t c = 0;
        for (int64_t v = 0; v < n; ++v) {
            while (v >= bounds[c + 1]) ++c;
            if (!(u[v] < cross_fraction)) continue;
            int64_t other = ((int64_t)c + (random01(&g) < 0.5 ? 1 : -1) + num_labels) % num_labels;
            int64_t lo = bounds[other], hi = bounds[other + 1];
            edges[2 * E] = (int32_t)v;
            edges[2 * E + 1] = (int32_t)(lo + bounded(&g, (uint64_t)(hi - lo) - 1));
            ++E;
        }
        free(u);
        for (int32_t cc = 0; cc < num_labels; ++cc) {
            int32_t nx = (cc + 1) % num_labels;
            int64_t lo = bounds[nx], hi = bounds[nx + 1];
            edges[2 * E] = (int32_t)bounds[cc];
            edges[2 * E + 1] = (int32_t)(lo + bounded(&g, (uint64_t)(hi - lo) - 1));
            ++E;
        }
    }
    free(bounds);
    *num_edges = E;
    /* graph.py:293-295: the SET Generator.choice(n, num_train, replace=False) picks */
    memset(train_mask, 0, (size_t)n);
    if (n > 10000 && num_train > n / 50) { /* tail shuffle of arange(n) */
        int32_t* idx = (int32_t*)malloc((size_t)n * sizeof(int32_t));
        for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
        int64_t first = n - num_train > 1 ? n - num_train : 1;
        for (int64_t i = n - 1; i >= first; --i) {
            int64_t j = bounded(&g, (uint64_t)i);
            int32_t tmp = idx[i];
            idx[i] = idx[j];
            idx[j] = tmp;
        }
        for (int64_t i = n - num_train; i < n; ++i) train_mask[idx[i]] = 1;
        free(idx);
    } else { /* Floyd's algorithm; membership is train_mask itself */
        for (int64_t j = n - num_train; j < n; ++j) {
            int64_t v = bounded(&g, (uint64_t)j);
            if (train_mask[v]) v = j;
            train_mask[v] = 1;
        }
    }
    return 0;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* graph.py:88-107 (undirected): CSR of the symmetrised, sorted, deduplicated
 * edge set without self-loops. `col` has room for 2 * E entries; returns the
 * number of CSR entries (offsets[n]). */
int64_t ref_csr_from_edges(const int32_t* edges, int64_t E, int64_t n, int64_t* offsets, int64_t* col) {
    int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < E; ++e) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a == b) continue;
        deg[a]++;
        deg[b]++;
    }
    int64_t* start = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
    start[0] = 0;
    for (int64_t v = 0; v < n; ++v) start[v + 1] = start[v] + deg[v];
    memcpy(deg, start, (size_t)n * sizeof(int64_t)); /* fill cursors */
    for (int64_t e = 0; e < E; ++e) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a == b) continue;
        col[deg[a]++] = b;
        col[deg[b]++] = a;
    }
    free(deg);
    int64_t* uniq_len = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t v = 0; v < n; ++v) {
        int64_t lo = start[v], len = start[v + 1] - lo;
        if (len > 24) {
            qsort(col + lo, (size_t)len, sizeof(int64_t), cmp_i64);
        } else {
            for (int64_t i = 1; i < len; ++i) { /* insertion sort of a short row */
                int64_t x = col[lo + i], j = i;
                for (; j > 0 && col[lo + j - 1] > x; --j) col[lo + j] = col[lo + j - 1];
                col[lo + j] = x;
            }
        }
        int64_t u = 0;
        for (int64_t i = 0; i < len; ++i)
            if (u == 0 || col[lo + i] != col[lo + u - 1]) col[lo + u++] = col[lo + i];
        uniq_len[v] = u;
    }
    offsets[0] = 0;
    for (int64_t v = 0; v < n; ++v) { /* compact in place, ascending rows */
        int64_t dst = offsets[v];
        if (dst != start[v]) memmove(col + dst, col + start[v], (size_t)uniq_len[v] * sizeof(int64_t));
        offsets[v + 1] = dst + uniq_len[v];
    }
    free(uniq_len);
    free(start);
    return offsets[n];
}
