// Native, bit-exact gnnio.graph.generate_power_law (graph.py:218-297): the
// reference's sequential preferential-attachment process with numpy's
// Generator(PCG64) primitives and CPython's set iteration order restated in
// C++ (oracle: oracle/graph_oracle.py; pinned to graphs produced by the
// reference, tests/golden/graph.npz). Host code: the process is one RNG
// stream with data-dependent control flow, so it is inherently sequential; the
// C2 shape (2.4M nodes, 62M edges) takes seconds here vs ~10 minutes in the
// reference. The CSR is then built on the device (graph.py:88-107).
#include <cmath>
#include <cstring>
#include <unordered_set>
#include <vector>

#include "common.cuh"

namespace {

typedef unsigned __int128 u128;
constexpr u128 kMult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;

// numpy Generator over PCG64 (numpy/random/src/pcg64 + distributions.c)
struct Gen {
    u128 s, inc;
    int has32;
    uint32_t u32;
    uint64_t next64() {
        s = s * kMult + inc;
        const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
        const uint64_t x = hi ^ lo;
        const unsigned rot = (unsigned)(hi >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    uint32_t next32() {   // low half first, high half buffered
        if (has32) {
            has32 = 0;
            return u32;
        }
        const uint64_t v = next64();
        has32 = 1;
        u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // uniform in [0, rng], rng < 2^32 (Lemire, 32-bit)
    uint32_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        const uint32_t excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
            while (left < thr) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
    uint32_t integers(uint64_t high) { return bounded(high - 1); }
};

// CPython 3.12 set of non-negative ints (hash == value): slot table with 9
// linear probes then perturbed probing; grows to the smallest power of two >
// 4 * used when fill * 5 >= mask * 3. Iteration = slot order.
struct PySet {
    std::vector<int64_t> table, spare;
    size_t mask = 7;
    int64_t fill = 0;
    PySet() : table(8, -1) {}
    void clear() {
        if (table.size() != 8) table.assign(8, -1);
        else std::fill(table.begin(), table.end(), -1);
        mask = 7;
        fill = 0;
    }
    static void insert_clean(std::vector<int64_t>& t, size_t mask, int64_t key) {
        size_t perturb = (size_t)key, i = (size_t)key & mask;
        while (true) {
            if (t[i] < 0) {
                t[i] = key;
                return;
            }
            if (i + 9 <= mask) {
                for (size_t j = 1; j <= 9; ++j)
                    if (t[i + j] < 0) {
                        t[i + j] = key;
                        return;
                    }
            }
            perturb >>= 5;
            i = (i * 5 + 1 + perturb) & mask;
        }
    }
    void add(int64_t key) {
        size_t i = (size_t)key & mask, perturb = (size_t)key;
        while (true) {
            int probes = (i + 9 <= mask) ? 9 : 0;
            size_t e = i;
            while (true) {
                if (table[e] < 0) {
                    table[e] = key;
                    ++fill;
                    if ((size_t)fill * 5 >= mask * 3) resize(fill > 50000 ? fill * 2 : fill * 4);
                    return;
                }
                if (table[e] == key) return;
                if (probes-- == 0) break;
                ++e;
            }
            perturb >>= 5;
            i = (i * 5 + 1 + perturb) & mask;
        }
    }
    void resize(int64_t minused) {
        size_t size = 8;
        while (size <= (size_t)minused) size <<= 1;
        spare.assign(size, -1);
        for (int64_t k : table)
            if (k >= 0) insert_clean(spare, size - 1, k);
        table.swap(spare);
        mask = size - 1;
    }
};

}  // namespace

extern "C" {

int64_t bgl_power_law_edge_bound(int64_t n, int64_t m, int32_t num_labels) {
    if (n < 2 || m < 1 || num_labels < 1) return 0;
    int64_t total = 0;
    for (int32_t c = 0; c < num_labels; ++c) {
        const int64_t size = (int64_t)(c + 1) * n / num_labels - (int64_t)c * n / num_labels;
        // sum_{t=1}^{size-1} min(m, t)
        const int64_t a = std::min<int64_t>(m, size - 1);
        if (a > 0) total += a * (a + 1) / 2 + (size - 1 - a) * m;
    }
    return total + n + num_labels;   // + cross edges (<= n) + one bridge per ring step
}

int bgl_power_law_generate(int64_t n, int64_t m, int32_t num_labels, double cross_fraction, int64_t num_train,
                           const uint64_t* pcg_state, int32_t* edges_out, int64_t max_edges,
                           int64_t* num_edges_out, uint8_t* train_mask_out) {
    BGL_CHECK_ARG(n >= 2 && n < (1ll << 31), "n must be in [2, 2^31)");
    BGL_CHECK_ARG(m >= 1, "m must be >= 1");
    BGL_CHECK_ARG(num_labels >= 1 && num_labels <= n, "num_labels must be in [1, n]");
    BGL_CHECK_ARG(num_train >= 0 && num_train <= n, "num_train must be in [0, n]");
    BGL_CHECK_ARG(pcg_state && edges_out && num_edges_out && train_mask_out, "bgl_power_law_generate: null pointer");
    BGL_CHECK_ARG(max_edges >= bgl_power_law_edge_bound(n, m, num_labels), "edge buffer below bgl_power_law_edge_bound");
    Gen g;
    g.s = ((u128)pcg_state[0] << 64) | pcg_state[1];
    g.inc = ((u128)pcg_state[2] << 64) | pcg_state[3];
    g.has32 = (int)pcg_state[4];
    g.u32 = (uint32_t)pcg_state[5];
    std::vector<int64_t> bounds(num_labels + 1);
    for (int32_t i = 0; i <= num_labels; ++i) bounds[i] = (int64_t)i * n / num_labels;
    int64_t E = 0;
    PySet chosen;
    std::vector<int32_t> endpoints;
    for (int32_t c = 0; c < num_labels; ++c) {   // graph.py:256-274
        const int64_t base = bounds[c], size = bounds[c + 1] - bounds[c];
        endpoints.clear();
        endpoints.reserve((size_t)std::max<int64_t>(0, 2 * m * size));
        for (int64_t t = 1; t < size; ++t) {
            const int64_t node = base + t, k = std::min<int64_t>(m, t);
            chosen.clear();
            while (chosen.fill < k) {
                int64_t cand;
                if (!endpoints.empty() && g.random() < 0.9) {
                    if (endpoints.size() > 0xFFFFFFFFull) {
                        bgl::set_error("endpoint list beyond 2^32 entries (numpy's 64-bit bounded path) unsupported");
                        return BGL_EUNSUPPORTED;
                    }
                    cand = endpoints[g.integers(endpoints.size())];
                } else {
                    cand = base + g.integers((uint64_t)t);
                }
                chosen.add(cand);
            }
            for (int64_t tgt : chosen.table) {
                if (tgt < 0) continue;
                edges_out[2 * E] = (int32_t)node;
                edges_out[2 * E + 1] = (int32_t)tgt;
                ++E;
                endpoints.push_back((int32_t)node);
                endpoints.push_back((int32_t)tgt);
            }
        }
    }
    if (num_labels > 1 && cross_fraction > 0) {   // graph.py:276-291
        std::vector<double> u((size_t)n);
        for (int64_t v = 0; v < n; ++v) u[v] = g.random();
        int32_t c = 0;
        for (int64_t v = 0; v < n; ++v) {
            while (v >= bounds[c + 1]) ++c;
            if (!(u[v] < cross_fraction)) continue;
            const int32_t other = (int32_t)(((int64_t)c + (g.random() < 0.5 ? 1 : -1) + num_labels) % num_labels);
            const int64_t lo = bounds[other], hi = bounds[other + 1];
            edges_out[2 * E] = (int32_t)v;
            edges_out[2 * E + 1] = (int32_t)(lo + g.integers((uint64_t)(hi - lo)));
            ++E;
        }
        for (int32_t cc = 0; cc < num_labels; ++cc) {
            const int32_t nx = (cc + 1) % num_labels;
            const int64_t lo = bounds[nx], hi = bounds[nx + 1];
            edges_out[2 * E] = (int32_t)bounds[cc];
            edges_out[2 * E + 1] = (int32_t)(lo + g.integers((uint64_t)(hi - lo)));
            ++E;
        }
    }
    *num_edges_out = E;
    // train nodes: the set Generator.choice(n, num_train, replace=False) picks (graph.py:293-295)
    std::memset(train_mask_out, 0, (size_t)n);
    if (n > 10000 && num_train > n / 50) {   // tail shuffle of arange(n)
        std::vector<int32_t> idx((size_t)n);
        for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
        const int64_t first = std::max<int64_t>(n - num_train, 1);
        for (int64_t i = n - 1; i >= first; --i) {
            const int64_t j = g.bounded((uint64_t)i);
            std::swap(idx[i], idx[j]);
        }
        for (int64_t i = n - num_train; i < n; ++i) train_mask_out[idx[i]] = 1;
    } else {                                  // Floyd's algorithm
        std::unordered_set<int64_t> picked;
        picked.reserve((size_t)num_train * 2 + 1);
        for (int64_t j = n - num_train; j < n; ++j) {
            int64_t v = g.bounded((uint64_t)j);
            if (!picked.insert(v).second) {
                v = j;
                picked.insert(v);
            }
            train_mask_out[v] = 1;
        }
    }
    return BGL_OK;
}

}  // extern "C"
