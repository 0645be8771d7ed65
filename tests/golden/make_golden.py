"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `gnnio` read-only from /root/reference/pkg/src and writes
sampler.npz / cache.npz / ordering.npz next to this file. The fixtures are
committed; nothing on the GPU box reads /root/reference.

What is pinned (the reference ships no golden arrays):
  * sampler: per-hop frontiers + parent_idx of `_sample_hop` chained exactly
    as `sample_batch` does (sampler.py:97-116), `sample_batch`'s distinct set,
    and `simulate_epoch` traces + EpochCommReport (sampler.py:119-167);
  * cache: per-batch counters, per-node outcome codes and the ring contents +
    tail of every level after every batch (cachesim.py:81-107, 275-363);
  * ordering: `generate_bfs_sequences`, `proximity_schedule`,
    `random_shuffle_schedule` (ordering.py:57-207).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from packing import put  # noqa: E402

from gnnio import cachesim as cs  # noqa: E402
from gnnio import ordering as od  # noqa: E402
from gnnio import sampler as sp  # noqa: E402
from gnnio.graph import build_graph, generate_power_law  # noqa: E402
from gnnio.partition import random_partition  # noqa: E402
from gnnio.sampler import AccessTrace  # noqa: E402


def make_graph(edges, n, train=None):
    g = build_graph(np.array(edges, dtype=np.int64).reshape(-1, 2), n, undirected=True)
    if train is not None:
        g.train_mask[:] = False
        g.train_mask[list(train)] = True
    return g


def graphs():
    gs = {}
    gs["planted"] = generate_power_law(2000, 8, seed=4, train_fraction=0.1, num_labels=8)
    gs["star6"] = make_graph([(0, i) for i in range(1, 6)], 6, train=range(6))
    gs["path5"] = make_graph([(0, 1), (1, 2), (2, 3), (3, 4)], 5, train=range(5))
    gs["isolated"] = make_graph([(0, 1), (1, 2), (3, 4)], 8, train=[0, 2, 5, 6, 7])
    gs["dense"] = generate_power_law(3000, 40, seed=3, train_fraction=0.2, num_labels=4)
    return gs


def store_graph(out, name, g):
    out[f"g_{name}_off"] = g.row_offsets.astype(np.int64)
    out[f"g_{name}_col"] = g.col_indices.astype(np.int64)
    out[f"g_{name}_train"] = g.train_mask.astype(np.uint8)


def sampler_cases(gs):
    rng = np.random.default_rng(2024)
    cases = []
    pl = gs["planted"]
    dn = gs["dense"]
    cases.append(("star6", [0], (3, 3), 7, 0))
    cases.append(("star6", [0, 0, 3], (10, 2), 1, 5))
    cases.append(("isolated", [5, 2, 5, 0], (4, 4), 0, 0))
    cases.append(("path5", [2], (1, 1, 1), 3, 9))
    for i in range(6):
        seeds = pl.train_nodes()[rng.integers(pl.num_train(), size=int(rng.integers(1, 80)))]
        fan = tuple(int(x) for x in rng.integers(1, 16, size=int(rng.integers(1, 4))))
        cases.append(("planted", seeds.tolist(), fan, int(rng.integers(100)), int(rng.integers(1000))))
    # high fanouts (> 32 and >= hub degrees) exercise the wide-k path
    for fan in ((40,), (64, 3), (200,), (15, 10, 5)):
        seeds = dn.train_nodes()[rng.integers(dn.num_train(), size=24)]
        cases.append(("dense", seeds.tolist(), fan, int(rng.integers(100)), int(rng.integers(1000))))
    return cases


def make_sampler(gs):
    out = {}
    for name, g in gs.items():
        store_graph(out, name, g)
    cases = sampler_cases(gs)
    meta, seeds_l, fan_l, fr_l, pi_l, dist_l = [], [], [], [], [], []
    hop_count = []
    for gname, seeds, fan, seed, bseed in cases:
        g = gs[gname]
        cfg = sp.SamplingConfig(fanouts=fan, seed=seed)
        rng = sp._batch_rng(cfg, bseed)
        parents = np.asarray(seeds, dtype=np.int64)
        for f in fan:
            ids, pidx = sp._sample_hop(g, parents, f, rng)
            fr_l.append(ids)
            pi_l.append(pidx)
            parents = ids
        frontiers, distinct = sp.sample_batch(g, np.asarray(seeds), cfg, batch_seed=bseed)
        for a, b in zip(frontiers, fr_l[-len(fan):]):
            assert np.array_equal(a, b)
        dist_l.append(distinct)
        seeds_l.append(seeds)
        fan_l.append(fan)
        hop_count.append(len(fan))
        meta.append((list(gs).index(gname), seed, bseed))
    out["graph_names"] = np.array(list(gs))
    out["case_meta"] = np.array(meta, dtype=np.int64)
    put(out, "case_seeds", seeds_l)
    put(out, "case_fanouts", fan_l)
    put(out, "hop_ids", fr_l)
    put(out, "hop_pidx", pi_l)
    put(out, "distinct", dist_l)

    # epochs: simulate_epoch over two schedules and two partitionings
    pl = gs["planted"]
    ep_meta, ep_trace, ep_batches = [], [], []
    ep_report = []
    for k, sched_kind, fan, seed in ((4, "prox", (5, 5), 7), (1, "rand", (10, 5), 0), (3, "rand", (15, 10, 5), 2)):
        part = random_partition(pl, k, seed=seed)
        if sched_kind == "prox":
            sched = od.proximity_schedule(pl, 2, 40, seed=0)
        else:
            sched = od.random_shuffle_schedule(pl, 64, seed=seed)
        trace, rep = sp.simulate_epoch(pl, part, sched, sp.SamplingConfig(fanouts=fan, seed=seed))
        ep_meta.append((k, seed, len(sched.batches)))
        ep_batches.append(sched.batches)
        ep_trace.append(trace.batches)
        ep_report.append((rep.local_accesses, rep.remote_accesses, rep.seed_load, rep.request_load, part.part_of))
        out[f"epoch{len(ep_meta) - 1}_fanouts"] = np.array(fan, dtype=np.int64)
    out["epoch_meta"] = np.array(ep_meta, dtype=np.int64)
    for e, (batches, trace, rep) in enumerate(zip(ep_batches, ep_trace, ep_report)):
        put(out, f"epoch{e}_batches", batches)
        put(out, f"epoch{e}_trace", trace)
        out[f"epoch{e}_local_remote"] = np.array(rep[:2], dtype=np.int64)
        out[f"epoch{e}_seed_load"] = rep[2]
        out[f"epoch{e}_request_load"] = rep[3]
        out[f"epoch{e}_part_of"] = rep[4].astype(np.int64)
    np.savez_compressed(os.path.join(HERE, "sampler.npz"), **out)


def cache_case_batches(rng, kind):
    universe = int(rng.integers(8, 300))
    batches = []
    remaining = int(rng.integers(50, 3000))
    while remaining > 0:
        size = int(min(remaining, rng.integers(1, min(universe, 64) + 1)))
        b = rng.choice(universe, size=size, replace=False)
        if kind == "sorted":
            b = np.sort(b)
        elif kind == "dups":
            b = np.concatenate([b, b[: max(1, size // 3)]])
            rng.shuffle(b)
        batches.append(b)
        remaining -= size
    return batches


def make_cache():
    rng = np.random.default_rng(42)
    out = {}
    specs = []
    all_batches, all_codes, all_counters = [], [], []
    dev_slots, dev_tails, host_slots, host_tails = [], [], [], []
    kinds = ["sorted"] * 40 + ["unsorted"] * 10 + ["dups"] * 10
    for ci, kind in enumerate(kinds):
        batches = cache_case_batches(rng, kind)
        d = int(rng.choice([1, 2, 4, 8]))
        cap = int(rng.integers(0, 65))
        hcap = int(rng.choice([0, 1, 8, 64]))
        use_bd = ci % 5 == 4
        bd = [int(x) for x in rng.integers(d, size=len(batches))] if use_bd else None
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy="fifo",
                             feature_bytes_per_node=400)
        state = cs.cold_state(cfg)
        codes_case, cnt_case = [], []
        ds, dt, hs, ht = [], [], [], []
        for i, b in enumerate(batches):
            rep = cs.simulate(AccessTrace(batches=[np.asarray(b, dtype=np.int64)]), cfg,
                              batch_devices=[bd[i] if bd else i % d], state=state, record_outcomes=True)
            codes_case.append(np.array(["DPHM".index(c) for c in rep.outcomes[0]], dtype=np.int64))
            cnt_case.append([rep.batch_queries[0], rep.batch_own_hits[0], rep.batch_peer_hits[0],
                             rep.batch_host_hits[0], rep.batch_misses[0], rep.batch_insertions[0],
                             rep.batch_evictions[0], rep.batch_metadata_updates[0]])
            ds.append(np.stack([lv.slots for lv in state.devices]).ravel())
            dt.append([lv.tail for lv in state.devices])
            hs.append(state.host.slots.copy())
            ht.append(state.host.tail)
        # the whole-trace call must agree with the batch-at-a-time replay
        whole = cs.simulate(AccessTrace(batches=[np.asarray(b, dtype=np.int64) for b in batches]), cfg,
                            batch_devices=bd, record_outcomes=True)
        assert whole.batch_misses == [c[4] for c in cnt_case]
        specs.append((d, cap, hcap, len(batches), int(use_bd), ["sorted", "unsorted", "dups"].index(kind)))
        all_batches.extend(batches)
        all_codes.extend(codes_case)
        all_counters.extend(cnt_case)
        dev_slots.extend(ds)
        dev_tails.extend(dt)
        host_slots.extend(hs)
        host_tails.append(ht)
        out[f"bd_{ci}"] = np.array(bd if bd else [], dtype=np.int64)
    out["specs"] = np.array(specs, dtype=np.int64)
    put(out, "batches", all_batches)
    put(out, "codes", all_codes, np.int8)
    out["counters"] = np.array(all_counters, dtype=np.int64)
    put(out, "dev_slots", dev_slots)
    put(out, "dev_tails", dev_tails)
    put(out, "host_slots", host_slots)
    put(out, "host_tails", host_tails)

    # a sampler-produced trace at desk scale (acceptance-style, 10% capacity)
    g = generate_power_law(5000, 10, seed=1, train_fraction=0.1, num_labels=16)
    sched = od.proximity_schedule(g, 4, 100, seed=1)
    trace, _ = sp.simulate_epoch(g, random_partition(g, 1, seed=0), sched,
                                 sp.SamplingConfig(fanouts=(10, 5), seed=1))
    put(out, "real_trace", trace.batches)
    real = []
    for d in (1, 2, 4, 8):
        rep = cs.simulate(trace, cs.CacheConfig(device_capacity=500 // d, host_capacity=250,
                                                num_devices=d, policy="fifo"), record_outcomes=True)
        real.append([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                     rep.batch_misses, rep.batch_insertions, rep.batch_evictions])
    out["real_counters"] = np.array(real, dtype=np.int64)   # [4 d-values, 7, nb]
    np.savez_compressed(os.path.join(HERE, "cache.npz"), **out)


def make_ordering(gs):
    out = {}
    for name, g in gs.items():
        store_graph(out, name, g)
    out["graph_names"] = np.array(list(gs))
    seq_meta, seqs, scheds, sched_meta = [], [], [], []
    for gname, S, seed in (("planted", 1, 0), ("planted", 3, 1), ("planted", 4, 2), ("planted", 7, 5),
                           ("dense", 4, 3), ("path5", 1, 4), ("star6", 2, 6), ("isolated", 2, 1),
                           ("isolated", 5, 8)):
        g = gs[gname]
        res = od.generate_bfs_sequences(g, S, seed=seed)
        seq_meta.append((list(gs).index(gname), S, seed))
        seqs.extend(res)
    # random small (mostly disconnected) graphs exercise restarts
    rng = np.random.default_rng(77)
    rnd_graphs = []
    for i in range(12):
        n = int(rng.integers(20, 400))
        m = int(rng.integers(n // 2, 2 * n))
        g = build_graph(rng.integers(n, size=(m, 2)), n)
        g.train_mask[rng.random(n) < 0.4] = True
        if g.num_train() < 6:
            g.train_mask[:6] = True
        store_graph(out, f"rnd{i}", g)
        S = int(rng.integers(1, 6))
        seed = int(rng.integers(1000))
        res = od.generate_bfs_sequences(g, S, seed=seed)
        seq_meta.append((100 + i, S, seed))
        seqs.extend(res)
        b = int(rng.integers(1, 30))
        sched = od.proximity_schedule(g, S, b, seed=seed)
        sched_meta.append((100 + i, S, b, seed, len(sched.batches), 0))
        scheds.extend(sched.batches)
        rs = od.random_shuffle_schedule(g, b, seed=seed)
        sched_meta.append((100 + i, 0, b, seed, len(rs.batches), 1))
        scheds.extend(rs.batches)
    for gname, S, b, seed in (("planted", 4, 64, 2), ("dense", 4, 100, 1), ("planted", 2, 40, 0)):
        g = gs[gname]
        sched = od.proximity_schedule(g, S, b, seed=seed)
        sched_meta.append((list(gs).index(gname), S, b, seed, len(sched.batches), 0))
        scheds.extend(sched.batches)
    out["seq_meta"] = np.array(seq_meta, dtype=np.int64)
    put(out, "seqs", seqs)
    out["sched_meta"] = np.array(sched_meta, dtype=np.int64)
    put(out, "sched_batches", scheds)
    np.savez_compressed(os.path.join(HERE, "ordering.npz"), **out)


def make_static(gs):
    out = {}
    for name, g in gs.items():
        store_graph(out, name, g)
    out["graph_names"] = np.array(list(gs))
    rng = np.random.default_rng(31)
    meta, dev_sets, host_sets, counters, codes, batches_all = [], [], [], [], [], []
    for gname in ("planted", "dense", "star6", "isolated"):
        g = gs[gname]
        n = g.num_nodes
        for d, cap, hcap in ((1, 0, 0), (1, 2, 0), (1, n // 10, n // 20), (2, 7, 3), (4, n // 8, 0), (3, n, n),
                             (4, 1, 5)):
            cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy="static-degree")
            state = cs.warm_static(g, cfg)
            batches = [np.unique(rng.integers(0, n, size=int(rng.integers(1, max(2, n // 4))))) for _ in range(6)]
            rep = cs.simulate(AccessTrace(batches=batches), cfg, g=g, record_outcomes=True)
            meta.append((list(gs).index(gname), d, cap, hcap, len(batches)))
            dev_sets.extend(sorted(lv.resident) for lv in state.devices)
            host_sets.append(sorted(state.host.resident))
            counters.extend(zip(rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                                rep.batch_misses, rep.batch_insertions, rep.batch_evictions))
            codes.extend(np.array(["DPHM".index(c) for c in oc], dtype=np.int64) for oc in rep.outcomes)
            batches_all.extend(batches)
    out["meta"] = np.array(meta, dtype=np.int64)
    put(out, "dev_sets", dev_sets)
    put(out, "host_sets", host_sets)
    put(out, "batches", batches_all)
    put(out, "codes", codes, np.int8)
    out["counters"] = np.array(counters, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "static.npz"), **out)


def make_shuffle(gs):
    """shuffling_error / select_num_sequences (ordering.py:157-231)."""
    out = {}
    graphs = {"planted": gs["planted"], "dense": gs["dense"],
              "one_label": generate_power_law(2000, 8, seed=4, train_fraction=0.1, num_labels=1),
              "two_comm": generate_power_law(5000, 10, seed=3, train_fraction=0.1, num_labels=2)}
    for name, g in graphs.items():
        store_graph(out, name, g)
        out[f"g_{name}_labels"] = g.labels.astype(np.int64)
    out["graph_names"] = np.array(list(graphs))
    meta, tvs, eps = [], [], []
    for gi, (name, g) in enumerate(graphs.items()):
        for kind, S, b, seed in (("prox", 1, 50, 0), ("prox", 3, 25, 1), ("prox", 4, 64, 2), ("rand", 0, 50, 3),
                                 ("rand", 0, 2000, 0)):
            sched = od.proximity_schedule(g, S, b, seed=seed) if kind == "prox" else \
                od.random_shuffle_schedule(g, b, seed=seed)
            rep = od.shuffling_error(sched, g.labels)
            meta.append((gi, 0 if kind == "prox" else 1, S, b, seed))
            tvs.append(rep.per_batch_tv)
            eps.append(rep.epsilon)
    sel = []
    for gi, (name, g) in enumerate(graphs.items()):
        for b, M, S_max, seed in ((50, 4, 8, 0), (250, 4, 10, 0), (25, 2, 5, 1)):
            S, rep = od.select_num_sequences(g, b, M, S_max, seed=seed)
            sel.append((gi, b, M, S_max, seed, S, int(rep.threshold_met)))
            eps.append(rep.epsilon)
    out["meta"] = np.array(meta, dtype=np.int64)
    put(out, "tvs", tvs, np.float64)
    out["eps"] = np.array(eps, dtype=np.float64)
    out["select"] = np.array(sel, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "shuffle.npz"), **out)


GRAPHGEN_SPECS = [  # (n, avg_degree, seed, train_fraction, num_labels, cross_fraction)
    (300, 6, 1, 0.1, 1, 0.05),
    (2000, 10, 2, 0.2, 3, 0.05),
    (12000, 9, 4, 0.05, 5, 0.05),      # choice(): tail shuffle branch (n > 10000, size > n // 50)
    (3000, 51, 5, 0.08, 4, 0.05),      # m = 26 (products' edges per node): set resizes 8 -> 32 -> 128
    (5000, 7, 9, 1.0, 2, 0.0),         # every node trains, no cross edges
    (15000, 4, 3, 0.3, 16, 0.2),
]


def make_graphgen():
    """gnnio.graph.generate_power_law outputs (graph.py:218-297) for the
    native generator (bgl_power_law_generate)."""
    out = {"specs": np.array([[n, d, s, nl] for n, d, s, _, nl, _ in GRAPHGEN_SPECS], dtype=np.int64),
           "fracs": np.array([[tf, cf] for _, _, _, tf, _, cf in GRAPHGEN_SPECS], dtype=np.float64)}
    for i, (n, d, seed, tf, nl, cf) in enumerate(GRAPHGEN_SPECS):
        g = generate_power_law(n, d, seed, train_fraction=tf, num_labels=nl, cross_fraction=cf)
        out[f"off_{i}"] = g.row_offsets.astype(np.int64)
        out[f"col_{i}"] = g.col_indices.astype(np.int32)
        out[f"train_{i}"] = np.packbits(g.train_mask)
        out[f"labels_{i}"] = g.labels.astype(np.int16)
    np.savez_compressed(os.path.join(HERE, "graphgen.npz"), **out)


def make_c1():
    """BASELINE.json configs[0], end to end by the reference itself:
    generate_power_law(100K, 20, seed=1, 0.1, 64) -> proximity_schedule(S=4,
    b=1024, seed=1) -> simulate_epoch([10, 5], seed=1) -> simulate(FIFO,
    10,000 device slots, d=1) with per-node outcomes."""
    g = generate_power_law(100_000, 20, seed=1, train_fraction=0.1, num_labels=64)
    sched = od.proximity_schedule(g, 4, 1024, seed=1)
    cfg = sp.SamplingConfig(fanouts=(10, 5), batch_size=1024, seed=1)
    trace, comm = sp.simulate_epoch(g, random_partition(g, 1), sched, cfg)
    rep = cs.simulate(trace, cs.CacheConfig(device_capacity=10_000, policy="fifo", feature_bytes_per_node=512),
                      record_outcomes=True)
    out = {"csr_entries": np.array([g.num_edges], dtype=np.int64)}
    put(out, "schedule", sched.batches, np.int32)
    put(out, "trace", trace.batches, np.int32)
    out["counters"] = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                                rep.batch_misses, rep.batch_insertions, rep.batch_evictions], dtype=np.int64).T
    put(out, "codes", [np.array(["DPHM".index(c) for c in o], dtype=np.uint8) for o in rep.outcomes], np.uint8)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)


def make_policies(gs):
    """compare_policies (cachesim.py:378-409) with its default policy set
    (POLICIES: static-degree, FIFO, LRU, LFU) + amortized_update_ops
    (:366-375) for the dynamic policies, on a sampled trace of the planted
    graph, d = 2 devices with a host level."""
    g = gs["dense"]
    sched = od.proximity_schedule(g, 2, 128, seed=3)
    trace, _ = sp.simulate_epoch(g, random_partition(g, 1), sched, sp.SamplingConfig(fanouts=(5, 3), seed=2))
    rows = cs.compare_policies(g, trace, [40, 150, 600], num_devices=2, host_capacity=100)
    amort = [cs.amortized_update_ops(cs.simulate(trace, cs.CacheConfig(device_capacity=150, host_capacity=100,
                                                                        num_devices=2, policy=p)))
             for p in ("fifo", "lru", "lfu")]
    out = {"rows": np.array([[list(cs.POLICIES).index(r["policy"]), r["capacity"], r["device_hits"],
                              r["host_hits"], r["misses"]] for r in rows], dtype=np.int64),
           "hit_ratio": np.array([r["hit_ratio"] for r in rows], dtype=np.float64),
           "amortized": np.array([[a[k] for k in ("lookups_per_batch", "insertions_per_batch",
                                                  "evictions_per_batch", "metadata_updates_per_batch")]
                                  for a in amort])}
    put(out, "trace", trace.batches, np.int32)
    np.savez_compressed(os.path.join(HERE, "policies.npz"), **out)


def make_c2(nbatches: int = 3):
    """BASELINE.json configs[1] (the bench workload) by the reference itself,
    for the first `nbatches` mini-batches: generate_power_law(2.4M, 51,
    seed=1, 0.08, 47) (~10 min in pure Python) -> proximity_schedule(S=4,
    b=1024, seed=1) -> sample_batch traces ([15, 10, 5], seed=1, batch_seed=i,
    as simulate_epoch keys them) -> simulate(FIFO, 240,000 slots) with
    per-node outcomes. Stores the graph's CSR size + a checksum, the schedule
    head, the traces, codes and counters."""
    g = generate_power_law(2_400_000, 51, seed=1, train_fraction=0.08, num_labels=47)
    sched = od.proximity_schedule(g, 4, 1024, seed=1)
    cfg = sp.SamplingConfig(fanouts=(15, 10, 5), batch_size=1024, seed=1)
    trace = sp.AccessTrace(batches=[sp.sample_batch(g, sched.batches[i], cfg, batch_seed=i)[1]
                                    for i in range(nbatches)])
    rep = cs.simulate(trace, cs.CacheConfig(device_capacity=240_000, policy="fifo", feature_bytes_per_node=400),
                      record_outcomes=True)
    col = g.col_indices.astype(np.int64)
    out = {"csr_entries": np.array([g.num_edges], dtype=np.int64),
           "csr_checksum": np.array([int((col * (np.arange(col.size) % 1000003 + 1)).sum() % (1 << 61))],
                                    dtype=np.int64),
           "offsets_tail": g.row_offsets[-1000:].astype(np.int64)}
    put(out, "schedule", sched.batches[:nbatches], np.int32)
    put(out, "trace", trace.batches, np.int32)
    out["counters"] = np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                                rep.batch_misses, rep.batch_insertions, rep.batch_evictions], dtype=np.int64).T
    put(out, "codes", [np.array(["DPHM".index(c) for c in o], dtype=np.uint8) for o in rep.outcomes], np.uint8)
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **out)


def digest(a) -> int:
    """Order-sensitive 61-bit polynomial digest of an int array (the C2 window
    fixture stores digests instead of ~30 MB of raw rows)."""
    a = np.asarray(a, dtype=np.int64).ravel()
    w = np.arange(a.size, dtype=np.int64) % 1000003 + 1
    return int(((a % (1 << 31)) * w).sum() % ((1 << 61) - 1))


_C2 = {}


def _c2_sample(i):
    g, sched, cfg = _C2["g"], _C2["sched"], _C2["cfg"]
    return sp.sample_batch(g, sched.batches[i], cfg, batch_seed=i)[1]


def make_c2_window(nbatches: int = 25, procs: int = 0):
    """The bench's whole default window (W=5 warm-up + K=20 timed batches of
    BASELINE.json configs[1]) by the reference itself: same graph / schedule /
    sampler / FIFO as make_c2 for batches 0..nbatches-1 (sample_batch over a
    process pool, batches are independent: SPEC.md:355), stored as per-batch
    sizes, sums and digests of the trace row and of the outcome codes, plus the
    counters and the ring's tail + a digest of its slots after the window."""
    import multiprocessing as mp
    g = generate_power_law(2_400_000, 51, seed=1, train_fraction=0.08, num_labels=47)
    sched = od.proximity_schedule(g, 4, 1024, seed=1)
    cfg = sp.SamplingConfig(fanouts=(15, 10, 5), batch_size=1024, seed=1)
    _C2.update(g=g, sched=sched, cfg=cfg)
    with mp.get_context("fork").Pool(procs or os.cpu_count()) as pool:
        batches = pool.map(_c2_sample, range(nbatches), chunksize=1)
    state = cs.cold_state(cs.CacheConfig(device_capacity=240_000, policy="fifo", feature_bytes_per_node=400))
    rep = cs.simulate(sp.AccessTrace(batches=batches),
                      cs.CacheConfig(device_capacity=240_000, policy="fifo", feature_bytes_per_node=400),
                      state=state, record_outcomes=True)
    codes = [np.array(["DPHM".index(c) for c in o], dtype=np.int64) for o in rep.outcomes]
    out = {"size": np.array([b.size for b in batches], dtype=np.int64),
           "sum": np.array([int(b.sum()) for b in batches], dtype=np.int64),
           "trace_digest": np.array([digest(b) for b in batches], dtype=np.int64),
           "codes_digest": np.array([digest(c) for c in codes], dtype=np.int64),
           "counters": np.array([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                                 rep.batch_misses, rep.batch_insertions, rep.batch_evictions], dtype=np.int64).T,
           "ring_tail": np.array([state.devices[0].tail], dtype=np.int64),
           "ring_digest": np.array([digest(state.devices[0].slots)], dtype=np.int64),
           "schedule_digest": np.array([digest(np.concatenate(sched.batches))], dtype=np.int64)}
    np.savez_compressed(os.path.join(HERE, "c2_window.npz"), **out)


def make_sparse():
    """Sparse / >= 2^31 int64 node IDs through gnnio's dict-based FIFO
    (cachesim.py:81-107, 275-363): each case draws its universe from a
    different ID range (just above 2^31, up to 2^40, up to 2^62, or dense IDs
    spread by a large stride), replays it batch by batch with a persistent
    state (every call grows the key set) and records codes, counters and the
    rings after every batch, plus the whole-trace call's counters."""
    rng = np.random.default_rng(7)
    out = {}
    specs, all_batches, all_codes, all_counters = [], [], [], []
    dev_slots, dev_tails, host_slots, host_tails, whole = [], [], [], [], []
    kinds = ["sorted", "unsorted", "dups"]
    ranges = [("above31", 2**31, 2**31 + 5000), ("p40", 0, 2**40), ("p62", 0, 2**62), ("stride", 0, 0)]
    for ci in range(16):
        kind = kinds[ci % 3]
        rname, lo, hi = ranges[ci % 4]
        usize = int(rng.integers(8, 300))
        if rname == "stride":
            universe = np.arange(usize, dtype=np.int64) * int(rng.integers(2**27, 2**29)) + int(rng.integers(0, 7))
        else:
            universe = np.unique(rng.integers(lo, hi, size=usize, dtype=np.int64))
        idx_batches = cache_case_batches(np.random.default_rng(1000 + ci), kind)
        batches = [universe[np.asarray(b) % universe.size] for b in idx_batches]
        if kind == "sorted":
            batches = [np.unique(b) for b in batches]
        d = int(rng.choice([1, 2, 3, 4, 8]))
        cap = int(rng.integers(0, 65))
        hcap = int(rng.choice([0, 1, 8, 64]))
        use_bd = ci % 4 == 3
        bd = [int(x) for x in rng.integers(d, size=len(batches))] if use_bd else None
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy="fifo",
                             feature_bytes_per_node=512)
        state = cs.cold_state(cfg)
        for i, b in enumerate(batches):
            rep = cs.simulate(AccessTrace(batches=[np.asarray(b, dtype=np.int64)]), cfg,
                              batch_devices=[bd[i] if bd else i % d], state=state, record_outcomes=True)
            all_codes.append(np.array(["DPHM".index(c) for c in rep.outcomes[0]], dtype=np.int64))
            all_counters.append([rep.batch_queries[0], rep.batch_own_hits[0], rep.batch_peer_hits[0],
                                 rep.batch_host_hits[0], rep.batch_misses[0], rep.batch_insertions[0],
                                 rep.batch_evictions[0], rep.batch_metadata_updates[0]])
            dev_slots.append(np.stack([lv.slots for lv in state.devices]).ravel())
            dev_tails.append([lv.tail for lv in state.devices])
            host_slots.append(state.host.slots.copy())
            host_tails.append([state.host.tail])
        rep = cs.simulate(AccessTrace(batches=[np.asarray(b, dtype=np.int64) for b in batches]), cfg,
                          batch_devices=bd)
        whole.append([sum(rep.batch_own_hits), sum(rep.batch_peer_hits), sum(rep.batch_host_hits),
                      sum(rep.batch_misses), sum(rep.batch_insertions), sum(rep.batch_evictions)])
        specs.append((d, cap, hcap, len(batches), int(use_bd), kinds.index(kind)))
        all_batches.extend(batches)
        out[f"bd_{ci}"] = np.array(bd if bd else [], dtype=np.int64)
    out["specs"] = np.array(specs, dtype=np.int64)
    out["whole"] = np.array(whole, dtype=np.int64)
    put(out, "batches", all_batches)
    put(out, "codes", all_codes, np.int8)
    out["counters"] = np.array(all_counters, dtype=np.int64)
    put(out, "dev_slots", dev_slots)
    put(out, "dev_tails", dev_tails)
    put(out, "host_slots", host_slots)
    put(out, "host_tails", host_tails)
    np.savez_compressed(os.path.join(HERE, "sparse.npz"), **out)


def make_ordered():
    """gnnio's LRU and LFU levels (cachesim.py:110-175) through simulate
    (cachesim.py:275-363), batch by batch on a persistent state: counters,
    codes, and every level after every batch -- LRU: `entries` in recency
    order; LFU: the residents in tick order with their `freq`, `tick_of` and
    the level's `tick`. Plus whole-trace counters of the desk-scale sampler
    trace for d = 1, 2, 4."""
    rng = np.random.default_rng(11)
    out = {}
    specs, all_batches, all_codes, all_counters = [], [], [], []
    logs, freqs, ticks, level_ticks = [], [], [], []
    kinds = ["sorted", "unsorted", "dups"]
    for ci in range(48):
        policy = ("lru", "lfu")[ci % 2]
        kind = kinds[(ci // 2) % 3]
        batches = cache_case_batches(rng, kind)
        d = int(rng.choice([1, 2, 3, 4, 8]))
        cap = int(rng.integers(0, 40))
        hcap = int(rng.choice([0, 1, 8, 30]))
        use_bd = ci % 5 == 4
        bd = [int(x) for x in rng.integers(d, size=len(batches))] if use_bd else None
        cfg = cs.CacheConfig(device_capacity=cap, host_capacity=hcap, num_devices=d, policy=policy,
                             feature_bytes_per_node=512)
        state = cs.cold_state(cfg)
        for i, b in enumerate(batches):
            rep = cs.simulate(AccessTrace(batches=[np.asarray(b, dtype=np.int64)]), cfg,
                              batch_devices=[bd[i] if bd else i % d], state=state, record_outcomes=True)
            all_codes.append(np.array(["DPHM".index(c) for c in rep.outcomes[0]], dtype=np.int64))
            all_counters.append([rep.batch_queries[0], rep.batch_own_hits[0], rep.batch_peer_hits[0],
                                 rep.batch_host_hits[0], rep.batch_misses[0], rep.batch_insertions[0],
                                 rep.batch_evictions[0], rep.batch_metadata_updates[0]])
            for lv in list(state.devices) + [state.host]:
                if policy == "lru":
                    logs.append(np.array(list(lv.entries.keys()), dtype=np.int64))
                    freqs.append(np.zeros(0, dtype=np.int64))
                    ticks.append(np.zeros(0, dtype=np.int64))
                    level_ticks.append(0)
                else:
                    order = sorted(lv.freq, key=lambda v: lv.tick_of[v])
                    logs.append(np.array(order, dtype=np.int64))
                    freqs.append(np.array([lv.freq[v] for v in order], dtype=np.int64))
                    ticks.append(np.array([lv.tick_of[v] for v in order], dtype=np.int64))
                    level_ticks.append(lv.tick)
        specs.append((d, cap, hcap, len(batches), int(use_bd), kinds.index(kind), ci % 2))
        all_batches.extend(batches)
        out[f"bd_{ci}"] = np.array(bd if bd else [], dtype=np.int64)
    out["specs"] = np.array(specs, dtype=np.int64)
    put(out, "batches", all_batches)
    put(out, "codes", all_codes, np.int8)
    out["counters"] = np.array(all_counters, dtype=np.int64)
    put(out, "logs", logs)
    put(out, "freqs", freqs)
    put(out, "ticks", ticks)
    out["level_ticks"] = np.array(level_ticks, dtype=np.int64)
    g = generate_power_law(5000, 10, seed=1, train_fraction=0.1, num_labels=16)
    sched = od.proximity_schedule(g, 4, 100, seed=1)
    trace, _ = sp.simulate_epoch(g, random_partition(g, 1, seed=0), sched,
                                 sp.SamplingConfig(fanouts=(10, 5), seed=1))
    put(out, "real_trace", trace.batches)
    real = []
    for policy in ("lru", "lfu"):
        for d in (1, 2, 4):
            rep = cs.simulate(trace, cs.CacheConfig(device_capacity=500 // d, host_capacity=250,
                                                    num_devices=d, policy=policy))
            real.append([rep.batch_queries, rep.batch_own_hits, rep.batch_peer_hits, rep.batch_host_hits,
                         rep.batch_misses, rep.batch_insertions, rep.batch_evictions, rep.batch_metadata_updates])
    out["real_counters"] = np.array(real, dtype=np.int64)   # [2 policies x 3 d, 8, nb]
    np.savez_compressed(os.path.join(HERE, "ordered.npz"), **out)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["sampler", "cache", "ordering", "static", "shuffle", "graphgen", "c1", "c2", "policies",
                             "c2_window", "sparse", "ordered"]
    gs = graphs()
    makers = {"sampler": lambda: make_sampler(gs), "cache": make_cache, "ordering": lambda: make_ordering(gs),
              "static": lambda: make_static(gs), "shuffle": lambda: make_shuffle(gs), "graphgen": make_graphgen,
              "c1": make_c1, "c2": make_c2, "policies": lambda: make_policies(gs), "c2_window": make_c2_window,
              "sparse": make_sparse, "ordered": make_ordered}
    for part in parts:
        makers[part]()
        f = part + ".npz"
        print(f, os.path.getsize(os.path.join(HERE, f)))
