"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``moepipe`` from /root/reference/pkg/src (read-only; nothing is
copied) and writes small fixtures next to this file.  The GPU box never runs
this script; tests there only read the committed outputs.

Fixtures
--------
routing_cases.json   full RoutingTable JSON for small seeded workloads, plus
                     digests (sha256 of experts_per_token, counts, transfer
                     matrix) for the bench-scale workloads.
schedules.json       per-rank sort_tokens_by_source layout and
                     resolve_layer0 / resolve_layer1 schedules (reference
                     TileSchedule.to_json_dict) for small instances drawn like
                     the reference's random_instance (test_resolver.py:38-63).
index_<name>.npz     bench-scale per-rank layouts and tile lists (flat int
                     arrays) from the reference resolver, for the bit-exact
                     GPU index-build tests at full size.
layer_small.npz      fp64 execute_naive / execute_scheduled /
                     execute_tp_sharded outputs on small instances (identity,
                     tanh activation, combine weights).
layer_c1.npz         Config 1 (E8 top2 M512 N512 K1024 EP8) execute_naive
                     output (stored float32) + digests of its inputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import moepipe as R  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a)).tobytes()).hexdigest()


def flat_index(routing, rank, tile_rows, tile_cols):
    m0 = R.meta_for_layer0(routing.model, routing.workload, tile_rows)
    m1 = R.meta_for_layer1(routing.model, routing.workload, tile_rows, tile_cols)
    s0 = R.resolve_layer0(routing, rank, m0)
    s1 = R.resolve_layer1(routing, rank, m1)
    lay = s0.layout
    hosted = sorted(lay)
    rows = [r for e in hosted for r in lay[e]]
    counts = [len(lay[e]) for e in hosted]
    out = {
        "row_offsets": np.concatenate([[0], np.cumsum(counts)]).astype(np.int64),
        "row_token": np.array([t for t, _ in rows], dtype=np.int64),
        "row_src": np.array([s for _, s in rows], dtype=np.int64),
        "n_local": np.array([sum(1 for _, s in lay[e] if s == rank) for e in hosted], np.int64),
        "tiles0": np.array([(t.expert, t.row_start, t.row_stop, len(t.deps)) for t in s0.tiles],
                           dtype=np.int64).reshape(-1, 4),
        "tiles1": np.array([(t.expert, t.row_start, t.row_stop, t.col_start, t.col_stop, len(t.deps))
                            for t in s1.tiles], dtype=np.int64).reshape(-1, 6),
        "chunks": np.array([(c.col_start, c.col_stop, min(c.prereq_tile_ids, default=0),
                             len(c.prereq_tile_ids)) for c in s1.reduce_chunks],
                           dtype=np.int64).reshape(-1, 4),
        "expert_counts": np.array(routing.expert_counts, dtype=np.int64),
        "transfer_counts": np.array(routing.transfer_counts, dtype=np.int64),
    }
    # prereq sets must be contiguous id ranges for the flat form to be lossless
    for c in s1.reduce_chunks:
        ids = sorted(c.prereq_tile_ids)
        assert ids == list(range(ids[0], ids[0] + len(ids))) if ids else True
    return out


def random_instance(seed, max_m=64, e_choices=(1, 2, 3, 4, 8)):
    """Same draw as the reference test helper (test_resolver.py:38-63)."""
    rng = np.random.default_rng(seed)
    e_count = int(rng.choice(e_choices))
    topk = int(rng.integers(1, e_count + 1))
    tp = int(rng.choice([1, 2]))
    ep = int(rng.choice([d for d in (1, 2, 4) if e_count % d == 0]))
    k_hidden = int(rng.choice([4, 8, 16])) * tp
    n_embed = int(rng.choice([4, 8, 16]))
    model = R.ModelConfig(L=1, E=e_count, topk=topk, N=n_embed, K=k_hidden)
    par = R.ParallelSpec(tp=tp, ep=ep)
    m_tokens = int(rng.integers(0, max_m + 1))
    target = float(rng.uniform(0, R.max_achievable_std(e_count, topk)))
    wl = R.WorkloadSpec(M=m_tokens, seed=int(rng.integers(0, 2**31)), std=target)
    routing = R.build_routing(model, par, wl)
    tile_rows = int(rng.choice([1, 2, 4, 8]))
    tile_cols = int(rng.integers(1, n_embed + 1))
    rank = int(rng.integers(0, par.world_size))
    return routing, rank, tile_rows, tile_cols


def routing_cases():
    cases = []
    rng = np.random.default_rng(2024)
    for i in range(40):
        E = int(rng.integers(1, 13))
        topk = int(rng.integers(1, E + 1))
        ep = int(rng.choice([d for d in (1, 2, 4) if E % d == 0]))
        tp = int(rng.choice([1, 2]))
        M = int(rng.integers(0, 130))
        std = float(rng.uniform(0, 1)) * R.max_achievable_std(E, topk)
        model = R.ModelConfig(L=1, E=E, topk=topk, N=8, K=8 * tp)
        r = R.build_routing(model, R.ParallelSpec(tp, ep), R.WorkloadSpec(M=M, seed=int(rng.integers(0, 2**31)), std=std))
        cases.append({"table": r.to_json_dict(), "expert_counts": list(r.expert_counts),
                      "transfer_counts": [list(x) for x in r.transfer_counts],
                      "sources": [r.source_rank_of(t) for t in range(M)]})
    return cases


BENCH = {
    # name: (E, topk, N, K, M, std, tp, ep)
    "c1": (8, 2, 512, 1024, 512, 0.0, 1, 8),
    "mx_ep8": (8, 2, 4096, 14336, 8192, 0.0, 1, 8),
    "mx_ep8_s032": (8, 2, 4096, 14336, 8192, 0.032, 1, 8),
    "mx_ep8_s05": (8, 2, 4096, 14336, 8192, 0.05, 1, 8),
    "mx_ep1": (8, 2, 4096, 14336, 8192, 0.0, 1, 1),
    "mx_ep1_s032": (8, 2, 4096, 14336, 8192, 0.032, 1, 1),
    "ph_tp2ep4_s032": (16, 2, 4096, 6400, 8192, 0.032, 2, 4),
    "qw_ep8_s032": (64, 8, 3584, 2560, 8192, 0.032, 1, 8),
}


def bench_digests():
    out = {}
    for name, (E, topk, N, K, M, std, tp, ep) in BENCH.items():
        model = R.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
        r = R.build_routing(model, R.ParallelSpec(tp, ep), R.WorkloadSpec(M=M, seed=0, std=std))
        arr = np.array(r.experts_per_token, dtype=np.int32).reshape(M, topk)
        out[name] = {"shape": [E, topk, N, K, M, std, tp, ep],
                     "experts_sha256": digest(arr),
                     "expert_counts": list(r.expert_counts),
                     "transfer_counts": [list(x) for x in r.transfer_counts],
                     "achieved_std": r.achieved_std}
    return out


def schedules():
    recs = []
    for seed in range(60):
        routing, rank, tile_rows, tile_cols = random_instance(1000 + seed)
        m0 = R.meta_for_layer0(routing.model, routing.workload, tile_rows)
        m1 = R.meta_for_layer1(routing.model, routing.workload, tile_rows, tile_cols)
        s0 = R.resolve_layer0(routing, rank, m0)
        s1 = R.resolve_layer1(routing, rank, m1)
        layout = R.sort_tokens_by_source(routing, rank)
        recs.append({
            "routing": routing.to_json_dict(), "rank": rank,
            "tile_rows": tile_rows, "tile_cols": tile_cols,
            "layout": {str(e): [list(r) for r in rows] for e, rows in layout.items()},
            "layer0": s0.to_json_dict(), "layer1": s1.to_json_dict(),
        })
    return recs


def bench_indices():
    for name in ("c1", "mx_ep8_s032", "mx_ep1_s032", "ph_tp2ep4_s032", "qw_ep8_s032"):
        E, topk, N, K, M, std, tp, ep = BENCH[name]
        model = R.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
        r = R.build_routing(model, R.ParallelSpec(tp, ep), R.WorkloadSpec(M=M, seed=0, std=std))
        tc = R.default_tile_cols(N)
        world = tp * ep
        ranks = sorted({0, world // 2, world - 1} | ({1} if world > 1 else set()))
        payload = {"meta": np.array([E, topk, N, K, M, tp, ep, 128, tc], dtype=np.int64),
                   "ranks": np.array(ranks, dtype=np.int64)}
        for rank in ranks:
            for k, v in flat_index(r, rank, 128, tc).items():
                payload[f"r{rank}_{k}"] = v
        np.savez_compressed(os.path.join(HERE, f"index_{name}.npz"), **payload)


def layer_small():
    payload = {}
    specs = [  # name, E, topk, N, K, M, tp, ep, seed, activation, weighted
        ("id_e3", 3, 2, 4, 8, 6, 1, 1, 5, None, False),
        ("id_e4_ep2", 4, 2, 32, 48, 64, 1, 2, 7, None, False),
        ("tanh_e4", 4, 2, 32, 48, 64, 1, 2, 8, "tanh", False),
        ("w_e8", 8, 2, 64, 96, 40, 1, 4, 9, None, True),
        ("tanh_w_e8_top3", 8, 3, 48, 64, 50, 1, 2, 10, "tanh", True),
        ("tp2_e4", 4, 2, 32, 64, 48, 2, 2, 11, None, False),
        ("tp2_tanh_w", 4, 2, 32, 64, 48, 2, 1, 12, "tanh", True),
    ]
    for name, E, topk, N, K, M, tp, ep, seed, act, weighted in specs:
        model = R.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
        par = R.ParallelSpec(tp=tp, ep=ep)
        wl = R.WorkloadSpec(M=M, seed=seed, std=0.0)
        routing = R.build_routing(model, par, wl)
        x = np.random.default_rng(seed + 1).standard_normal((M, N))
        w = R.random_weights(model, seed=seed + 2)
        cw = np.random.default_rng(3).random((M, topk)) if weighted else None
        fn = np.tanh if act == "tanh" else None
        if tp == 1:
            y = R.execute_naive(x, w, routing, activation=fn, combine_weights=cw)
            m0 = R.meta_for_layer0(model, wl, 4)
            m1 = R.meta_for_layer1(model, wl, 4, max(1, N // 4))
            s0 = [R.resolve_layer0(routing, g * tp, m0) for g in range(ep)]
            s1 = [R.resolve_layer1(routing, g * tp, m1) for g in range(ep)]
            ys = R.execute_scheduled(x, w, routing, s0, s1, activation=fn, combine_weights=cw)
            assert np.array_equal(y, ys)
        else:
            y = R.execute_tp_sharded(x, w, routing, tp, activation=fn, combine_weights=cw)
        payload[f"{name}__spec"] = np.array([E, topk, N, K, M, tp, ep, seed, int(weighted)], np.int64)
        payload[f"{name}__act"] = np.array(act or "none")
        payload[f"{name}__experts"] = np.array(routing.experts_per_token, np.int64).reshape(M, topk)
        payload[f"{name}__x"] = x
        payload[f"{name}__w0"] = w.w0
        payload[f"{name}__w1"] = w.w1
        if cw is not None:
            payload[f"{name}__cw"] = cw
        payload[f"{name}__y"] = y
    np.savez_compressed(os.path.join(HERE, "layer_small.npz"), **payload)


def layer_c1():
    E, topk, N, K, M, std, tp, ep = BENCH["c1"]
    model = R.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    wl = R.WorkloadSpec(M=M, seed=0, std=std)
    routing = R.build_routing(model, R.ParallelSpec(tp, ep), wl)
    x = np.random.default_rng(1).standard_normal((M, N))
    w = R.random_weights(model, seed=2)
    y = R.execute_naive(x, w, routing)
    np.savez_compressed(os.path.join(HERE, "layer_c1.npz"),
                        y=y.astype(np.float32),
                        x_sha256=np.array(digest(x)), w0_sha256=np.array(digest(w.w0)),
                        w1_sha256=np.array(digest(w.w1)),
                        experts=np.array(routing.experts_per_token, np.int16).reshape(M, topk))


def main():
    with open(os.path.join(HERE, "routing_cases.json"), "w") as f:
        json.dump({"cases": routing_cases(), "bench": bench_digests()}, f, sort_keys=True)
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump({"instances": schedules()}, f, sort_keys=True)
    bench_indices()
    layer_small()
    layer_c1()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
