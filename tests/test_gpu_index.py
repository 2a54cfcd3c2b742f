"""GPU index build (moe_index_build) vs the reference resolver: bit-exact.

Fixtures come from the reference package itself (tests/golden/); random
instances are checked against the oracle restatement, which is pinned to
the reference by tests/test_oracle_golden.py."""

import json
import os
from dataclasses import replace

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import moe_oracle as O
from paper_2502_19811_b200 import (ConfigurationError, ModelConfig, ParallelSpec, RoutingTable, WorkloadSpec,
                                   build_routing, device_index, max_achievable_std, meta_for_layer0,
                                   meta_for_layer1, resolve_layer0, resolve_layer1, sort_tokens_by_source,
                                   validate_schedule)
from paper_2502_19811_b200.resolver import N_DIM, ReduceChunk, SharedTensorMeta

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ("expert_counts", "transfer_counts", "row_offsets", "row_token", "row_src", "n_local", "tiles0",
        "tiles1", "chunks")


@pytest.mark.parametrize("name", ["c1", "mx_ep8_s032", "mx_ep1_s032", "ph_tp2ep4_s032", "qw_ep8_s032"])
def test_index_bit_exact_vs_reference_bench_scale(name):
    z = np.load(os.path.join(GOLD, f"index_{name}.npz"))
    E, topk, N, K, M, tp, ep, tr, tc = z["meta"].tolist()
    r = build_routing(ModelConfig(L=1, E=E, topk=topk, N=N, K=K), ParallelSpec(tp, ep),
                      WorkloadSpec(M=M, seed=0, std=0.0 if name == "c1" else 0.032))
    for rank in z["ranks"].tolist():
        got = device_index(r, rank, tr, tc)
        for k in KEYS:
            np.testing.assert_array_equal(got[k], z[f"r{rank}_{k}"], err_msg=f"{name} rank {rank} {k}")


def test_schedules_match_reference_json_small_instances():
    insts = json.load(open(os.path.join(GOLD, "schedules.json")))["instances"]
    for inst in insts:
        r = RoutingTable.from_json_dict(inst["routing"])
        rank, tr, tc = inst["rank"], inst["tile_rows"], inst["tile_cols"]
        assert {str(e): [list(x) for x in rows] for e, rows in sort_tokens_by_source(r, rank).items()} == inst["layout"]
        s0 = resolve_layer0(r, rank, meta_for_layer0(r.model, r.workload, tr))
        s1 = resolve_layer1(r, rank, meta_for_layer1(r.model, r.workload, tr, tc))
        assert s0.to_json_dict() == inst["layer0"]
        assert s1.to_json_dict() == inst["layer1"]
        assert validate_schedule(s0, r) == [] and validate_schedule(s1, r) == []


def random_instance(seed, max_m=64, e_choices=(1, 2, 3, 4, 8)):
    """The reference's generator (test_resolver.py:38-63)."""
    rng = np.random.default_rng(seed)
    e_count = int(rng.choice(e_choices))
    topk = int(rng.integers(1, e_count + 1))
    tp = int(rng.choice([1, 2]))
    ep = int(rng.choice([d for d in (1, 2, 4) if e_count % d == 0]))
    model = ModelConfig(L=1, E=e_count, topk=topk, N=int(rng.choice([4, 8, 16])), K=int(rng.choice([4, 8, 16])) * tp)
    par = ParallelSpec(tp=tp, ep=ep)
    wl = WorkloadSpec(M=int(rng.integers(0, max_m + 1)), seed=int(rng.integers(0, 2**31)),
                      std=float(rng.uniform(0, max_achievable_std(e_count, topk))))
    routing = build_routing(model, par, wl)
    tile_rows = int(rng.choice([1, 2, 4, 8]))
    tile_cols = int(rng.integers(1, model.N + 1))
    return routing, int(rng.integers(0, par.world_size)), tile_rows, tile_cols


@settings(max_examples=60, deadline=None)
@given(seed=st.integers(0, 100_000))
def test_index_matches_oracle_random_instances(seed):
    r, rank, tr, tc = random_instance(seed, max_m=200)
    got = device_index(r, rank, tr, tc)
    want = O.index_for_rank(r.as_array(), r.model.E, r.parallel.tp, r.parallel.ep, rank, tr, tc, r.model.N)
    for k in KEYS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)


@settings(max_examples=40, deadline=None)
@given(seed=st.integers(0, 10_000))
def test_layer0_prefix_locality_and_layer1_waves(seed):  # test_resolver.py:171-178, 232-242
    r, rank, tr, tc = random_instance(seed)
    s0 = resolve_layer0(r, rank, meta_for_layer0(r.model, r.workload, tr))
    deps = [len(t.deps) for t in s0.tiles]
    assert deps == sorted(deps) and validate_schedule(s0, r) == []
    s1 = resolve_layer1(r, rank, meta_for_layer1(r.model, r.workload, tr, tc))
    assert [t.col_start for t in s1.tiles] == sorted(t.col_start for t in s1.tiles)
    assert validate_schedule(s1, r) == []


def hand_routing(model, par, rows):
    t = RoutingTable(model=model, parallel=par, workload=WorkloadSpec(M=len(rows)),
                     experts_per_token=tuple(tuple(sorted(a)) for a in rows), achieved_std=0.0)
    t.validate()
    return t


def test_known_answers():  # test_resolver.py:131-141, 163-168, 186-195, 208-222
    m = ModelConfig(L=1, E=2, topk=1, N=4, K=4)
    r = hand_routing(m, ParallelSpec(1, 2), [(0,)] * 8)
    s = resolve_layer0(r, 0, meta_for_layer0(m, r.workload, 4))
    assert len(s.tiles) == 2 and s.tiles[0].deps == frozenset()
    assert s.tiles[0].rows == ((0, 0), (1, 0), (2, 0), (3, 0))
    assert s.tiles[1].deps == frozenset({(4, 1), (5, 1), (6, 1), (7, 1)})
    r = hand_routing(m, ParallelSpec(), [(0,)] * 5)
    s = resolve_layer0(r, 0, meta_for_layer0(m, r.workload, 4))
    assert [len(t.rows) for t in s.tiles] == [4, 1]
    m2 = ModelConfig(L=1, E=2, topk=2, N=4, K=4)
    r = hand_routing(m2, ParallelSpec(), [(0, 1)] * 3)
    s = resolve_layer1(r, 0, meta_for_layer1(m2, r.workload, tile_rows=8, tile_cols=2))
    assert [(t.expert, t.col_start) for t in s.tiles] == [(0, 0), (1, 0), (0, 2), (1, 2)]
    assert [c.prereq_tile_ids for c in s.reduce_chunks] == [frozenset({0, 1}), frozenset({2, 3})]
    m3 = ModelConfig(L=1, E=3, topk=3, N=8, K=4)
    r = hand_routing(m3, ParallelSpec(), [(0, 1, 2)] * 4)
    s = resolve_layer1(r, 0, meta_for_layer1(m3, r.workload, tile_rows=8, tile_cols=2))
    assert len(s.reduce_chunks) == 4
    with pytest.raises(ConfigurationError):
        resolve_layer0(r, 0, SharedTensorMeta(global_rows=4, cols=8, decomposed_dim=N_DIM, tile_cols=2))
    with pytest.raises(ConfigurationError):
        resolve_layer1(r, 0, meta_for_layer0(m3, r.workload))
    with pytest.raises(ConfigurationError):
        sort_tokens_by_source(build_routing(m, ParallelSpec(), WorkloadSpec(M=4)), 1)


def test_validator_mutations():  # test_resolver.py:265-311
    seed = 123
    while True:
        r, rank, tr, tc = random_instance(seed, max_m=40)
        s0 = resolve_layer0(r, rank, meta_for_layer0(r.model, r.workload, tr))
        s1 = resolve_layer1(r, rank, meta_for_layer1(r.model, r.workload, tr, tc))
        if s0.tiles and len(s1.reduce_chunks) >= 2 and s1.reduce_chunks[0].prereq_tile_ids:
            break
        seed += 1
    codes = lambda s: {v.code for v in validate_schedule(s, r)}  # noqa: E731
    assert "missing-tile" in codes(replace(s0, tiles=s0.tiles[1:]))
    assert "duplicate-tile" in codes(replace(s0, tiles=s0.tiles + (s0.tiles[0],)))
    v = s0.tiles[0]
    assert "bad-deps" in codes(replace(s0, tiles=(replace(v, deps=v.deps | {(v.rows[0][0], 999)}),) + s0.tiles[1:]))
    c = s1.reduce_chunks[0]
    starved = ReduceChunk(c.chunk_id, c.col_start, c.col_stop, frozenset(list(c.prereq_tile_ids)[1:]))
    assert "premature-reduce" in codes(replace(s1, reduce_chunks=(starved,) + s1.reduce_chunks[1:]))
    swapped = (s1.reduce_chunks[1], s1.reduce_chunks[0]) + s1.reduce_chunks[2:]
    assert "reduce-order" in codes(replace(s1, reduce_chunks=swapped))
