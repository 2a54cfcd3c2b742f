"""Host-side mirror of the reference config/routing tests
(pkg/tests/test_config.py, pkg/tests/test_routing.py) run against this
package's config/routing modules.  No GPU needed."""

import json
import math

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2502_19811_b200 import (
    MODEL_PRESETS, ConfigurationError, InfeasibleStdError, ModelConfig, ParallelSpec, RoutingTable,
    WorkloadSpec, buffer_bytes, build_routing, expert_placement, experts_on_rank, fraction_std,
    max_achievable_std, model_preset, validate_sharding)

MIB = 1024 * 1024


def recount(table):
    counts = [0] * table.model.E
    for row in table.experts_per_token:
        for e in row:
            counts[e] += 1
    return counts


def test_presets_match_published_shapes():  # test_config.py:24-34
    m = model_preset("mixtral-8x7b")
    assert (m.L, m.E, m.topk, m.N, m.K) == (32, 8, 2, 4096, 14336)
    q = model_preset("qwen2-moe")
    assert (q.L, q.E, q.topk, q.N, q.K) == (24, 64, 4, 2048, 1408)
    p = model_preset("phi-3.5-moe")
    assert (p.L, p.E, p.topk, p.N, p.K) == (32, 16, 2, 4096, 6400)
    assert all(v.dtype_bytes == 2 for v in MODEL_PRESETS.values())
    with pytest.raises(ConfigurationError):
        model_preset("mixtral-9x9b")


@pytest.mark.parametrize("field,value", [("L", 0), ("E", 0), ("topk", 0), ("topk", 9), ("N", 0),
                                         ("K", 0), ("dtype_bytes", 3)])
def test_model_invariants(field, value):
    base = dict(L=1, E=8, topk=2, N=16, K=32, dtype_bytes=2)
    base[field] = value
    with pytest.raises(ConfigurationError):
        ModelConfig(**base)


def test_placement_examples():  # test_config.py:59-88
    assert expert_placement(ModelConfig(L=1, E=4, topk=2, N=8, K=8), ParallelSpec(1, 2)) == \
        {0: (0,), 1: (0,), 2: (1,), 3: (1,)}
    model = ModelConfig(L=1, E=8, topk=2, N=8, K=8)
    assert expert_placement(model, ParallelSpec(tp=2, ep=4)) == {e: (2 * (e // 2), 2 * (e // 2) + 1) for e in range(8)}
    with pytest.raises(ConfigurationError):
        expert_placement(ModelConfig(L=1, E=6, topk=2, N=8, K=8), ParallelSpec(tp=1, ep=4))
    with pytest.raises(ConfigurationError):
        validate_sharding(ModelConfig(L=1, E=4, topk=2, N=8, K=6), ParallelSpec(tp=4, ep=1))


@given(ep=st.integers(1, 8), tp=st.integers(1, 4), per_group=st.integers(1, 4))
def test_placement_totality(ep, tp, per_group):  # test_config.py:91-108
    model = ModelConfig(L=1, E=ep * per_group, topk=1, N=8, K=tp * 4)
    par = ParallelSpec(tp=tp, ep=ep)
    placement = expert_placement(model, par)
    covered = set()
    for ranks in placement.values():
        assert len(ranks) == tp
        covered.update(ranks)
    assert covered == set(range(par.world_size))
    for rank in range(par.world_size):
        assert [e for e, r in placement.items() if rank in r] == list(experts_on_rank(model, par, rank))


@pytest.mark.parametrize("preset,m,mib", [("mixtral-8x7b", 4096, 32), ("mixtral-8x7b", 8192, 64),
                                          ("qwen2-moe", 4096, 16), ("qwen2-moe", 8192, 32),
                                          ("phi-3.5-moe", 4096, 32), ("phi-3.5-moe", 8192, 64)])
def test_buffer_bytes_published_table(preset, m, mib):  # test_config.py:111-124
    assert buffer_bytes(model_preset(preset), m) == mib * MIB


def test_json_round_trips():
    model = ModelConfig(L=2, E=4, topk=2, N=8, K=16, dtype_bytes=4)
    assert model.to_json_dict() == {"L": 2, "E": 4, "topk": 2, "N": 8, "K": 16, "dtype_bytes": 4}
    assert ModelConfig.from_json_dict(json.loads(json.dumps(model.to_json_dict()))) == model
    par = ParallelSpec(tp=2, ep=4)
    assert ParallelSpec.from_json_dict(par.to_json_dict()) == par
    wl = WorkloadSpec(M=128, seed=3, std=0.25)
    assert WorkloadSpec.from_json_dict(wl.to_json_dict()) == wl
    with pytest.raises(ConfigurationError):
        WorkloadSpec(M=-1)


def test_uniform_routing_is_exactly_even():  # test_routing.py:36-40
    t = build_routing(model_preset("mixtral-8x7b"), ParallelSpec(tp=1, ep=8), WorkloadSpec(M=8192))
    assert recount(t) == [2048] * 8 and t.achieved_std == 0.0


def test_skewed_routing_hits_target():  # test_routing.py:50-59
    t = build_routing(ModelConfig(L=1, E=8, topk=2, N=8, K=16), ParallelSpec(),
                      WorkloadSpec(M=8192, seed=42, std=0.05))
    assert 0.049 <= fraction_std(recount(t)) <= 0.051


def test_infeasible_std():  # test_routing.py:94-99
    with pytest.raises(InfeasibleStdError) as err:
        build_routing(ModelConfig(L=1, E=8, topk=2, N=8, K=16), ParallelSpec(), WorkloadSpec(M=128, std=0.9))
    assert math.isclose(err.value.achievable, math.sqrt(3) / 8)


def test_source_ranks_and_transfer_counts():  # test_routing.py:128-149
    t = build_routing(ModelConfig(L=1, E=8, topk=2, N=8, K=16), ParallelSpec(tp=1, ep=4), WorkloadSpec(M=10))
    assert [t.source_rank_of(i) for i in range(10)] == [0, 0, 1, 1, 2, 2, 3, 3, 3, 3]
    assert t.token_range_of_rank(3) == (6, 10)
    t = build_routing(ModelConfig(L=1, E=4, topk=2, N=8, K=16), ParallelSpec(tp=2, ep=2), WorkloadSpec(M=40, seed=4))
    expected = [[0] * 4 for _ in range(4)]
    for tok, row in enumerate(t.experts_per_token):
        for e in row:
            for dst in ((0, 1) if e < 2 else (2, 3)):
                expected[min(tok // 10, 3)][dst] += 1
    assert [list(r) for r in t.transfer_counts] == expected


def test_m_less_than_world_puts_everything_on_last_rank():
    t = build_routing(ModelConfig(L=1, E=4, topk=1, N=8, K=8), ParallelSpec(tp=1, ep=4), WorkloadSpec(M=3))
    assert [t.source_rank_of(i) for i in range(3)] == [3, 3, 3]


def test_json_round_trip_and_array_view():
    t = build_routing(ModelConfig(L=1, E=8, topk=2, N=8, K=16), ParallelSpec(tp=1, ep=2),
                      WorkloadSpec(M=64, seed=2, std=0.02))
    assert RoutingTable.from_json_dict(t.to_json_dict()) == t
    arr = t.as_array()
    assert arr.dtype == np.int32 and arr.shape == (64, 2)
    assert np.all(np.diff(arr, axis=1) > 0)


@settings(max_examples=60, deadline=None)
@given(e_count=st.integers(1, 12), data=st.data(), m_tokens=st.integers(0, 120),
       seed=st.integers(0, 2**32 - 1))
def test_conservation_and_distinctness(e_count, data, m_tokens, seed):  # test_routing.py:152-170
    topk = data.draw(st.integers(1, e_count))
    target = data.draw(st.floats(0.0, 1.0)) * max_achievable_std(e_count, topk)
    t = build_routing(ModelConfig(L=1, E=e_count, topk=topk, N=4, K=4), ParallelSpec(),
                      WorkloadSpec(M=m_tokens, seed=seed, std=target))
    counts = recount(t)
    assert sum(counts) == m_tokens * topk and max(counts, default=0) <= m_tokens
    for row in t.experts_per_token:
        assert len(set(row)) == topk and list(row) == sorted(row)
