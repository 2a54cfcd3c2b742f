"""Router oracle (oracle/moe_oracle.router_topk) on CPU: the definition the
GPU router is checked against bit-exactly.  The reference has no router
(routing.py:283-307 synthesises counts), so these pin the definition by
brute force and by the reference's router-output validation
(RoutingTable.validate, routing.py:146-163)."""

import numpy as np
import pytest

from oracle import moe_oracle as O
from paper_2502_19811_b200 import ModelConfig, ParallelSpec, RoutingTable, WorkloadSpec


def brute(row, k):
    def key(e):
        v = row[e]
        nan = np.isnan(v)
        return (1 if nan else 0, 0.0 if nan else -float(v) + 0.0, e)
    return sorted(sorted(range(len(row)), key=key)[:k])


@pytest.mark.parametrize("E,k", [(8, 2), (16, 2), (64, 8), (7, 7), (130, 3)])
def test_matches_brute_force_with_ties(E, k):
    rng = np.random.default_rng(E * 100 + k)
    lg = np.round(rng.standard_normal((200, E)) * 2) / 2  # many exact ties
    lg[0, :] = 0.0
    lg[1, ::2] = -0.0
    lg[2, 1] = np.nan
    lg[3, :] = -np.inf
    lg[3, E - 1] = np.nan
    ex, _ = O.router_topk(lg, k, None)
    for t in range(lg.shape[0]):
        assert list(ex[t]) == brute(lg[t], k), t


def test_output_is_a_valid_router_output():
    rng = np.random.default_rng(1)
    model = ModelConfig(L=1, E=64, topk=8, N=64, K=64)
    lg = rng.standard_normal((333, 64)).astype(np.float32)
    ex, w = O.router_topk(lg, 8, "topk")
    RoutingTable.from_array(model, ParallelSpec(1, 8), WorkloadSpec(M=333, seed=0, std=0.0), ex)  # validates
    np.testing.assert_allclose(w.sum(1), 1.0, rtol=1e-12)


def test_weight_modes():
    lg = np.array([[0.0, 1.0, 2.0, 3.0]])
    ex, w = O.router_topk(lg, 2, "topk")
    assert ex.tolist() == [[2, 3]]
    e2, e3 = np.exp(2.0), np.exp(3.0)
    np.testing.assert_allclose(w, [[e2 / (e2 + e3), e3 / (e2 + e3)]])
    _, wa = O.router_topk(lg, 2, "all")
    tot = np.exp(lg).sum()
    np.testing.assert_allclose(wa, [[e2 / tot, e3 / tot]])
