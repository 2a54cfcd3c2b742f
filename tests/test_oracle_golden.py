"""Pin the CPU oracle (oracle/moe_oracle.py) and the host routing generator
against fixtures produced by the reference package itself
(tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from oracle import moe_oracle as O
from paper_2502_19811_b200 import config as C
from paper_2502_19811_b200 import routing as Rt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load_json(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _table(d):
    return Rt.RoutingTable.from_json_dict(d)


def test_routing_generator_reproduces_reference_tables():
    cases = _load_json("routing_cases.json")["cases"]
    assert len(cases) >= 40
    for case in cases:
        ref = _table(case["table"])
        mine = Rt.build_routing(ref.model, ref.parallel, ref.workload)
        assert mine.to_json_dict() == case["table"]
        assert list(mine.expert_counts) == case["expert_counts"]
        assert [list(r) for r in mine.transfer_counts] == case["transfer_counts"]
        assert [mine.source_rank_of(t) for t in range(ref.workload.M)] == case["sources"]


@pytest.mark.parametrize("name", sorted(_load_json("routing_cases.json")["bench"]))
def test_routing_generator_bench_digests(name):
    import hashlib
    d = _load_json("routing_cases.json")["bench"][name]
    E, topk, N, K, M, std, tp, ep = d["shape"]
    r = Rt.build_routing(C.ModelConfig(L=1, E=E, topk=topk, N=N, K=K),
                         C.ParallelSpec(tp, ep), C.WorkloadSpec(M=M, seed=0, std=std))
    assert hashlib.sha256(r.as_array().tobytes()).hexdigest() == d["experts_sha256"]
    assert list(r.expert_counts) == d["expert_counts"]
    assert [list(x) for x in r.transfer_counts] == d["transfer_counts"]
    assert r.achieved_std == d["achieved_std"]


def test_oracle_counts_match_routing_cases():
    for case in _load_json("routing_cases.json")["cases"]:
        t = _table(case["table"])
        ex = t.as_array()
        assert list(O.expert_counts(ex, t.model.E)) == case["expert_counts"]
        tc = O.transfer_counts(ex, t.model.E, t.parallel.tp, t.parallel.ep)
        assert tc.tolist() == case["transfer_counts"]
        assert O.source_ranks(t.workload.M, t.parallel.world_size).tolist() == case["sources"]


def test_oracle_schedules_match_reference_small_instances():
    insts = _load_json("schedules.json")["instances"]
    for inst in insts:
        t = _table(inst["routing"])
        rank, tr, tc = inst["rank"], inst["tile_rows"], inst["tile_cols"]
        lay = O.sort_layout(t.as_array(), t.model.E, t.parallel.tp, t.parallel.ep, rank)
        assert {str(e): rows.tolist() for e, rows in lay.items()} == inst["layout"]
        t0 = O.layer0_tiles(lay, rank, tr)
        ref0 = inst["layer0"]["tiles"]
        assert [[e, a, b] for e, a, b, _ in t0.tolist()] == [[x["expert"]] + x["rows"] for x in ref0]
        assert [nd for *_, nd in t0.tolist()] == [len(x["deps"]) for x in ref0]
        t1, ch = O.layer1_tiles(lay, rank, tr, tc, t.model.N)
        ref1 = inst["layer1"]["tiles"]
        assert [[e, a, b, c0, c1] for e, a, b, c0, c1, _ in t1.tolist()] == \
            [[x["expert"]] + x["rows"] + x["cols"] for x in ref1]
        assert [x["tile_id"] for x in ref1] == list(range(len(ref1)))
        refc = inst["layer1"]["reduce_chunks"]
        assert len(ch) == len(refc)
        for (c0, c1, first, n), rc in zip(ch.tolist(), refc):
            assert [c0, c1] == rc["cols"]
            assert list(range(first, first + n)) == rc["prereq_tile_ids"]


@pytest.mark.parametrize("name", ["c1", "mx_ep8_s032", "mx_ep1_s032", "ph_tp2ep4_s032", "qw_ep8_s032"])
def test_oracle_index_matches_reference_bench_scale(name):
    z = np.load(os.path.join(GOLD, f"index_{name}.npz"))
    E, topk, N, K, M, tp, ep, tr, tc = z["meta"].tolist()
    std = {"c1": 0.0}.get(name, 0.032)
    r = Rt.build_routing(C.ModelConfig(L=1, E=E, topk=topk, N=N, K=K),
                         C.ParallelSpec(tp, ep), C.WorkloadSpec(M=M, seed=0, std=std))
    for rank in z["ranks"].tolist():
        got = O.index_for_rank(r.as_array(), E, tp, ep, rank, tr, tc, N)
        for key, val in got.items():
            np.testing.assert_array_equal(val, z[f"r{rank}_{key}"], err_msg=f"{name} r{rank} {key}")


def _small_cases():
    z = np.load(os.path.join(GOLD, "layer_small.npz"))
    names = sorted({k.split("__")[0] for k in z.files})
    return z, names


def test_oracle_layer_forward_matches_reference_fp64():
    z, names = _small_cases()
    for name in names:
        E, topk, N, K, M, tp, ep, seed, weighted = z[f"{name}__spec"].tolist()
        act = str(z[f"{name}__act"])
        fn = np.tanh if act == "tanh" else None
        cw = z[f"{name}__cw"] if weighted else None
        args = (z[f"{name}__x"], z[f"{name}__w0"], z[f"{name}__w1"], z[f"{name}__experts"])
        if tp == 1:
            y = O.layer_forward(*args, activation=fn, combine_weights=cw)
        else:
            y = O.layer_forward_tp(*args, tp, activation=fn, combine_weights=cw)
        ref = z[f"{name}__y"]
        mx, fr = O.relative_error(y, ref)
        assert mx <= 1e-12 and fr <= 1e-12, (name, mx, fr)


def test_oracle_layer_forward_matches_reference_config1():
    import hashlib
    z = np.load(os.path.join(GOLD, "layer_c1.npz"))
    model = C.ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    r = Rt.build_routing(model, C.ParallelSpec(1, 8), C.WorkloadSpec(M=512, seed=0))
    np.testing.assert_array_equal(r.as_array(), z["experts"])
    x = np.random.default_rng(1).standard_normal((512, 512))
    rng = np.random.default_rng(2)
    scale = 1.0 / np.sqrt(512)
    w0 = rng.standard_normal((8, 512, 1024)) * scale
    w1 = rng.standard_normal((8, 1024, 512)) * scale
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["x_sha256"])
    assert hashlib.sha256(w0.tobytes()).hexdigest() == str(z["w0_sha256"])
    assert hashlib.sha256(w1.tobytes()).hexdigest() == str(z["w1_sha256"])
    y = O.layer_forward(x, w0, w1, r.as_array())
    mx, fr = O.relative_error(y, z["y"])
    assert mx < 1e-6 and fr < 1e-6


def test_round_bf16_matches_torch():
    import torch
    a = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 100
    ours = O.round_bf16(a)
    theirs = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(ours, theirs)


def test_literal_execute_naive_reproduces_reference_bitwise():
    """The literal loop-nest restatement (the Config-1 CPU timing arm) gives
    the reference's own execute_naive output bitwise (at the fixture's
    float32 storage precision) on a slice of Config 1
    (same float64 operations in the same order), and a weighted / tanh small
    case equal to the vectorised oracle within fp64 rounding."""
    z = np.load(os.path.join(GOLD, "layer_c1.npz"))
    model = C.ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    r = Rt.build_routing(model, C.ParallelSpec(1, 8), C.WorkloadSpec(M=512, seed=0))
    x = np.random.default_rng(1).standard_normal((512, 512))
    rng = np.random.default_rng(2)
    scale = 1.0 / np.sqrt(512)
    w0 = rng.standard_normal((8, 512, 1024)) * scale
    w1 = rng.standard_normal((8, 1024, 512)) * scale
    ex = r.as_array()
    y = O.execute_naive_literal(x[:24], w0, w1, ex[:24])
    np.testing.assert_array_equal(y.astype(np.float32), z["y"][:24])  # fixture stored as float32
    cw = np.random.default_rng(3).random((24, 2))
    y2 = O.execute_naive_literal(x[:24], w0, w1, ex[:24], activation=np.tanh, combine_weights=cw)
    ref = O.layer_forward(x[:24], w0, w1, ex[:24], activation=np.tanh, combine_weights=cw)
    np.testing.assert_allclose(y2, ref, rtol=1e-12, atol=1e-12)
