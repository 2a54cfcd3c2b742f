"""B200 cost model: fit recovers known parameters, the
committed fit predicts the measured latencies it was validated on, and
predict_split answers an unprofiled shape with a reference-schema record."""

import json

import numpy as np
import pytest

from paper_2502_19811_b200 import (ModelConfig, ParallelSpec, SplitMetadata, UnprofiledConfigError, WorkloadSpec,
                                   build_routing, select_split)
from paper_2502_19811_b200 import costmodel as CM


def test_fit_recovers_parameters():
    rng = np.random.default_rng(0)
    flops = rng.choice([1.07e9, 3.76e9, 0.5e9], 400)
    rate, alpha = 23e12, 2e-6
    secs = alpha + flops / rate + rng.normal(0, 1e-8, 400)
    cm = CM.fit([{"unit_flops": flops, "unit_s": secs, "cta_rates": [30e9, 32e9, 28e9], "fixed_s": 5e-5}])
    assert abs(cm.compute_flops_per_s / rate - 1) < 0.01 and abs(cm.alpha_tile_s - alpha) < 2e-7
    assert cm.intra_node_bytes_per_s == 30e9 and cm.fixed_s == 5e-5


def test_committed_fit_matches_its_validation():
    with open(CM.PRESET_PATH) as fh:
        data = json.load(fh)
    cm = CM.CostModel.from_json_dict(data["model"])
    assert cm.blocks == 148 and cm.compute_flops_per_s > 1e13
    shapes = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}
    for v in data["validation"]:
        shape, ep, tp, M, std, nc = v["config"]
        E, topk, N, K = shapes[shape]
        r = build_routing(ModelConfig(L=1, E=E, topk=topk, N=N, K=K), ParallelSpec(tp, ep),
                          WorkloadSpec(M=M, seed=0, std=std))
        pred = max(CM.simulate(r, rk, cm, nc) for rk in range(r.parallel.world_size)) * 1e3
        assert pred == pytest.approx(v["predicted_ms"], rel=1e-3)
        if shape == "MX" and M >= 4096:
            # Mixtral shapes within 20% of the measurement (small-M split-K
            # tails and PH / QW fold tails are under-predicted)
            assert abs(v["rel_err"]) < 0.2, v


def test_predict_split_answers_unprofiled_shapes():
    model = ModelConfig(L=1, E=8, topk=2, N=4096, K=14336)
    par = ParallelSpec(1, 8)
    wl = WorkloadSpec(M=6000, seed=0)
    with pytest.raises(UnprofiledConfigError):
        select_split(SplitMetadata(records=[]), None)
    rec = CM.predict_split(model, par, wl, stride=16, max_nc=64)
    assert rec.key.cost == "b200-model" and rec.key.blocks == 148
    assert [nc for nc, _ in rec.curve] == [2, 18, 34, 50]
    split = select_split(SplitMetadata(records=[rec]), rec.key)
    assert split.n_c == rec.optimal_nc and split.n_p == 148 - rec.optimal_nc
    # EP=1 has no dispatch: n_c does not change the prediction
    r1 = build_routing(model, ParallelSpec(1, 1), WorkloadSpec(M=4096, seed=0))
    cm = CM.preset()
    assert CM.simulate(r1, 0, cm, 2) == CM.simulate(r1, 0, cm, 64)


def test_fold_loads_and_epilogue_fit():
    """Fold counts per pair from the routing (a token's last hosted row folds
    the others) and the epilogue / per-fold-row fit."""
    qw = build_routing(ModelConfig(L=1, E=64, topk=8, N=3584, K=2560), ParallelSpec(1, 8), WorkloadSpec(M=8192, seed=0))
    sh = CM.rank_shape(qw, 0)
    assert [f for (j, _, _), f in zip(sh.pairs, sh.folds) if j == 7] == [7.0] * 4
    assert all(f == 0.0 for (j, _, _), f in zip(sh.pairs, sh.folds) if j != 7)
    mx = build_routing(ModelConfig(L=1, E=8, topk=2, N=4096, K=14336), ParallelSpec(1, 1), WorkloadSpec(M=4096, seed=0))
    sh1 = CM.rank_shape(mx, 0)  # world 1: experts {2k, 2k+1} -> the odd expert's rows fold one row
    assert all(f == (1.0 if j % 2 else 0.0) for (j, _, _), f in zip(sh1.pairs, sh1.folds))
    rng = np.random.default_rng(1)
    flops = rng.choice([1.07e9, 3.76e9], 200)
    epi = [10e-6] * 50 + [10e-6 + 7 * 6e-6] * 20 + [5e-6 + 3.5 * 6e-6] * 10
    cm = CM.fit([{"unit_flops": flops, "unit_s": 2e-6 + flops / 23e12, "cta_rates": [30e9], "fixed_s": 5e-5,
                  "epi_s": epi, "epi_folds": [0] * 50 + [7] * 20 + [3.5] * 10, "epi_scale": [1] * 70 + [0.5] * 10}])
    assert cm.epilogue_s == pytest.approx(10e-6) and cm.fold_row_s == pytest.approx(6e-6)
    assert CM.default_split1(qw, 148) == 55 and CM.default_split1(mx, 148) == -1
