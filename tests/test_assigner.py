"""Split chooser semantics (ref assigner.py:44-292) with synthetic measured
curves; no GPU."""

import pytest

from paper_2502_19811_b200 import (ConfigurationError, KernelSplit, ModelConfig, ParallelSpec, SplitKey,
                                   SplitMetadata, UnprofiledConfigError, WorkloadSpec, select_split,
                                   split_for, sweep_split)
from paper_2502_19811_b200.assigner import SplitRecord, candidate_ncs, record_from_curve

MX = ModelConfig(L=32, E=8, topk=2, N=4096, K=14336)


def key(m, ep=8, blocks=148):
    return SplitKey.for_config(MX, ParallelSpec(1, ep), m, "b200", blocks)


def test_kernel_split_invariants():
    assert split_for(148, 8) == KernelSplit(148, 140, 8)
    with pytest.raises(ConfigurationError):
        KernelSplit(148, 148, 0)
    with pytest.raises(ConfigurationError):
        KernelSplit(148, 100, 8)


def test_sweep_argmin_ties_to_smaller_nc():
    curve = {2: 500, 4: 400, 6: 400, 8: 450}
    rec = sweep_split(MX, ParallelSpec(1, 8), WorkloadSpec(M=8192), blocks=148, max_nc=8,
                      measure=lambda nc: curve[nc] * 1e-9)
    assert (rec.optimal_nc, rec.latency_ns) == (4, 400)
    assert rec.curve == ((2, 500), (4, 400), (6, 400), (8, 450))
    assert rec.key == key(8192)


def test_record_rejects_non_argmin():
    with pytest.raises(ConfigurationError):
        SplitRecord(key=key(4096), optimal_nc=2, latency_ns=9, curve=((2, 9), (4, 3)))


def test_select_exact_then_nearest_log2_bucket(tmp_path):
    md = SplitMetadata(records=[])
    md.add(record_from_curve(key(4096), [(2, 10), (4, 5)]))
    md.add(record_from_curve(key(16384), [(2, 3), (4, 7)]))
    path = tmp_path / "meta.json"
    md.save(str(path))
    md2 = SplitMetadata.load(str(path))
    assert md2.to_json_str() == md.to_json_str()
    assert select_split(md2, key(4096)).n_c == 4
    assert select_split(md2, key(16384)).n_c == 2
    assert select_split(md2, key(8192)).n_c == 4          # equidistant -> smaller bucket
    assert select_split(md2, key(12000)).n_c == 2
    with pytest.raises(UnprofiledConfigError):
        select_split(md2, key(8192, ep=4))
    with pytest.raises(UnprofiledConfigError):
        select_split(SplitMetadata(records=[]), key(8192))


def test_candidates_even_cluster_multiples():
    assert candidate_ncs(148, 2, 12) == [2, 4, 6, 8, 10, 12]
    assert all(nc % 2 == 0 for nc in candidate_ncs(148, 3, 40))


def test_product_chooser_uses_measured_metadata_then_cost_model():
    """The layer's n_c (MoELayer.split_choice -> assigner.choose_split) is the
    committed B200 sweep's select_split answer for profiled shapes (exact
    key, else nearest log2 bucket) and the fitted cost model's
    predict_split answer for unprofiled ones (ref cli.py:228-235)."""
    from paper_2502_19811_b200 import costmodel
    from paper_2502_19811_b200.assigner import choose_split, default_metadata
    meta = default_metadata()
    assert meta.records, "split_b200.json (tools/sweep_b200.py) must be committed"
    par = ParallelSpec(1, 8)
    for m in (8192, 6000, 50000):
        split, src = choose_split(MX, par, m, 148)
        assert src == "measured"
        assert split == select_split(meta, key(m))
        assert split.n == 148 and split.n_c % 2 == 0
    # every committed record is the argmin of its own measured curve
    for r in meta.records:
        assert r.key.cost == "b200" and r.key.blocks == 148
        assert (r.optimal_nc, r.latency_ns) == min(r.curve, key=lambda pt: (pt[1], pt[0]))
    # unprofiled shape (an embed no sweep covered): the cost model answers
    odd = ModelConfig(L=1, E=8, topk=2, N=2048, K=8192)
    split, src = choose_split(odd, ParallelSpec(1, 4), 4096, 148)
    assert src == "model"
    assert split.n_c == costmodel.predict_split(odd, ParallelSpec(1, 4), WorkloadSpec(M=4096, seed=0)).optimal_nc


def test_joint_group_sweep_and_record_round_trip():
    """B200 extension: sweep_split over (n_c, group0) keeps the best group's
    curve and the group; the JSON keeps the reference schema plus an
    optional "group0"; choose_knobs returns it (default group otherwise)."""
    from paper_2502_19811_b200.assigner import choose_knobs, default_group0
    lat = {(nc, g): 1000 - 10 * nc + (0 if g == 4 else 50) for nc in (2, 4, 6) for g in (2, 4, 8)}
    rec = sweep_split(MX, ParallelSpec(1, 8), WorkloadSpec(M=8192), blocks=148, candidates=[2, 4, 6],
                      groups=[2, 4, 8], measure=lambda nc, g: lat[(nc, g)] * 1e-9)
    assert (rec.optimal_nc, rec.group0, rec.latency_ns) == (6, 4, 940)
    assert rec.curve == ((2, 980), (4, 960), (6, 940))
    meta = SplitMetadata(records=[rec])
    back = SplitMetadata.from_json_str(meta.to_json_str())
    assert back.records == [rec]
    split, src, g0 = choose_knobs(MX, ParallelSpec(1, 8), 8192, 148, meta)
    assert (split.n_c, src, g0) == (6, "measured", 4)
    plain = record_from_curve(key(8192), [(2, 5), (4, 3)])
    assert "group0" not in plain.to_json_dict()
    split, src, g0 = choose_knobs(MX, ParallelSpec(1, 8), 8192, 148, SplitMetadata(records=[plain]))
    assert (split.n_c, g0) == (4, default_group0(8))


def test_sweep_passes_keep_each_points_minimum():
    """passes > 1: the grid is measured round-robin and each point keeps its
    minimum (a drifting clock between the points of a flat curve)."""
    calls = []
    noisy = {(2, 4): [900, 700], (4, 4): [800, 800], (2, 8): [850, 860], (4, 8): [990, 600]}

    def measure(nc, g):
        i = sum(1 for c in calls if c == (nc, g))
        calls.append((nc, g))
        return noisy[(nc, g)][i] * 1e-9
    rec = sweep_split(MX, ParallelSpec(1, 8), WorkloadSpec(M=8192), blocks=148, candidates=[2, 4],
                      groups=[4, 8], passes=2, measure=measure)
    assert (rec.group0, rec.optimal_nc, rec.latency_ns) == (8, 4, 600)
    assert rec.curve == ((2, 850), (4, 600))
    assert calls[:4] == [(2, 4), (4, 4), (2, 8), (4, 8)]  # round robin over the grid
