"""Measured timeline of an emulated EP=2 forward (NVLink-path comm CTAs),
scored with the reference's overlap metrics and audited; measured split
sweep through the reference's SplitMetadata/select_split."""

import numpy as np
import pytest

from paper_2502_19811_b200 import (LayerKnobs, ModelConfig, ParallelSpec, SplitKey, SplitMetadata, WorkloadSpec,
                                   build_routing, random_weights, select_split, sweep_split)
from paper_2502_19811_b200 import timeline as TL
from paper_2502_19811_b200.executor import _group_cache, run_emulated

pytestmark = pytest.mark.gpu


def _decode_layer0(u, P, NB, G, n_pairs=None):
    """Pair of layer0 unit u (moe_layers.cu decode_unit + make_sched tail split)."""
    if n_pairs is not None:
        U = P * NB
        R, rem = divmod(U, n_pairs)
        if rem and 2 * rem <= n_pairs and u >= R * n_pairs:
            u = R * n_pairs + (u - R * n_pairs) // 2
    per_group = G * NB
    g = u // per_group
    ge = min(G, P - g * G)
    rem = u - g * per_group
    return g * G + rem % ge  # pair (claim-order position)


def test_measured_timeline_overlap_and_dependency_audit():
    import torch
    model = ModelConfig(L=1, E=4, topk=2, N=512, K=2048)
    par = ParallelSpec(1, 2)
    routing = build_routing(model, par, WorkloadSpec(M=2048, seed=3))
    w = random_weights(model, seed=4)
    x = np.random.default_rng(5).standard_normal((2048, 512))
    knobs = LayerKnobs(n_comm0=2, n_comm1=2, group0=4)
    run_emulated(x, w, routing, par, knobs=knobs)                      # build + place tokens
    layers = _group_cache[(model, par, 2048)]
    ex = torch.from_numpy(routing.as_array().copy()).cuda()
    ys = [torch.empty(l.token_range(2048)[1] - l.token_range(2048)[0], 512, dtype=torch.bfloat16,
                      device="cuda") for l in layers]
    for layer in layers:
        layer.ctx.timeline_enable(64)
        layer.ctx.index_build(ex, 2048, flags=2)
    for layer in layers:
        layer.ctx.signal_tokens_ready()
    for layer in layers:
        layer.ctx.layer0(layer.weights.w0t, 0, knobs.n_comm0, knobs.group0)
    torch.cuda.synchronize()
    for layer in layers:
        recs = layer.ctx.timeline_dump()
        ivs = TL.from_records(recs)
        m = TL.metrics(ivs)
        assert 0.0 <= m["hidden_fraction"] <= 1.0 and m["total_latency_ns"] > 0
        assert any(iv.block_kind == "comm" for iv in ivs), "no NVLink dispatch tasks recorded"
        # compute roles are serial per CTA (comm CTAs are pipelined engines: their
        # task intervals may overlap by design)
        for role in ("load", "mma", "epilogue"):
            sub = [TL.Interval(c, "compute", t, s, e) for c, r, t, s, e in recs if r == role]
            assert not [p for p in TL.audit(sub) if "overlaps" in p], role
        # dependency audit: each CTA's loads of unit u start only after the
        # NVLink tile holding its 128 A rows (tile 2*pair + cta) was published
        meta = layer.ctx.index_meta()
        P, NB = int(meta[3]), -(-layer.ctx.k_local // 512)
        # (a tile's remote rows are pulled in 16-row chunks by several dispatch
        # CTAs: one comm interval per chunk, task = tile; the audit takes the
        # tile's last chunk)
        comm_ivs = [TL.Interval(c, "comm", t, s, e) for c, r, t, s, e in recs if r == "comm"]
        load_ivs = [TL.Interval(c, "compute", 2 * t + (c & 1), s, e) for c, r, t, s, e in recs if r == "load"]
        # unit claims are dynamic over every pair (dispatch pairs join the GEMMs)
        n_pairs = torch.cuda.get_device_properties(0).multi_processor_count // 2
        deps = {2 * u + c: [2 * _decode_layer0(u, P, NB, knobs.group0, n_pairs) + c]
                for u in range(2 * P * NB) for c in (0, 1)}
        bad = [p for p in TL.audit(comm_ivs + load_ivs, deps) if "overlaps" not in p]
        assert bad == [], bad[:5]
    for layer, y in zip(layers, ys):
        layer.ctx.layer1(layer.weights.w1t, None, y, knobs.n_comm1, knobs.wave1)
    for layer, y in zip(layers, ys):
        layer.ctx.combine_finish(y)
    torch.cuda.synchronize()
    for layer in layers:
        recs = layer.ctx.timeline_dump()
        m = TL.metrics(TL.from_records(recs))
        # world > 1: the combine is fused into the epilogue (NVLink pushes), no comm CTAs
        assert m["comm_busy_ns"] == 0 and m["compute_busy_ns"] > 0
        assert any(r == "epilogue" for _, r, _, _, _ in recs)
        csv = TL.timeline_csv(TL.from_records(recs))
        assert csv.startswith("block_id,block_kind,task_id,start_ns,end_ns\n")
        layer.ctx.timeline_enable(0)


def test_measured_split_sweep_and_select(tmp_path):
    model = ModelConfig(L=1, E=4, topk=2, N=512, K=1024)
    rec = sweep_split(model, ParallelSpec(1, 2), WorkloadSpec(M=1024, seed=0), max_nc=6, repeats=3)
    assert [nc for nc, _ in rec.curve] == [2, 4, 6]
    assert all(ns > 0 for _, ns in rec.curve)
    md = SplitMetadata(records=[rec])
    md.save(str(tmp_path / "split.json"))
    split = select_split(SplitMetadata.load(str(tmp_path / "split.json")),
                         SplitKey.for_config(model, ParallelSpec(1, 2), 2048, "b200", rec.key.blocks))
    assert split.n_c == rec.optimal_nc and split.n == rec.key.blocks


def test_layer_takes_n_c_from_the_chooser():
    """The product path (MoELayer with default knobs) launches with the n_c
    the adaptive chooser picks: the committed measured sweep for a profiled
    Mixtral EP=8 shape, the fitted cost model for an unprofiled one; an
    explicit knob overrides both; world 1 has no dispatch CTAs."""
    import torch
    from paper_2502_19811_b200 import MoELayer, RankWeights, _lib
    from paper_2502_19811_b200.assigner import choose_split
    sms = _lib.device_info(0)["sms"]
    for model, par, M, src in ((ModelConfig(L=1, E=8, topk=2, N=4096, K=14336), ParallelSpec(1, 8), 8192, "measured"),
                               (ModelConfig(L=1, E=8, topk=2, N=512, K=1024), ParallelSpec(1, 2), 1000, "model")):
        kl = model.K // par.tp
        w = RankWeights(torch.zeros(model.E // par.ep, kl, model.N, dtype=torch.bfloat16, device="cuda"),
                        torch.zeros(model.E // par.ep, model.N, kl, dtype=torch.bfloat16, device="cuda"))
        layer = MoELayer(model, par, 0, M, w)
        nc, got_src = layer.split_choice(M)
        assert got_src == src
        assert nc == choose_split(model, par, M, sms)[0].n_c
        # the layer0 pair group measured with that n_c (default rule without a record)
        from paper_2502_19811_b200.assigner import choose_knobs
        assert layer.group0(M) == choose_knobs(model, par, M, sms)[2]
        layer.knobs = LayerKnobs.for_world(par.world_size, n_comm0=6, group0=3)
        assert layer.split_choice(M) == (6, "knob") and layer.group0(M) == 3
        layer.close()
    w1 = RankWeights(torch.zeros(8, 1024, 512, dtype=torch.bfloat16, device="cuda"),
                     torch.zeros(8, 512, 1024, dtype=torch.bfloat16, device="cuda"))
    l1 = MoELayer(ModelConfig(L=1, E=8, topk=2, N=512, K=1024), ParallelSpec(), 0, 100, w1)
    assert l1.split_choice(100) == (0, "world1")
    l1.close()
