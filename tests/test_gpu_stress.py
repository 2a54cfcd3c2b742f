"""Randomised stress of the fused layer against the torch fp32 reference.

Each case draws a shape (experts, top-k, N, K incl. ragged multiples of 64,
token count down to 1), a parallel layout (EP x TP, every rank emulated on
this GPU), routing skew, an activation, combine weights or none, and kernel
knobs (dispatch CTAs, pair groups, split-K slices, split-tail halves, one or
two launches, stream-K tails) -- the paths the layer kernel can take: narrow
last n-blocks, split-K with 2..8 slices and chunk helpers, fold chains up to
top-8 (one folder, or chained folds of stride 2/3/8), layer1 halves, the
per-n-block H gating.  Every case must match the reference within the
stated tolerance and be bitwise identical when run twice (deterministic
reductions and folds).  Seeded: a failure names its case.
"""

import os

import numpy as np
import pytest

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing
from paper_2502_19811_b200.executor import run_emulated
from tests.refs import assert_close, torch_reference

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("COMET_STRESS_CASES", 48))  # a longer hunt: COMET_STRESS_CASES=500


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    E = int(r.choice([4, 8, 16]))
    topk = int(r.choice([k for k in (1, 2, 3, 4, 8) if k <= E]))
    tp = int(r.choice([1, 2]))
    ep = int(r.choice([e for e in (1, 2, 4, 8) if E % e == 0 and e * tp <= 8]))
    N = int(r.choice([256, 512, 768, 1024]))
    K = int(r.choice([512, 1024, 1536, 2048, 3200 // 2])) * tp  # K/tp in {512..2048, 1600}
    M = int(r.choice([1, 7, 100, 333, 1024, 2500]))
    std = float(r.choice([0.0, 0.032, 0.05])) if topk < E else 0.0  # top-k = E: every token on every expert
    act = r.choice([None, "silu", "tanh"])
    weighted = bool(r.integers(0, 2))
    knobs = dict(n_comm0=int(r.choice([2, 4, 8, 16, 32])), n_comm1=0, group0=int(r.choice([1, 2, 4, 8, 16])),
                 ksplit_max=int(r.choice([0, 2, 3, 8])), split1=int(r.choice([-1, 0, 8, 74])),
                 fused=bool(r.integers(0, 4) > 0), streamk=bool(r.integers(0, 4) == 0),
                 wave1=int(r.choice([1, 2, 4, 8])), chunk_rows=int(r.choice([0, 1, 7, 16, 32])),
                 dedup=int(r.integers(0, 4) == 0), fold_order=bool(r.integers(0, 3) == 0),
                 pull_local=bool(r.integers(0, 4) > 0), group1=int(r.choice([0, 0, 1, 4])),
                 fold_stride=int(r.choice([0, 2, 2, 3, 8])))
    return E, topk, tp, ep, N, K, M, std, act, weighted, knobs


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_layer_case(seed):
    import torch
    E, topk, tp, ep, N, K, M, std, act, weighted, knobs = _case(seed)
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=seed, std=std))
    g = torch.Generator(device="cuda").manual_seed(seed)
    w0 = torch.randn(E, N, K, device="cuda", generator=g) / N ** 0.5
    w1 = torch.randn(E, K, N, device="cuda", generator=g) / K ** 0.5
    x = torch.randn(M, N, device="cuda", generator=g)
    cw = torch.rand(M, topk, device="cuda", generator=g) if weighted else None
    kn = LayerKnobs(**knobs)
    what = f"seed={seed} E={E} topk={topk} tp={tp} ep={ep} N={N} K={K} M={M} std={std} act={act} cw={weighted} {knobs}"
    y1 = run_emulated(x, (w0, w1), routing, par, activation=act, combine_weights=cw, knobs=kn)
    y2 = run_emulated(x, (w0, w1), routing, par, activation=act, combine_weights=cw, knobs=kn)
    assert torch.equal(y1, y2), f"{what}: not run-to-run bitwise"
    ex = torch.from_numpy(routing.as_array().copy()).cuda().long()
    ref = torch_reference(x, w0, w1, ex, act, cw, tp=tp)
    if M * topk < 4:  # a couple of rows: compare absolute (max-normalisation is ill-posed)
        np.testing.assert_allclose(y1.cpu().numpy(), ref.cpu().numpy(), atol=3e-2, rtol=3e-2, err_msg=what)
    else:
        assert_close(y1.cpu().numpy(), ref.cpu().numpy(), what=what)


@pytest.mark.parametrize("seed", range(N_CASES // 4))
def test_random_host_forward_case(seed):
    """The single-GPU forward on pinned host buffers (zero-copy: token rows
    read over PCIe by the dispatch CTAs, output rows written back by
    downloader CTAs or the epilogues; streamed; chunk pipeline) with random
    shapes and knobs vs the torch fp32 reference, run-to-run bitwise."""
    import torch
    from paper_2502_19811_b200 import MoELayer, RankWeights
    r = np.random.default_rng(5000 + seed)
    E = int(r.choice([4, 8, 16]))
    topk = int(r.choice([k for k in (1, 2, 4, 8) if k <= E]))
    N = int(r.choice([512, 1024]))
    K = int(r.choice([512, 1024, 1600]))
    M = int(r.choice([1, 100, 777, 3000]))
    mode = str(r.choice(["zerocopy", "zerocopy", "chunks", "stream"]))
    knobs = dict(zc_n_comm=int(r.choice([2, 8, 16, 32])), zc_group0=int(r.choice([1, 4, 16])),
                 zc_dedup=bool(r.integers(0, 3) > 0), zc_interleave=int(r.choice([0, 1, 2])),
                 zc_download=int(r.choice([0, 4, 8])), stream_n_comm=int(r.choice([4, 16])))
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec()
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=seed, std=0.032 if topk < E else 0.0))
    g = torch.Generator(device="cuda").manual_seed(seed)
    w0 = torch.randn(E, N, K, device="cuda", generator=g) / N ** 0.5
    w1 = torch.randn(E, K, N, device="cuda", generator=g) / K ** 0.5
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w0, w1, model, par, 0), activation="tanh",
                     knobs=LayerKnobs(**knobs))
    x = torch.randn(M, N, generator=torch.Generator().manual_seed(seed)).to(torch.bfloat16).pin_memory()
    ex = torch.from_numpy(routing.as_array().copy()).pin_memory()
    cw = torch.rand(M, topk, generator=torch.Generator().manual_seed(seed + 1)).pin_memory()
    outs = []
    for _ in range(2):
        out = torch.full((M, N), float("nan"), dtype=torch.bfloat16).pin_memory()
        layer.forward_host(x, ex, cw, out=out, mode=mode)
        torch.cuda.synchronize()
        outs.append(out)
    what = f"host seed={seed} E={E} topk={topk} N={N} K={K} M={M} mode={mode} {knobs}"
    assert torch.equal(outs[0], outs[1]), f"{what}: not run-to-run bitwise"
    ref = torch_reference(x.cuda(), w0, w1, ex.cuda().long(), "tanh", cw.cuda())
    if M * topk < 4:
        np.testing.assert_allclose(outs[0].float().numpy(), ref.cpu().numpy(), atol=3e-2, rtol=3e-2, err_msg=what)
    else:
        assert_close(outs[0].float().numpy(), ref.cpu().numpy(), what=what)
    layer.close()
