"""Layer parity at every BASELINE.json shape at full size (M = 8192), all
ranks of the ParallelSpec emulated on the one GPU through the C-ABI, against
a plain PyTorch fp32 reference of the same op (tests/refs.py, TP partials per
executor.py:221-246).  Tolerance: max|d|/max|ref| <= 1e-2,
||d||_F/||ref||_F <= 5e-3.  Also run-to-run bitwise determinism at size, and
the equality of the per-token deduplicated dispatch with the per-row one.

Shapes: MX = Mixtral-8x7B (E8 top-2 N4096 K14336) at EP=8;
PH = Phi-3.5-MoE (E16 top-2 N4096 K6400) at EP=4 x TP=2 (K/tp = 3200: a
narrow last n-block); QW = Qwen2-style (E64 top-8 N3584 K2560) at EP=8
(8 hosted experts per rank, 7-row fold chains, split-tail halves)."""

import numpy as np
import pytest

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing
from paper_2502_19811_b200.executor import run_emulated
from tests.refs import assert_close, torch_reference

pytestmark = pytest.mark.gpu

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}


def _inputs(shape, seed=0):
    import torch
    E, topk, N, K = SHAPES[shape]
    g = torch.Generator(device="cuda").manual_seed(seed)
    w0 = torch.randn(E, N, K, device="cuda", generator=g) / N ** 0.5
    w1 = torch.randn(E, K, N, device="cuda", generator=g) / N ** 0.5
    x = torch.randn(8192, N, device="cuda", generator=g)
    cw = torch.rand(8192, topk, device="cuda", generator=g)
    return w0, w1, x, cw


@pytest.mark.parametrize("shape,tp,ep,std,act", [
    ("MX", 1, 8, 0.0, None), ("MX", 1, 8, 0.05, "silu"), ("MX", 1, 4, 0.032, None), ("MX", 1, 2, 0.0, None),
    ("PH", 2, 4, 0.0, None), ("PH", 2, 4, 0.032, "silu"),
    ("QW", 1, 8, 0.0, None), ("QW", 1, 8, 0.032, "silu")])
def test_full_size_vs_torch_fp32(shape, tp, ep, std, act):
    import torch
    E, topk, N, K = SHAPES[shape]
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=8192, seed=0, std=std))
    w0, w1, x, cw = _inputs(shape)
    y = run_emulated(x, (w0, w1), routing, par, activation=act, combine_weights=cw)
    y2 = run_emulated(x, (w0, w1), routing, par, activation=act, combine_weights=cw)
    assert torch.equal(y, y2), "run-to-run bitwise determinism"
    ex = torch.from_numpy(routing.as_array().copy()).cuda().long()
    ref = torch_reference(x, w0, w1, ex, activation=act, combine_w=cw, tp=tp)
    mx, fr = assert_close(y.cpu().numpy(), ref.cpu().numpy(), what=f"{shape} tp={tp} ep={ep} std={std}")
    print(f"{shape} tp={tp} ep={ep} std={std}: max {mx:.2e} frob {fr:.2e}")


@pytest.mark.parametrize("shape,tp,ep,std", [("QW", 1, 8, 0.032), ("MX", 1, 8, 0.0), ("PH", 2, 4, 0.0)])
def test_full_size_dedup_dispatch_bitwise(shape, tp, ep, std):
    """Per-(token, rank) deduplicated pulls move the same bytes into the same
    rows as the per-row pulls: bitwise equal at full size."""
    import torch
    E, topk, N, K = SHAPES[shape]
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=8192, seed=0, std=std))
    w0, w1, x, cw = _inputs(shape, seed=1)
    outs = [run_emulated(x, (w0, w1), routing, par, combine_weights=cw,
                         knobs=LayerKnobs.for_world(par.world_size, dedup=d)) for d in (0, 1)]
    assert torch.equal(outs[0], outs[1])


def test_full_size_unfused_baseline_vs_torch_fp32():
    """The unfused comparison path (unfused.py: permutation, grouped GEMMs,
    index-add combine) computes the same layer at full Mixtral size."""
    import torch
    from paper_2502_19811_b200.unfused import UnfusedLayer
    E, topk, N, K = SHAPES["MX"]
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec()
    routing = build_routing(model, par, WorkloadSpec(M=8192, seed=0, std=0.032))
    w0, w1, x, cw = _inputs("MX", seed=2)
    layer = UnfusedLayer(model, par, 0, w0.to(torch.bfloat16), w1.to(torch.bfloat16))
    ex = torch.from_numpy(routing.as_array().copy()).cuda()
    y = layer.forward(x.to(torch.bfloat16), ex, cw)
    ref = torch_reference(x, w0, w1, ex.long(), combine_w=cw)
    assert_close(y.float().cpu().numpy(), ref.cpu().numpy(), what="unfused MX")
    for chunks in (2, 4):
        yc = layer.forward(x.to(torch.bfloat16), ex, cw, chunks=chunks)
        assert_close(yc.float().cpu().numpy(), ref.cpu().numpy(), what=f"coarse unfused chunks={chunks}")
