"""GPU router front-end (comet_router_topk) vs the oracle: expert ids
bit-exact (==), weights within 1e-6 absolute of the fp64 oracle; and
router -> fused layer end to end within the layer tolerance."""

import numpy as np
import pytest

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu


def _run(lg_np, k, norm, dtype="f32"):
    import torch
    from paper_2502_19811_b200.router import route_topk
    t = torch.from_numpy(lg_np.astype(np.float32)).cuda()
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
    ex, w = route_topk(t, k, norm)
    torch.cuda.synchronize()
    src = t.float().cpu().numpy()
    return ex.cpu().numpy(), (None if w is None else w.cpu().numpy()), src


@pytest.mark.parametrize("M,E,k", [(1, 8, 2), (1000, 8, 2), (8192, 8, 2), (777, 16, 2), (8192, 64, 8),
                                   (300, 128, 6), (257, 256, 8), (100, 512, 32), (50, 33, 32), (64, 5, 1)])
@pytest.mark.parametrize("norm", ["topk", "all", None])
def test_router_bit_exact(M, E, k, norm):
    rng = np.random.default_rng(M + E + k)
    lg = rng.standard_normal((M, E)).astype(np.float32)
    lg[::3] = np.round(lg[::3] * 2) / 2  # exact ties on every third token
    ex, w, src = _run(lg, k, norm)
    ref_e, ref_w = O.router_topk(src, k, norm)
    assert np.array_equal(ex, ref_e)
    if norm is None:
        assert w is None
    else:
        np.testing.assert_allclose(w, ref_w, rtol=0, atol=1e-6)


def test_router_bf16_logits_and_special_values():
    rng = np.random.default_rng(5)
    lg = rng.standard_normal((512, 64)).astype(np.float32)
    lg[0] = 0.0
    lg[1, ::2] = -0.0
    lg[2, 3] = np.nan
    lg[3] = -np.inf
    lg[3, 63] = np.nan
    lg[4, 10] = np.inf
    ex, _, src = _run(lg, 8, None, "bf16")
    ref_e, _ = O.router_topk(src, 8, None)
    assert np.array_equal(ex, ref_e)
    ex32, _, src32 = _run(lg, 8, None)
    assert np.array_equal(ex32, O.router_topk(src32, 8, None)[0])


def test_router_empty_and_errors():
    import torch
    from paper_2502_19811_b200 import ConfigurationError
    from paper_2502_19811_b200.router import route_topk
    ex, w = route_topk(torch.zeros(0, 8, device="cuda"), 2)
    assert ex.shape == (0, 2) and w.shape == (0, 2)
    with pytest.raises(ConfigurationError):
        route_topk(torch.zeros(4, 8, device="cuda"), 9)
    with pytest.raises(ConfigurationError):
        route_topk(torch.zeros(4, 600, device="cuda"), 2)
    with pytest.raises(ConfigurationError):
        route_topk(torch.zeros(4, 8, device="cuda", dtype=torch.float16), 2)


def test_router_feeds_the_fused_layer():
    """logits -> GPU router -> MoELayer.forward (ids and combine weights stay
    on the device) == oracle layer on the oracle's routing, within the layer
    tolerance."""
    import torch
    from paper_2502_19811_b200 import ModelConfig, MoELayer, ParallelSpec, RankWeights, random_weights
    from paper_2502_19811_b200.router import route_topk
    model = ModelConfig(L=1, E=16, topk=4, N=256, K=512)
    M = 700
    rng = np.random.default_rng(9)
    lg = rng.standard_normal((M, 16)).astype(np.float32)
    x = rng.standard_normal((M, 256)).astype(np.float32)
    w = random_weights(model, seed=3)
    par = ParallelSpec(1, 1)
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w.w0, w.w1, model, par, 0))
    ex, cw = route_topk(torch.from_numpy(lg).cuda(), 4, "topk")
    y = layer.forward(torch.from_numpy(x).cuda(), ex, cw, M=M).float().cpu().numpy()
    ref_e, ref_w = O.router_topk(lg, 4, "topk")
    rb = lambda a: O.round_bf16(np.asarray(a, np.float32)).astype(np.float64)  # noqa: E731
    ref = O.layer_forward(rb(x), rb(w.w0), rb(w.w1), ref_e, combine_weights=ref_w)
    mx, fr = O.relative_error(y, ref)
    assert mx <= 1e-2 and fr <= 5e-3, (mx, fr)
    layer.close()
