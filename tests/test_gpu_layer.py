"""Fused layer numerics on the GPU, through the C-ABI (ctypes binding).

Parity targets: the reference's own fp64 outputs (tests/golden/, produced by
moepipe.execute_naive / execute_tp_sharded), the oracle restatement on
bf16-rounded inputs, and a plain PyTorch fp32 reference for full-size
shapes.  Tolerance (tests/refs.py): max|d|/max|ref| <= 1e-2 and
||d||_F/||ref||_F <= 5e-3 (bf16 storage, fp32 accumulation)."""

import os

import numpy as np
import pytest

from oracle import moe_oracle as O
from paper_2502_19811_b200 import (ConfigurationError, ExpertWeights, LayerKnobs, ModelConfig, MoELayer,
                                   ParallelSpec, RankWeights, WorkloadSpec, build_routing, execute_naive,
                                   execute_scheduled, execute_tp_sharded, meta_for_layer0, meta_for_layer1,
                                   random_weights, resolve_layer0, resolve_layer1)
from paper_2502_19811_b200.executor import run_emulated
from tests.refs import assert_close, oracle_bf16_inputs, torch_reference

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _small_cases():
    z = np.load(os.path.join(GOLD, "layer_small.npz"))
    return z, sorted({k.split("__")[0] for k in z.files})


@pytest.mark.parametrize("name", _small_cases()[1])
def test_reference_golden_small(name):
    z, _ = _small_cases()
    E, topk, N, K, M, tp, ep, seed, weighted = z[f"{name}__spec"].tolist()
    act = str(z[f"{name}__act"])
    fn = np.tanh if act == "tanh" else None
    cw = z[f"{name}__cw"] if weighted else None
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    routing = build_routing(model, ParallelSpec(tp=1 if tp > 1 else tp, ep=ep), WorkloadSpec(M=M, seed=seed))
    np.testing.assert_array_equal(routing.as_array(), z[f"{name}__experts"])
    w = ExpertWeights(z[f"{name}__w0"], z[f"{name}__w1"])
    x = z[f"{name}__x"]
    if tp == 1:
        y = execute_naive(x, w, routing, activation=fn, combine_weights=cw)
    else:
        y = execute_tp_sharded(x, w, routing, tp, activation=fn, combine_weights=cw)
    ref = z[f"{name}__y"]
    # vs the reference's fp64 output (includes bf16 input quantisation)
    assert_close(y, ref, max_rel=2e-2, frob_rel=1e-2, what=f"{name} vs reference fp64")
    # vs the oracle on bf16-rounded inputs (kernel error only)
    ora = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), fn, cw, tp=tp)
    assert_close(y, ora, what=f"{name} vs oracle(bf16 inputs)")


def test_reference_golden_config1_ep8_emulated():
    z = np.load(os.path.join(GOLD, "layer_c1.npz"))
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    routing = build_routing(model, ParallelSpec(1, 8), WorkloadSpec(M=512, seed=0))
    x = np.random.default_rng(1).standard_normal((512, 512))
    w = random_weights(model, seed=2)
    y = execute_naive(x, w, routing)
    assert_close(y, z["y"], what="config1 EP=8 vs reference execute_naive")
    s0 = [resolve_layer0(routing, g, meta_for_layer0(model, routing.workload)) for g in range(8)]
    s1 = [resolve_layer1(routing, g, meta_for_layer1(model, routing.workload)) for g in range(8)]
    y2 = execute_scheduled(x, w, routing, s0, s1)
    np.testing.assert_array_equal(y, y2)  # tile order never changes the arithmetic
    with pytest.raises(ConfigurationError):
        execute_scheduled(x, w, routing, s0[1:], s1)
    with pytest.raises(ConfigurationError):
        execute_scheduled(x[:10], w, routing, s0, s1)


@pytest.mark.parametrize("tp,ep,std", [(1, 1, 0.0), (1, 2, 0.05), (1, 4, 0.032), (1, 8, 0.0), (2, 2, 0.032),
                                       (2, 4, 0.0)])
def test_emulated_parallel_layouts_vs_oracle(tp, ep, std):
    model = ModelConfig(L=1, E=8, topk=2, N=256, K=512)
    routing = build_routing(model, ParallelSpec(tp, ep), WorkloadSpec(M=600, seed=5, std=std))
    w = random_weights(model, seed=6)
    x = np.random.default_rng(7).standard_normal((600, 256))
    cw = np.random.default_rng(3).random((600, 2))
    y = run_emulated(x, w, routing, ParallelSpec(tp, ep), combine_weights=cw,
                     knobs=LayerKnobs(n_comm0=2, n_comm1=2)).cpu().numpy()
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), combine_weights=cw, tp=tp)
    assert_close(y, ref, what=f"tp={tp} ep={ep} std={std}")


@pytest.mark.parametrize("n_comm1", [0, 2, 6, "fused"])
def test_combine_paths_agree(n_comm1):
    """world 1: local combine kernel, combine CTAs, and the epilogue-fused
    combine (LayerKnobs.fuse1: last hosted row folds the earlier ones) agree."""
    fuse1 = n_comm1 == "fused"
    if fuse1:
        n_comm1 = 0
    model = ModelConfig(L=1, E=8, topk=3, N=512, K=1024)
    routing = build_routing(model, ParallelSpec(), WorkloadSpec(M=777, seed=9, std=0.05))
    w = random_weights(model, seed=1)
    x = np.random.default_rng(2).standard_normal((777, 512))
    y = run_emulated(x, w, routing, ParallelSpec(), activation="tanh",
                     knobs=LayerKnobs(n_comm1=n_comm1, fuse1=fuse1)).cpu().numpy()
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), np.tanh)
    assert_close(y, ref, what=f"n_comm1={n_comm1}")


@pytest.mark.parametrize("ep,std", [(2, 0.0), (4, 0.05)])
def test_fused_combine_long_fold_chains(ep, std):
    """Qwen-style top-8: a token's hosted experts form fold chains of up to 7
    earlier rows in other pairs; the last row's epilogue waits for their tiles
    and pushes the weighted sum to the source rank."""
    model = ModelConfig(L=1, E=16, topk=8, N=256, K=512)
    routing = build_routing(model, ParallelSpec(1, ep), WorkloadSpec(M=700, seed=11, std=std))
    w = random_weights(model, seed=12)
    x = np.random.default_rng(13).standard_normal((700, 256))
    cw = np.random.default_rng(14).random((700, 8))
    y = run_emulated(x, w, routing, ParallelSpec(1, ep), combine_weights=cw).cpu().numpy()
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), combine_weights=cw)
    assert_close(y, ref, what=f"top-8 ep={ep}")


def test_edge_cases():
    model = ModelConfig(L=1, E=4, topk=2, N=64, K=128)
    w = random_weights(model, seed=3)
    # M = 0, M < world (all tokens on the last rank), one expert unused
    r0 = build_routing(model, ParallelSpec(1, 2), WorkloadSpec(M=0))
    assert execute_naive(np.zeros((0, 64)), w, r0).shape == (0, 64)
    r1 = build_routing(model, ParallelSpec(1, 4), WorkloadSpec(M=3, seed=1))
    x1 = np.random.default_rng(0).standard_normal((3, 64))
    assert_close(execute_naive(x1, w, r1), oracle_bf16_inputs(x1, w.w0, w.w1, r1.as_array()), what="M<W")
    r2 = build_routing(model, ParallelSpec(1, 2), WorkloadSpec(M=300, seed=2, std=max_std(4, 2)))
    assert 0 in r2.expert_counts
    x2 = np.random.default_rng(1).standard_normal((300, 64))
    assert_close(execute_naive(x2, w, r2), oracle_bf16_inputs(x2, w.w0, w.w1, r2.as_array()), what="skew")
    # zero input -> zero output (linearity, SPEC examples)
    assert np.abs(execute_naive(np.zeros((300, 64)), w, r2)).max() == 0.0
    # non-64-multiple shapes are zero-padded on the device
    m3 = ModelConfig(L=1, E=3, topk=2, N=40, K=72)
    r3 = build_routing(m3, ParallelSpec(), WorkloadSpec(M=50, seed=4))
    w3 = random_weights(m3, seed=5)
    x3 = np.random.default_rng(6).standard_normal((50, 40))
    assert_close(execute_naive(x3, w3, r3), oracle_bf16_inputs(x3, w3.w0, w3.w1, r3.as_array()), what="pad")
    with pytest.raises(ConfigurationError):
        execute_naive(x3, w3, r3, activation=lambda a: a * 2)


def max_std(E, k):
    from paper_2502_19811_b200 import max_achievable_std
    return max_achievable_std(E, k)


def test_mixtral_full_size_vs_torch_fp32_and_determinism():
    import torch
    model = ModelConfig(L=1, E=8, topk=2, N=4096, K=14336)
    par = ParallelSpec()
    routing = build_routing(model, par, WorkloadSpec(M=8192, seed=0, std=0.032))
    g = torch.Generator(device="cuda").manual_seed(0)
    w0 = torch.randn(8, 4096, 14336, device="cuda", generator=g) / 64.0
    w1 = torch.randn(8, 14336, 4096, device="cuda", generator=g) / 64.0
    x = torch.randn(8192, 4096, device="cuda", generator=g)
    cw = torch.rand(8192, 2, device="cuda", generator=g)
    layer = MoELayer(model, par, 0, 8192, RankWeights.from_full(w0, w1, model, par, 0))
    ex = torch.from_numpy(routing.as_array().copy()).cuda()
    y1 = layer.forward(x, ex, cw)
    y2 = layer.forward(x, ex, cw)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)  # run-to-run bitwise deterministic (ordered combine)
    ref = torch_reference(x, w0, w1, ex.long(), combine_w=cw)
    assert_close(y1.float().cpu().numpy(), ref.cpu().numpy(), what="Mixtral M=8192 EP=1")
    # size-independent property at full size: permuting the tokens permutes
    # the output rows bitwise (a row's products accumulate in a fixed order
    # wherever its tile lands; the combine order is per token)
    perm = torch.randperm(8192, generator=torch.Generator().manual_seed(5)).cuda()
    yp = layer.forward(x[perm], ex[perm].contiguous(), cw[perm].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(yp, y1[perm])
    # the zero-copy host forward (tokens read / output written over PCIe by
    # the layer kernel) at full size: same tolerance, run-to-run bitwise
    x_h, ex_h, cw_h = x.to(torch.bfloat16).cpu().pin_memory(), ex.cpu().pin_memory(), cw.cpu().pin_memory()
    yh = [layer.forward_host(x_h, ex_h, cw_h) for _ in range(2)]
    torch.cuda.synchronize()
    assert torch.equal(yh[0], yh[1])
    assert_close(yh[0].float().numpy(), ref.cpu().numpy(), what="Mixtral M=8192 EP=1 zero-copy host forward")
    layer.close()


@pytest.mark.parametrize("tp,ep,topk,std", [(1, 1, 2, 0.032), (1, 4, 2, 0.05), (1, 8, 2, 0.0), (2, 2, 3, 0.032),
                                            (1, 2, 8, 0.0)])
def test_launch_modes_bitwise_equal(tp, ep, topk, std):
    """One fused launch for both layers (dynamic unit claims, layer1 tiles
    gated on per-tile H counters, dispatch CTAs joining the GEMMs) vs
    separate layer0 / layer1 launches, and every layer1 tail split: each
    output element accumulates the same products in the same order, so the
    results are bitwise identical -- and match the oracle."""
    E = 16 if topk == 8 else 8
    model = ModelConfig(L=1, E=E, topk=topk, N=512, K=1024)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=1500, seed=21, std=std))
    w = random_weights(model, seed=22)
    x = np.random.default_rng(23).standard_normal((1500, 512))
    cw = np.random.default_rng(24).random((1500, topk))
    outs = []
    for fused, split1 in ((False, 0), (True, 0), (True, 74), (True, 100000)):
        outs.append(run_emulated(x, w, routing, par, activation="silu", combine_weights=cw,
                                 knobs=LayerKnobs(n_comm0=4, n_comm1=0, fused=fused, split1=split1)).cpu().numpy())
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])
    silu = lambda a: a / (1.0 + np.exp(-a))  # noqa: E731
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), silu, cw, tp=tp)
    assert_close(outs[0], ref, what=f"modes tp={tp} ep={ep} topk={topk}")


@pytest.mark.parametrize("ep,M", [(1, 6000), (8, 49152)])
def test_streamk_tail_split(ep, M):
    """COMET_OPT_STREAMK: layer1's single partial round (pairs/2 < tiles <
    pairs, no fold chains) as uneven head / tail K slices, the finisher
    decided at epilogue start and adding the other slice's partial while it
    drains (sched.cuh, moe_layers.cu).  Against the oracle, and run-to-run
    bitwise (the two-slice sum is order-fixed whichever slice finishes)."""
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    par = ParallelSpec(1, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=51, std=0.0))
    # tiles of layer1 on each rank (N = 512: one n-block) = its 256-row pairs
    counts = np.asarray(routing.expert_counts).reshape(ep, -1)
    tiles = [int(sum((c + 255) // 256 for c in row)) for row in counts]
    assert all(37 < t < 73 for t in tiles), tiles
    w = random_weights(model, seed=52)
    x = np.random.default_rng(53).standard_normal((M, 512))
    outs = [run_emulated(x, w, routing, par, knobs=LayerKnobs(n_comm0=4 if ep > 1 else 0, n_comm1=0, streamk=sk))
            .cpu().numpy() for sk in (True, True, False)]
    np.testing.assert_array_equal(outs[0], outs[1])
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array())
    assert_close(outs[0], ref, what=f"streamk ep={ep}")
    assert_close(outs[2], ref, what=f"whole units ep={ep}")


@pytest.mark.parametrize("chunks", [1, 3, None, [512, 2000, 2000, 488]])
def test_forward_host_pipeline(chunks):
    """Host-buffer end-to-end form: chunked H2D / forward / D2H pipeline
    (single GPU) == the device forward on the same tokens."""
    import torch
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    par = ParallelSpec()
    M = 5000
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=31, std=0.032))
    w = random_weights(model, seed=32)
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w.w0, w.w1, model, par, 0))
    x = torch.from_numpy(np.random.default_rng(33).standard_normal((M, 512)).astype(np.float32)).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy())
    cw = torch.from_numpy(np.random.default_rng(34).random((M, 2)).astype(np.float32))
    out = layer.forward_host(x.pin_memory(), ex.pin_memory(), cw.pin_memory(), chunks=chunks)
    out2 = layer.forward_host(x.pin_memory(), ex.pin_memory(), cw.pin_memory(), chunks=chunks)  # slot reuse
    torch.cuda.synchronize()
    ref = oracle_bf16_inputs(x.float().numpy(), w.w0, w.w1, routing.as_array(), combine_weights=cw.numpy())
    assert_close(out.float().numpy(), ref, what=f"forward_host chunks={chunks}")
    assert torch.equal(out, out2)
    layer.close()


@pytest.mark.parametrize("tp,ep,n_comm1", [(1, 1, 0), (1, 1, 2), (2, 2, 0), (1, 4, 0)])
def test_narrow_last_blocks(tp, ep, n_comm1):
    """Ragged last n-blocks of <= 256 columns run as half units (K/tp = 640,
    N = 640): per-tile H counters, combine-CTA and peer-flag targets count
    halves, results match the oracle."""
    model = ModelConfig(L=1, E=8, topk=2, N=640, K=1280)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=900, seed=41, std=0.032))
    w = random_weights(model, seed=42)
    x = np.random.default_rng(43).standard_normal((900, 640))
    cw = np.random.default_rng(44).random((900, 2))
    y = run_emulated(x, w, routing, par, combine_weights=cw,
                     knobs=LayerKnobs(n_comm0=8, n_comm1=n_comm1)).cpu().numpy()
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), combine_weights=cw, tp=tp)
    assert_close(y, ref, what=f"narrow tp={tp} ep={ep} n_comm1={n_comm1}")


@pytest.mark.parametrize("tp,ep,M", [(1, 8, 300), (1, 1, 200), (2, 4, 500), (1, 4, 64)])
def test_split_k_small_m(tp, ep, M):
    """Few output tiles per rank -> split-K (fp32 partials, the last slice
    reduces in slice order): within tolerance of the oracle, run-to-run
    bitwise deterministic, and close to the unsplit path."""
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=2048)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=51, std=0.032))
    w = random_weights(model, seed=52)
    x = np.random.default_rng(53).standard_normal((M, 512))
    cw = np.random.default_rng(54).random((M, 2))
    ys = []
    for ks in (8, 8, 0):
        ys.append(run_emulated(x, w, routing, par, activation="gelu_tanh", combine_weights=cw,
                               knobs=LayerKnobs(n_comm0=8, n_comm1=0, ksplit_max=ks)).cpu().numpy())
    np.testing.assert_array_equal(ys[0], ys[1])
    gelu = lambda a: 0.5 * a * (1 + np.tanh(0.7978845608028654 * (a + 0.044715 * a ** 3)))  # noqa: E731
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), gelu, cw, tp=tp)
    assert_close(ys[0], ref, what=f"split-K tp={tp} ep={ep} M={M}")
    assert_close(ys[2], ref, what=f"unsplit tp={tp} ep={ep} M={M}")


@pytest.mark.parametrize("ks", [3, 5, 6])
def test_split_k_slice_counts(ks):
    """S > 2 slices finish the tile's 64-column chunks round robin (chunk c
    by slice c mod S, sum of all S partials in slice order): every slice
    count, including ones that do not divide the 8 chunks, matches the
    oracle, is run-to-run bitwise deterministic, and equals the S = 8 result
    up to the fp32 partial-sum order (tolerance)."""
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=2048)
    par = ParallelSpec(1, 8)
    routing = build_routing(model, par, WorkloadSpec(M=300, seed=61, std=0.0))
    w = random_weights(model, seed=62)
    x = np.random.default_rng(63).standard_normal((300, 512))
    cw = np.random.default_rng(64).random((300, 2))
    ys = [run_emulated(x, w, routing, par, combine_weights=cw,
                       knobs=LayerKnobs(n_comm0=8, n_comm1=0, ksplit_max=ks)).cpu().numpy() for _ in range(2)]
    np.testing.assert_array_equal(ys[0], ys[1])
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), None, cw)
    assert_close(ys[0], ref, what=f"split-K S<={ks}")


@pytest.mark.parametrize("E,topk,M,N,K", [(8, 2, 5000, 512, 1024), (8, 3, 3000, 512, 2048), (16, 4, 700, 256, 512),
                                          (8, 2, 100, 512, 2048)])
def test_streamed_host_forward(E, topk, M, N, K):
    """comet_forward_host: upload chunks gate the dispatch, the fused combine
    (folder = each token's last-claimed row, all other rows folded) counts
    finished rows per chunk, downloads wait on the counts -- one launch.
    Matches the oracle; run-to-run bitwise deterministic."""
    import torch
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec()
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=61, std=0.032))
    w = random_weights(model, seed=62)
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w.w0, w.w1, model, par, 0),
                     activation="silu", knobs=LayerKnobs(n_comm0=16))
    x = torch.from_numpy(np.random.default_rng(63).standard_normal((M, N)).astype(np.float32)).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy())
    cw = torch.from_numpy(np.random.default_rng(64).random((M, topk)).astype(np.float32))
    outs = []
    for _ in range(2):
        out = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
        layer.forward_host(x.pin_memory(), ex.pin_memory(), cw.pin_memory(), out=out, mode="stream")
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    silu = lambda a: a / (1.0 + np.exp(-a))  # noqa: E731
    ref = oracle_bf16_inputs(x.float().numpy(), w.w0, w.w1, routing.as_array(), silu, cw.numpy())
    assert_close(outs[0].float().numpy(), ref, what=f"streamed E={E} topk={topk} M={M}")
    layer.close()


@pytest.mark.parametrize("E,topk,M,N,K,dedup,ilv,dl", [
    (8, 2, 5000, 512, 1024, "1", "2", "8"), (8, 2, 5000, 512, 1024, "0", "2", "8"),
    (8, 2, 5000, 512, 1024, "1", "0", "0"), (8, 2, 5000, 512, 1024, "1", "1", "16"),
    (8, 3, 3000, 1024, 2048, "1", "2", "8"), (16, 4, 700, 512, 512, "1", "2", "2"),
    (16, 4, 700, 512, 512, "1", "0", "8"), (8, 2, 100, 512, 2048, "1", "2", "8"),
    (8, 1, 1000, 512, 1024, "1", "2", "0"), (8, 2, 6000, 1024, 3200, "1", "3", "8"),
    (8, 2, 300, 512, 2048, "1", "0", "8"), (8, 2, 1, 512, 1024, "1", "3", "8"), (8, 4, 129, 512, 512, "1", "1", "4")])
def test_zerocopy_host_forward(E, topk, M, N, K, dedup, ilv, dl):
    """comet_forward_zerocopy: dispatch CTAs read token rows from pinned host
    memory (once per token with dedup, fanned out to every hosted row), the
    fused combine writes output rows straight to pinned host memory; layer1
    groups interleaved with layer0 groups at lag ``ilv`` (0 = after layer0);
    ``dl`` dispatch CTAs download the output afterwards (0: epilogues write
    the host rows; M=300 runs layer1 split-K).
    Matches the oracle; run-to-run bitwise deterministic; equal to the
    device-resident forward."""
    import torch
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec()
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=71, std=0.032))
    w = random_weights(model, seed=72)
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w.w0, w.w1, model, par, 0), activation="silu",
                     knobs=LayerKnobs(n_comm0=16, zc_dedup=dedup == "1", zc_interleave=int(ilv), zc_download=int(dl)))
    x = torch.from_numpy(np.random.default_rng(73).standard_normal((M, N)).astype(np.float32)).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy())
    cw = torch.from_numpy(np.random.default_rng(74).random((M, topk)).astype(np.float32))
    outs = []
    for _ in range(2):
        out = torch.full((M, N), float("nan"), dtype=torch.bfloat16).pin_memory()
        layer.forward_host(x.pin_memory(), ex.pin_memory(), cw.pin_memory(), out=out)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    silu = lambda a: a / (1.0 + np.exp(-a))  # noqa: E731
    ref = oracle_bf16_inputs(x.float().numpy(), w.w0, w.w1, routing.as_array(), silu, cw.numpy())
    assert_close(outs[0].float().numpy(), ref, what=f"zero-copy E={E} topk={topk} M={M} dedup={dedup} ilv={ilv} dl={dl}")
    layer.close()


@pytest.mark.parametrize("E,topk,tp,ep,M", [(16, 4, 1, 4, 3000), (64, 8, 1, 8, 2000), (8, 2, 2, 4, 4000)])
def test_dispatch_dedup_bitwise(E, topk, tp, ep, M):
    """Per-token dedup of the NVLink pulls (LayerKnobs.dedup=1, dispatch_rows_dedup:
    one read per (token, rank), fanned out to its hosted rows) moves the same
    bytes into the same rows: bitwise equal to the per-row dispatch, and
    within tolerance of the oracle."""
    model = ModelConfig(L=1, E=E, topk=topk, N=512, K=1024)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=81, std=0.032))
    w = random_weights(model, seed=82)
    x = np.random.default_rng(83).standard_normal((M, 512))
    cw = np.random.default_rng(84).random((M, topk))
    outs = []
    for dd in (0, 1, 1):
        outs.append(run_emulated(x, w, routing, par, activation="silu", combine_weights=cw,
                                 knobs=LayerKnobs(n_comm0=8, n_comm1=0, dedup=dd)).cpu().numpy())
    np.testing.assert_array_equal(outs[1], outs[0])
    np.testing.assert_array_equal(outs[2], outs[0])
    silu = lambda a: a / (1.0 + np.exp(-a))  # noqa: E731
    ref = oracle_bf16_inputs(x, w.w0, w.w1, routing.as_array(), silu, cw, tp=tp)
    assert_close(outs[1], ref, what=f"dedup E={E} topk={topk} tp={tp} ep={ep}")


@pytest.mark.parametrize("E,topk,tp,ep,M", [(8, 2, 1, 8, 2048), (16, 4, 2, 2, 3000), (64, 8, 1, 8, 1500)])
def test_dispatch_item_rows_bitwise(E, topk, tp, ep, M):
    """The dispatch item size (COMET_OPT_CHUNK_ROWS: 0 = auto, ~one item per
    dispatch CTA; 1..32 fixed; with and without per-token dedup) only changes
    which CTA copies which rows: the result is bitwise the same."""
    model = ModelConfig(L=1, E=E, topk=topk, N=512, K=1024)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=91, std=0.032))
    w = random_weights(model, seed=92)
    x = np.random.default_rng(93).standard_normal((M, 512))
    cw = np.random.default_rng(94).random((M, topk))
    outs = [run_emulated(x, w, routing, par, activation="silu", combine_weights=cw,
                         knobs=LayerKnobs(n_comm0=16, n_comm1=0, chunk_rows=cr, dedup=dd)).cpu().numpy()
            for cr, dd in ((0, 0), (1, 0), (5, 0), (32, 0), (0, 1), (8, 1))]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


@pytest.mark.parametrize("act", ["gelu_tanh", "relu", None])
def test_zerocopy_unweighted_activations(act):
    """Zero-copy host forward without combine weights (plain sum over the
    token's experts, executor.py:102-120) and with each epilogue activation."""
    import torch
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    par = ParallelSpec()
    M = 2000
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=91, std=0.032))
    w = random_weights(model, seed=92)
    layer = MoELayer(model, par, 0, M, RankWeights.from_full(w.w0, w.w1, model, par, 0), activation=act,
                     knobs=LayerKnobs(n_comm0=16))
    x = torch.from_numpy(np.random.default_rng(93).standard_normal((M, 512)).astype(np.float32)).to(torch.bfloat16)
    ex = torch.from_numpy(routing.as_array().copy())
    out = torch.empty(M, 512, dtype=torch.bfloat16).pin_memory()
    layer.forward_host(x.pin_memory(), ex.pin_memory(), None, out=out)
    torch.cuda.synchronize()
    fns = {"gelu_tanh": lambda a: 0.5 * a * (1 + np.tanh(0.7978845608028654 * (a + 0.044715 * a ** 3))),
           "relu": lambda a: np.maximum(a, 0.0), None: None}
    ref = oracle_bf16_inputs(x.float().numpy(), w.w0, w.w1, routing.as_array(), fns[act])
    assert_close(out.float().numpy(), ref, what=f"zero-copy unweighted act={act}")
    layer.close()


@pytest.mark.parametrize("tp,ep,topk", [(1, 2, 2), (2, 2, 3), (1, 4, 8)])
def test_emulated_unfused_matches_fused(tp, ep, topk):
    """measure.EmulatedUnfused (the unfused all-to-all + grouped-GEMM path,
    every rank emulated on this GPU, the comparison baseline of
    tools/matrix.py at EP > 1) computes the same layer as the fused group:
    both within tolerance of a torch fp32 reference of the same weights."""
    import torch
    from paper_2502_19811_b200.measure import EmulatedGroup, EmulatedUnfused
    E = 16 if topk == 8 else 8
    model = ModelConfig(L=1, E=E, topk=topk, N=512, K=1024)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=1024, seed=81, std=0.032))
    grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs(n_comm0=8, n_comm1=0))
    cw = torch.rand(1024, topk, device="cuda", generator=torch.Generator(device="cuda").manual_seed(82))
    un = EmulatedUnfused(grp)
    outs, _ = un.forward(combine_w=cw)
    y_un = torch.cat(outs).float()
    # fp32 reference from the group's own bf16 weights and tokens
    x = torch.cat(un.xs).float()
    ex = grp.ex.long()
    y_ref = torch.zeros(1024, 512, device="cuda")
    kl = model.K // tp
    for r, l in enumerate(grp.layers):
        e_lo = par.ep_group_of_rank(r) * (E // par.ep)
        for j in range(E // par.ep):
            hit = (ex == e_lo + j)
            t_idx, slot = hit.nonzero(as_tuple=True)
            if t_idx.numel() == 0:
                continue
            h = (x[t_idx] @ l.weights.w0t[j, :kl, :512].float().t()).to(torch.bfloat16).float()
            yr = (h @ l.weights.w1t[j, :512, :kl].float().t()).to(torch.bfloat16).float()
            y_ref.index_add_(0, t_idx, yr * cw[t_idx, slot].unsqueeze(1))
    assert_close(y_un.cpu().numpy(), y_ref.cpu().numpy(), what=f"emulated unfused tp={tp} ep={ep} topk={topk}")
    lat = un.measure(iters=2, warmup=1)
    assert lat["latency_ms"] > 0 and len(lat["per_rank_ms"]) == par.world_size
    grp.close()
