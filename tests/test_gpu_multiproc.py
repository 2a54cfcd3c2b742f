"""The multi-rank protocol with real processes: one process (own CUDA
context and symmetric heap) per rank, IPC-mapped peer heaps, forwards running
concurrently -- on a single-GPU box every rank shares GPU 0 with the SMs split
between the ranks' persistent kernels (LayerKnobs.grid); with enough GPUs
visible, the same workers run one GPU per rank over NCCL bootstrap, and one
process drives several GPUs through comet_link_local."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tp,ep,topk", [(1, 2, 2), (2, 1, 2), (1, 2, 3), (1, 4, 2), (2, 2, 2), (1, 8, 2)])
def test_processes_share_the_protocol(tp, ep, topk):
    import torch
    world = tp * ep
    grid = torch.cuda.get_device_properties(0).multi_processor_count // world // 2 * 2
    env = dict(os.environ, COMET_SAME_DEVICE="1", COMET_TEST_GRID=str(grid), MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + tp * 100 + ep * 10 + topk),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(tp), str(ep), str(topk)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "MP_OK" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("tp,ep,topk", [(1, 2, 2), (2, 2, 2), (1, 4, 3), (1, 8, 2)])
def test_processes_on_distinct_gpus(tp, ep, topk):
    """The same protocol with one GPU per rank (NCCL bootstrap, peer heaps
    over NVLink, full grids): needs world GPUs, skipped otherwise."""
    import torch
    world = tp * ep
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    env = dict(os.environ, COMET_TEST_BACKEND="nccl", MASTER_ADDR="127.0.0.1")
    env.pop("COMET_SAME_DEVICE", None)
    env.pop("COMET_TEST_GRID", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29900 + tp * 100 + ep * 10 + topk),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(tp), str(ep), str(topk)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "MP_OK" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("ep", [2, 4])
def test_one_process_several_gpus(ep):
    """comet_link_local across devices: one process drives ep GPUs (peer
    access enabled by the library, per-device kernel attributes); the ranks'
    forwards run concurrently on their own GPUs.  Oracle parity and
    run-to-run bitwise equality."""
    import numpy as np
    import torch
    if torch.cuda.device_count() < ep:
        pytest.skip(f"needs {ep} GPUs, {torch.cuda.device_count()} visible")
    sys.path.insert(0, ROOT)
    from oracle import moe_oracle as O
    from paper_2502_19811_b200 import (LayerKnobs, ModelConfig, MoELayer, ParallelSpec, RankWeights, WorkloadSpec,
                                       _lib, build_routing, random_weights)
    model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    par = ParallelSpec(1, ep)
    M = 1200
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=81, std=0.032))
    w = random_weights(model, seed=82)
    x = np.random.default_rng(83).standard_normal((M, 512)).astype(np.float32)
    layers = [MoELayer(model, par, r, M, RankWeights.from_full(w.w0, w.w1, model, par, r, device=r), device=r,
                       knobs=LayerKnobs.for_world(ep, n_comm0=8)) for r in range(ep)]
    _lib.Context.link_local([l.ctx for l in layers])
    outs = []
    for _ in range(2):
        ys = []
        for l in layers:
            lo, hi = l.token_range(M)
            with torch.cuda.device(l.device):
                ex = torch.from_numpy(routing.as_array().copy()).cuda(l.device)
                l.place_tokens(torch.from_numpy(x[lo:hi]).to(torch.bfloat16).cuda(l.device), M)
                y = torch.empty(hi - lo, l.n_pad, dtype=torch.bfloat16, device=f"cuda:{l.device}")
                l.run(ex, M, y)  # asynchronous: the other GPUs' launches follow at once
                ys.append(y)
        for l in layers:
            torch.cuda.synchronize(l.device)
        outs.append(np.concatenate([y.float().cpu().numpy() for y in ys]))
    np.testing.assert_array_equal(outs[0], outs[1])
    rb = lambda a: O.round_bf16(np.asarray(a, np.float32)).astype(np.float64)  # noqa: E731
    ref = O.layer_forward(rb(x), rb(w.w0), rb(w.w1), routing.as_array())
    mx, fr = O.relative_error(outs[0], ref)
    assert mx <= 1e-2 and fr <= 5e-3, (mx, fr)
    for l in layers:
        l.close()
