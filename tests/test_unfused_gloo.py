"""The unfused NCCL all-to-all + GroupGEMM comparison path (unfused.py) and
its coarse-grained chunked pipeline (simulate_coarse analogue,
simulator.py:624-743) across real processes: world 2 (EP=2) and world 4
(EP=2 x TP=2) over gloo on CPU -- the same all_to_all_single calls the NCCL
run makes on GPUs.  Gathered outputs are checked against the oracle on
bf16-rounded inputs (test infrastructure) within the stated tolerance."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, tp, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec, build_routing, random_weights
        from paper_2502_19811_b200.unfused import UnfusedLayer
        model = ModelConfig(L=1, E=8, topk=2, N=64, K=128)
        par = ParallelSpec(tp=tp, ep=world // tp)
        M = 203
        routing = build_routing(model, par, WorkloadSpec(M=M, seed=4, std=0.05))
        w = random_weights(model, seed=5)
        x = np.random.default_rng(6).standard_normal((M, 64)).astype(np.float32)
        cw = np.random.default_rng(7).random((M, 2)).astype(np.float32)
        e_per, kl = 8 // par.ep, 128 // tp
        g, s = par.ep_group_of_rank(rank), par.tp_index_of_rank(rank)
        bf = torch.bfloat16
        w0 = torch.from_numpy(w.w0[g * e_per:(g + 1) * e_per, :, s * kl:(s + 1) * kl].astype(np.float32)).to(bf)
        w1 = torch.from_numpy(w.w1[g * e_per:(g + 1) * e_per, s * kl:(s + 1) * kl, :].astype(np.float32)).to(bf)
        layer = UnfusedLayer(model, par, rank, w0, w1, activation="tanh")
        base = M // world
        lo, hi = rank * base, (M if rank == world - 1 else (rank + 1) * base)
        ex = torch.from_numpy(routing.as_array().copy())
        outs = {c: layer.forward(torch.from_numpy(x[lo:hi]).to(bf), ex, torch.from_numpy(cw), chunks=c).float().numpy()
                for c in (1, 3)}
        q.put((rank, lo, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world,tp", [(2, 1), (4, 2)])
def test_unfused_all_to_all_across_processes(world, tp):
    from oracle import moe_oracle as O
    from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec, build_routing, random_weights
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, tp, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in procs]
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    M = 203
    model = ModelConfig(L=1, E=8, topk=2, N=64, K=128)
    routing = build_routing(model, ParallelSpec(tp=tp, ep=world // tp), WorkloadSpec(M=M, seed=4, std=0.05))
    w = random_weights(model, seed=5)
    x = np.random.default_rng(6).standard_normal((M, 64)).astype(np.float32)
    cw = np.random.default_rng(7).random((M, 2)).astype(np.float32)
    rb = lambda a: O.round_bf16(np.asarray(a, np.float32)).astype(np.float64)  # noqa: E731
    args = (rb(x), rb(w.w0), rb(w.w1), routing.as_array())
    ref = O.layer_forward(*args, activation=np.tanh, combine_weights=cw) if tp == 1 else \
        O.layer_forward_tp(*args, tp, activation=np.tanh, combine_weights=cw)
    for chunks in (1, 3):
        y = np.zeros((M, 64))
        for _, lo, outs in res:
            y[lo:lo + outs[chunks].shape[0]] = outs[chunks]
        mx, fr = O.relative_error(y, ref)
        assert mx <= 1e-2 and fr <= 1e-2, (chunks, mx, fr)
