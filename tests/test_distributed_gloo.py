"""Multi-process host logic of the multi-GPU bootstrap, world_size 2 over
gloo on CPU: IPC-handle all-gather ordering, routing broadcast, token
partition and world-size checks."""

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


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_19811_b200 import distributed as D
        from paper_2502_19811_b200 import ConfigurationError, ModelConfig, ParallelSpec, WorkloadSpec, build_routing
        handle = bytes([rank + 1]) * 64
        allh = D.exchange_handles(handle)
        model = ModelConfig(L=1, E=4, topk=2, N=64, K=64)
        par = ParallelSpec(tp=1, ep=world)
        arr = build_routing(model, par, WorkloadSpec(M=37, seed=3)).as_array() if rank == 0 else None
        arr = D.broadcast_array(arr)
        lo, hi = D.token_slice(37, rank, world)
        bad = False
        try:
            D.check_world(ParallelSpec(tp=2, ep=world), world)
        except ConfigurationError:
            bad = True
        q.put((rank, allh, arr.tolist(), (lo, hi), bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_bootstrap_host_logic_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    (r0, h0, a0, s0, b0), (r1, h1, a1, s1, b1) = res
    assert h0 == h1 == bytes([1]) * 64 + bytes([2]) * 64
    assert a0 == a1 and len(a0) == 37
    assert s0 == (0, 18) and s1 == (18, 37)
    assert b0 and b1
