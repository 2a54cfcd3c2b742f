"""Worker for tests/test_gpu_multiproc.py (torchrun, one process per rank).

Every rank runs its own MoELayer (own CUDA context, own symmetric heap), the
IPC handles are exchanged over gloo (NCCL on distinct GPUs), and three consecutive forwards run
concurrently across the processes -- the real multi-rank protocol (IPC-mapped
peer heaps, system-scope epoch flags, dispatch pulls / combine pushes).  With
COMET_SAME_DEVICE=1 all ranks share GPU 0 (LayerKnobs.grid splits the SMs so the
persistent kernels are co-resident).  Rank 0 checks the gathered output
against the oracle (test infrastructure only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_19811_b200 import (LayerKnobs, ModelConfig, ParallelSpec, RankWeights, WorkloadSpec,  # noqa: E402
                                   build_routing, distributed, random_weights)


def main():
    tp, ep, topk = (int(v) for v in sys.argv[1:4])
    backend = os.environ.get("COMET_TEST_BACKEND", "gloo")
    if backend == "nccl":  # distinct GPUs: NCCL bootstrap, as bench.py / deployments use
        torch.cuda.set_device(distributed.local_device())
        dist.init_process_group("nccl", device_id=torch.device("cuda", distributed.local_device()))
    else:
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    model = ModelConfig(L=1, E=8, topk=topk, N=512, K=1024)
    par = ParallelSpec(tp, ep)
    M = 1000
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=71, std=0.032))
    w = random_weights(model, seed=72)
    x = np.random.default_rng(73).standard_normal((M, 512)).astype(np.float32)
    cw = np.random.default_rng(74).random((M, topk)).astype(np.float32)
    dev = distributed.local_device()
    rw = RankWeights.from_full(w.w0, w.w1, model, par, rank, device=dev)
    grid = int(os.environ.get("COMET_TEST_GRID", 148))  # SMs per rank when ranks share one GPU
    layer = distributed.init_layer(model, par, M, rw, activation="tanh",
                                   knobs=LayerKnobs(n_comm0=min(8, max(2, grid // 2 // 2 * 2)),
                                                    grid=grid if grid < 148 else None))
    lo, hi = layer.token_range(M)
    ex = torch.from_numpy(routing.as_array().copy()).cuda(dev)
    outs = []
    for _ in range(3):  # epoch reuse of the flags and buffers
        y = layer.forward(torch.from_numpy(x[lo:hi]).cuda(dev), ex, torch.from_numpy(cw).cuda(dev), M=M)
        torch.cuda.synchronize(dev)
        outs.append(y.float().cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:]), "forwards differ across epochs"
    # the reference-named per-rank entry point, with this rank's validated
    # schedules, on the same layer: the same rows
    from paper_2502_19811_b200 import (execute_scheduled_rank, meta_for_layer0, meta_for_layer1, resolve_layer0,
                                       resolve_layer1)
    s0 = resolve_layer0(routing, rank, meta_for_layer0(model, routing.workload))
    s1 = resolve_layer1(routing, rank, meta_for_layer1(model, routing.workload))
    y = execute_scheduled_rank(x[lo:hi], rw, routing, s0, s1, activation="tanh", combine_weights=cw, layer=layer)
    torch.cuda.synchronize(dev)
    assert np.array_equal(y.float().cpu().numpy(), outs[-1]), "execute_scheduled_rank differs from forward"
    parts = [None] * world
    dist.all_gather_object(parts, (lo, outs[-1]))
    if rank == 0:
        from oracle import moe_oracle as O
        y = np.zeros((M, 512))
        for a, part in parts:
            y[a:a + part.shape[0]] = part
        rb = lambda a: O.round_bf16(np.asarray(a, np.float32)).astype(np.float64)  # noqa: E731
        args = (rb(x), rb(w.w0), rb(w.w1), routing.as_array())
        ref = O.layer_forward(*args, activation=np.tanh, combine_weights=cw) if tp == 1 else \
            O.layer_forward_tp(*args, tp, activation=np.tanh, combine_weights=cw)
        mx, fr = O.relative_error(y, ref)
        assert mx <= 1e-2 and fr <= 5e-3, (mx, fr)
        print(f"MP_OK world={world} tp={tp} ep={ep} max={mx:.2e} frob={fr:.2e}", flush=True)
    dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
