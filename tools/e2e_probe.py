"""End-to-end (host buffers) forward: chunk-count sweep and PCIe copy rates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import rank_weights_random  # noqa: E402
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, MoELayer, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402

M, N = 8192, 4096
model = ModelConfig(L=1, E=8, topk=2, N=N, K=14336)
par = ParallelSpec()
routing = build_routing(model, par, WorkloadSpec(M=M, seed=0))
layer = MoELayer(model, par, 0, M, rank_weights_random(model, par, 0, torch.device("cuda", 0)), knobs=LayerKnobs())
x_host = torch.randn(M, N).to(torch.bfloat16).pin_memory()
ex_host = torch.from_numpy(routing.as_array().copy()).pin_memory()
y_host = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
x_dev = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


t = timed(lambda: x_dev.copy_(x_host, non_blocking=True))
print(f"H2D 64 MiB: {t:.3f} ms = {x_host.numel() * 2 / t / 1e6:.1f} GB/s")
t = timed(lambda: y_host.copy_(x_dev, non_blocking=True))
print(f"D2H 64 MiB: {t:.3f} ms = {x_host.numel() * 2 / t / 1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        x_dev.copy_(x_host, non_blocking=True)
    with torch.cuda.stream(s2):
        y_host.copy_(x_dev, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(both)
print(f"H2D || D2H 64 MiB each: {t:.3f} ms")
ex_dev = ex_host.cuda()
y_dev = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
layer.place_tokens(x_dev, M)
t = timed(lambda: layer.run(ex_dev, M, y_dev))
print(f"device forward: {t:.3f} ms")
for rep in range(2):
    t = timed(lambda: layer.forward_host(x_host, ex_host, out=y_host, chunks=3))
    print(f"forward_host chunk pipeline (3): {t:.3f} ms")
    for dd in ("1", "0"):
        os.environ["COMET_ZC_DEDUP"] = dd
        for nc in (8, 16, 32):
            t = timed(lambda: layer.ctx.forward_zerocopy(x_host, ex_host, None, y_host, M, layer.weights.w0t,
                                                         layer.weights.w1t, 0, n_comm0=nc, group0=8, wave1=4))
            print(f"zero-copy dedup={dd} n_comm0={nc}: {t:.3f} ms")
    os.environ["COMET_ZC_DEDUP"] = "1"
ref = y_host.clone()
layer.forward_host(x_host, ex_host, out=y_host, chunks=3)
torch.cuda.synchronize()
print("zero-copy == chunk pipeline:", torch.equal(ref, y_host), (ref.float() - y_host.float()).abs().max().item())
