"""Overlap evidence on a real link: the single-GPU forward on HOST buffers
(tokens in, output out over PCIe 5), Mixtral layer M=8192.

    no overlap   H2D of the tokens, device forward, D2H of the output, serial
                 (forward_host mode "chunks" with one chunk)
    coarse:k     k token chunks: H2D of chunk c+1 and D2H of chunk c-1 on copy
                 streams under the forward of chunk c
    fine         ONE launch: dispatch CTAs read each token row once from pinned
                 host memory in the GEMMs' claim order, the fused combine's rows
                 go back while layer1 runs (comet_forward_zerocopy)

plus the PCIe copy rates and the device-resident forward.  Prints one JSON
line.

    python tools/e2e_probe.py [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import rank_weights_random  # noqa: E402
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, MoELayer, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
M, N = 8192, 4096
model = ModelConfig(L=1, E=8, topk=2, N=N, K=14336)
par = ParallelSpec()
routing = build_routing(model, par, WorkloadSpec(M=M, seed=0))
layer = MoELayer(model, par, 0, M, rank_weights_random(model, par, 0, torch.device("cuda", 0)),
                 knobs=LayerKnobs.for_world(1))
x_host = torch.randn(M, N).to(torch.bfloat16).pin_memory()
ex_host = torch.from_numpy(routing.as_array().copy()).pin_memory()
y_host = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
x_dev = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")


def timed(fn, n=a.reps):
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


out = {"workload": "Mixtral-8x7B layer, M=8192, EP=1, host (pinned) tokens and output"}
out["h2d_ms"] = timed(lambda: x_dev.copy_(x_host, non_blocking=True))
out["d2h_ms"] = timed(lambda: y_host.copy_(x_dev, non_blocking=True))
out["h2d_GBps"] = x_host.numel() * 2 / out["h2d_ms"] / 1e6
ex_dev = ex_host.cuda()
y_dev = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
layer.place_tokens(x_dev, M)
out["device_forward_ms"] = timed(lambda: layer.run(ex_dev, M, y_dev))
out["no_overlap_ms"] = timed(lambda: layer.forward_host(x_host, ex_host, out=y_host, mode="chunks", chunks=1))
for k in (2, 3, 4):
    out[f"coarse{k}_ms"] = timed(lambda: layer.forward_host(x_host, ex_host, out=y_host, mode="chunks", chunks=k))
out["fine_zerocopy_ms"] = timed(lambda: layer.forward_host(x_host, ex_host, out=y_host, mode="zerocopy"))
ref = y_host.clone()
layer.forward_host(x_host, ex_host, out=y_host, mode="chunks", chunks=1)
torch.cuda.synchronize()
out["fine_vs_no_overlap_max_abs_diff"] = (ref.float() - y_host.float()).abs().max().item()
out = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}
print(json.dumps(out))
layer.close()
