"""A few zero-copy host forwards (Mixtral M=8192, EP=1) for ncu captures:
ncu -k regex:moe_layer_kernel --launch-skip 2 --launch-count 1 python tools/zc_once.py"""
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
layer = MoELayer(model, par, 0, M, rank_weights_random(model, par, 0, torch.device("cuda", 0)),
                 knobs=LayerKnobs(n_comm0=16, group0=8))
x_host = torch.randn(M, N).to(torch.bfloat16).pin_memory()
ex_host = torch.from_numpy(routing.as_array().copy()).pin_memory()
y_host = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
for _ in range(int(os.environ.get("REPS", 3))):
    layer.forward_host(x_host, ex_host, out=y_host)
torch.cuda.synchronize()
print("done")
