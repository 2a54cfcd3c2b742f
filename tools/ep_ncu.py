"""One emulated EP forward for ncu, product knobs (LayerKnobs.for_world:
chooser n_c and pair group): 3 warm forwards, then the profiled one (capture
rank 0's layer kernel with -k regex:moe_layer -s <3*ranks> -c 1).

    python tools/ep_ncu.py [--shape MX] [--ep 8] [--tp 1] [--M 8192]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402
from paper_2502_19811_b200.measure import EmulatedGroup  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="MX")
ap.add_argument("--ep", type=int, default=8)
ap.add_argument("--tp", type=int, default=1)
ap.add_argument("--M", type=int, default=8192)
a = ap.parse_args()
E, topk, N, K = SHAPES[a.shape]
model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
par = ParallelSpec(a.tp, a.ep)
routing = build_routing(model, par, WorkloadSpec(M=a.M, seed=0))
grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs.for_world(par.world_size))
for _ in range(4):
    grp._forward_timed(False)
torch.cuda.synchronize()
print("done", a.shape, a.ep, a.tp, "n_c", grp.layers[0].n_comm0(a.M), "group0", grp.layers[0].group0(a.M))
