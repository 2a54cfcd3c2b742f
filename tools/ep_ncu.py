"""One emulated EP forward for ncu: 2 warm forwards, then the profiled one
(capture rank 0's layer kernel with -k regex:moe_layer -s <2*W> -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402
from paper_2502_19811_b200.measure import EmulatedGroup  # noqa: E402

ep = int(sys.argv[1]) if len(sys.argv) > 1 else 8
model = ModelConfig(L=1, E=8, topk=2, N=4096, K=14336)
par = ParallelSpec(1, ep)
routing = build_routing(model, par, WorkloadSpec(M=8192, seed=0))
grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs(n_comm0=64, group0=4))
for _ in range(3):
    grp._forward_timed(False)
torch.cuda.synchronize()
print("done")
