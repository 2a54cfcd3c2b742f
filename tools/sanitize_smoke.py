"""One small emulated-EP forward for compute-sanitizer (racecheck /
synccheck / memcheck), checked against the oracle afterwards.

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py [EP] [M]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import moe_oracle as O  # noqa: E402  (checker only)
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing, random_weights  # noqa: E402
from paper_2502_19811_b200.executor import run_emulated  # noqa: E402

ep = int(sys.argv[1]) if len(sys.argv) > 1 else 2
M = int(sys.argv[2]) if len(sys.argv) > 2 else 300
model = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
par = ParallelSpec(tp=1, ep=ep)
routing = build_routing(model, par, WorkloadSpec(M=M, seed=0, std=0.032))
w = random_weights(model, seed=1)
x = np.random.default_rng(2).standard_normal((M, 512))
cw = np.random.default_rng(3).random((M, 2))
knobs = LayerKnobs(n_comm0=2, n_comm1=2) if ep > 1 else LayerKnobs(n_comm0=0, n_comm1=0)
y = run_emulated(x, w, routing, par, activation="tanh", combine_weights=cw, knobs=knobs).cpu().numpy()
rb = lambda a: O.round_bf16(np.asarray(a, np.float32)).astype(np.float64)  # noqa: E731
ref = O.layer_forward(rb(x), rb(w.w0), rb(w.w1), routing.as_array(), activation=np.tanh, combine_weights=cw)
mx, fr = O.relative_error(y, ref)
print(f"EP={ep} M={M}: max|d|/max|ref|={mx:.2e} frob={fr:.2e} {'OK' if mx <= 1e-2 else 'FAIL'}")
