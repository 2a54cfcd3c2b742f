"""Fit the B200 cost model (paper_2502_19811_b200/costmodel.py) to measured
timelines and validate its predictions; writes costmodel_b200.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402
from paper_2502_19811_b200 import costmodel as CM  # noqa: E402
from paper_2502_19811_b200.measure import EmulatedGroup  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}
FIT = [("MX", 1, 1, 8192, 0.0, 0), ("MX", 8, 1, 8192, 0.0, 64), ("MX", 4, 1, 4096, 0.032, 32),
       ("QW", 8, 1, 8192, 0.0, 64)]
VALIDATE = FIT + [("MX", 2, 1, 8192, 0.0, 32), ("MX", 8, 1, 2048, 0.0, 64), ("MX", 8, 1, 16384, 0.032, 16),
                  ("PH", 4, 2, 8192, 0.0, 64), ("MX", 8, 1, 8192, 0.0, 16), ("MX", 1, 1, 2048, 0.0, 0)]


def run(cfg):
    shape, ep, tp, M, std, nc = cfg
    E, topk, N, K = SHAPES[shape]
    model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
    par = ParallelSpec(tp, ep)
    routing = build_routing(model, par, WorkloadSpec(M=M, seed=0, std=std))
    grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs(n_comm0=nc, n_comm1=0))
    try:
        m = grp.measure(iters=5)
        lat = m["per_rank_ms"][0] * 1e-3
        ctx = grp.layers[0].ctx
        ctx.timeline_enable(1024)
        grp._forward_timed(False)
        torch.cuda.synchronize()
        recs = ctx.timeline_dump()
        ctx.timeline_enable(0)
    finally:
        grp.close()
    return routing, lat, m["latency_ms"] * 1e-3, recs


samples, results = [], {}
for cfg in VALIDATE:
    routing, lat0, lat, recs = run(cfg)
    results[cfg] = (routing, lat0, lat)
    if cfg in FIT:
        samples.append(CM.sample_from_timeline(recs, routing, 0, lat0))
cm = CM.fit(samples)
print("fitted:", cm.to_json_dict())
val = []
for cfg, (routing, lat0, lat) in results.items():
    pred = max(CM.simulate(routing, r, cm, cfg[5]) for r in range(routing.parallel.world_size))
    val.append({"config": list(cfg), "measured_ms": round(lat * 1e3, 4), "predicted_ms": round(float(pred) * 1e3, 4),
                "rel_err": round(float(pred) / lat - 1, 3), "fitted_on": cfg in FIT})
    print(val[-1])
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "costmodel_b200.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
with open(out, "w") as fh:
    json.dump({"model": cm.to_json_dict(), "validation": val,
               "how": "tools/fit_costmodel.py: least squares over measured MMA / dispatch-item intervals "
                      "(per-CTA %globaltimer timelines of emulated rank 0), fixed = latency - kernel span"},
              fh, indent=1)
print("wrote", out)
