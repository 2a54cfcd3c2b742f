"""Measure the n_c (layer0 dispatch CTA) curve of the fused layer on B200 for
the BASELINE shapes and write the product chooser's metadata
(paper_2502_19811_b200/split_b200.json, the reference's SplitMetadata schema,
assigner.py:44-197; cost "b200", blocks = SM count).

Every rank of a configuration is emulated on the one GPU
(measure.EmulatedGroup: latency = max over ranks of the rank's kernel time,
other knobs at LayerKnobs.for_world).  World-1 shapes have no dispatch CTAs
and are not swept.

    python tools/sweep_b200.py [--quick] [--out paper_2502_19811_b200/split_b200.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec  # noqa: E402
from paper_2502_19811_b200.assigner import SplitMetadata, sweep_split  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}
CANDIDATES = [8, 16, 24, 32, 48, 64, 80, 96]
GROUPS = [2, 4, 8]  # layer0 pair-group sizes swept jointly with n_c (SplitRecord.group0)


def configs(quick):
    out = []
    for ep in (2, 4, 8):
        for M in ((8192,) if quick else (1024, 2048, 4096, 8192, 16384, 32768)):
            out.append(("MX", ep, 1, M))
    for M in ((8192,) if quick else (2048, 8192, 32768)):
        out.append(("PH", 4, 2, M))
        out.append(("QW", 8, 1, M))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2502_19811_b200", "split_b200.json"))
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--passes", type=int, default=3, help="round-robin passes over the grid, minimum per point")
    a = ap.parse_args()
    meta = SplitMetadata(records=[])
    for shape, ep, tp, M in configs(a.quick):
        E, topk, N, K = SHAPES[shape]
        model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
        t0 = time.time()
        rec = sweep_split(model, ParallelSpec(tp=tp, ep=ep), WorkloadSpec(M=M, seed=0, std=0.0),
                          cost_name="b200", candidates=CANDIDATES, repeats=a.repeats, groups=GROUPS,
                          passes=a.passes)
        meta.add(rec)
        torch.cuda.empty_cache()
        print(json.dumps({"shape": shape, "ep": ep, "tp": tp, "M": M, "optimal_nc": rec.optimal_nc,
                          "group0": rec.group0,
                          "latency_ms": rec.latency_ns / 1e6, "curve_ms": {nc: ns / 1e6 for nc, ns in rec.curve},
                          "wall_s": round(time.time() - t0, 1)}), flush=True)
        meta.save(a.out)
    print("wrote", a.out, len(meta.records), "records")


if __name__ == "__main__":
    main()
