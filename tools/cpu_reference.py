"""The reference algorithm timed on this box's host cores (SURVEY.md §8(d)'s
CPU baseline, reported, not optimised): the literal execute_naive loop nest
(oracle.execute_naive_literal, bitwise equal to the reference) at Config 1,
and the vectorised restatement (oracle.layer_forward / layer_forward_tp, one
GEMM pair per expert, validated against the literal oracle and the
reference's own outputs by tests/test_oracle_golden.py) in fp32 and fp64 on
the FULL layer of every BASELINE shape (all tokens, all experts; the EP / TP
partition does not change the CPU work).  Test infrastructure only -- the
oracle is the checker, never the product path.  Prints one JSON line.

    python tools/cpu_reference.py [--reps 1]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from bench import _blas_threads  # noqa: E402
from oracle import moe_oracle as O  # noqa: E402
from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336, 1, 8), "PH": (16, 2, 4096, 6400, 2, 4), "QW": (64, 8, 3584, 2560, 1, 8)}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--skip-fp64", action="store_true")
a = ap.parse_args()
limits, threads = _blas_threads()
out = {"host_cpu_count": os.cpu_count(), "blas_threads": threads}
with limits:
    c1 = ModelConfig(L=1, E=8, topk=2, N=512, K=1024)
    r1 = build_routing(c1, ParallelSpec(tp=1, ep=8), WorkloadSpec(M=512, seed=0, std=0.0))
    g = np.random.default_rng(1)
    x1 = g.standard_normal((512, 512))
    w01 = g.standard_normal((8, 512, 1024)) / math.sqrt(512)
    w11 = g.standard_normal((8, 1024, 512)) / math.sqrt(512)
    t0 = time.perf_counter()
    y_lit = O.execute_naive_literal(x1, w01, w11, r1.as_array())
    out["c1_literal_execute_naive_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
    t0 = time.perf_counter()
    y_vec = O.layer_forward(x1, w01, w11, r1.as_array())
    out["c1_vectorised_fp64_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    out["c1_vectorised_vs_literal_max_abs"] = float(np.abs(y_vec - y_lit).max())
    for name, (E, topk, N, K, tp, ep) in SHAPES.items():
        model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
        routing = build_routing(model, ParallelSpec(tp=tp, ep=ep), WorkloadSpec(M=8192, seed=0, std=0.0))
        ex = routing.as_array()
        rng = np.random.default_rng(3)
        for dt, tag in ((np.float32, "fp32"), (np.float64, "fp64")):
            if dt is np.float64 and a.skip_fp64:
                continue
            x = rng.standard_normal((8192, N)).astype(dt)
            w0 = (rng.standard_normal((E, N, K)) / math.sqrt(N)).astype(dt)
            w1 = (rng.standard_normal((E, K, N)) / math.sqrt(K)).astype(dt)
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                if tp == 1:
                    O.layer_forward(x, w0, w1, ex, dtype=dt)
                else:
                    O.layer_forward_tp(x, w0, w1, ex, tp, dtype=dt)
                ts.append(time.perf_counter() - t0)
            out[f"{name}_{tag}_ms"] = round(min(ts) * 1e3, 1)
            del x, w0, w1
print(json.dumps(out))
