"""Measurement matrix of SURVEY.md §8(d) on one B200.

Every configuration runs the full fused forward with all EP x TP ranks
emulated on this GPU (paper_2502_19811_b200.measure.EmulatedGroup): latency =
max over ranks of the rank's kernel-time sum.  EP=1 rows are real
single-GPU forwards.  Every row also times the unfused all-to-all + cuBLAS
grouped-GEMM path (EP > 1: measure.EmulatedUnfused, the same emulation).
Roofline per §8(d) at the measured burst and sustained bf16 peaks.

    python tools/matrix.py [--quick] [--out gpurun_out/matrix.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import load_peaks  # noqa: E402
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402
from paper_2502_19811_b200.measure import EmulatedGroup, roofline  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}


def configs(quick):
    out = [("MX", 1, 1, 8192, 0.0), ("MX", 8, 1, 8192, 0.0), ("MX", 4, 1, 8192, 0.0), ("MX", 2, 1, 8192, 0.0),
           ("MX", 8, 1, 8192, 0.032), ("MX", 8, 1, 8192, 0.05), ("PH", 4, 2, 8192, 0.0), ("QW", 8, 1, 8192, 0.0),
           ("QW", 8, 1, 8192, 0.032), ("PH", 1, 1, 8192, 0.0), ("QW", 1, 1, 8192, 0.0)]
    if not quick:
        for ep in (1, 2, 4, 8):
            for std in (0.0, 0.032):
                for M in (1024, 2048, 4096, 8192, 16384, 32768):
                    c = ("MX", ep, 1, M, std)
                    if c not in out:
                        out.append(c)
    return out


SPEC_BF16_TFLOPS = 2250.0  # nominal dense bf16 (B200 spec sheet), labelled as such


def extra_terms(routing, latency_ms, hbm_gbs):
    """SURVEY §8(d)'s secondary terms: the spec-peak roofline variant and the
    weight-streaming time max_r(E_r * 2 * N * K/tp * 2 B) / HBM."""
    model, par = routing.model, routing.parallel
    rf = roofline(routing, SPEC_BF16_TFLOPS)
    w_bytes = (model.E // par.ep) * 2 * model.N * (model.K // par.tp) * 2
    return {"roofline_ms_spec_2250tf": round(rf.ms, 4), "pct_roofline_spec": round(100 * rf.ms / latency_ms, 1),
            "t_weights_hbm_ms": round(w_bytes / (hbm_gbs * 1e9) * 1e3, 4)}


def unfused_ms(grp, iters=10):
    from paper_2502_19811_b200.unfused import UnfusedLayer
    l = grp.layers[0]
    m = grp.model
    kl = m.K
    ul = UnfusedLayer(m, grp.parallel, 0, l.weights.w0t[:, :kl, :m.N].transpose(1, 2).contiguous(),
                      l.weights.w1t[:, :m.N, :kl].transpose(1, 2).contiguous())
    x = l.ctx.token_buffer()[:grp.M, :m.N]
    for _ in range(3):
        ul.forward(x, grp.ex, M=grp.M)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        ul.forward(x, grp.ex, M=grp.M)
    e.record()
    torch.cuda.synchronize()
    del ul
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "matrix.jsonl"))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--knobs", default="", help="extra LayerKnobs fields, e.g. streamk=0,split1=16")
    ap.add_argument("--reps", type=int, default=1, help="measure each config this many times (best kept)")
    ap.add_argument("--only", default="", help="comma list of SHAPE:EP:TP:M:STD (replaces the matrix)")
    ap.add_argument("--nc0", default="auto",
                    help="layer0 comm-CTA counts tried for EP>1 (best kept); 'auto' = the product chooser "
                         "(assigner.choose_split on split_b200.json)")
    a = ap.parse_args()
    burst, sust, hbm, src = load_peaks()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        todo = configs(a.quick)
        if a.only:
            todo = [(f[0], int(f[1]), int(f[2]), int(f[3]), float(f[4])) for f in
                    (c.split(":") for c in a.only.split(","))]
        for shape, ep, tp, M, std in todo:
            E, topk, N, K = SHAPES[shape]
            model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
            par = ParallelSpec(tp=tp, ep=ep)
            routing = build_routing(model, par, WorkloadSpec(M=M, seed=0, std=std))
            rf_b, rf_s = roofline(routing, burst), roofline(routing, sust)
            t0 = time.time()
            extra = {k: int(v) for k, v in (kv.split("=") for kv in a.knobs.split(",") if kv)}
            grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs(n_comm0=2, n_comm1=0, **extra))
            best = None
            cands = [0] if par.world_size == 1 else ([None] if a.nc0 == "auto" else [int(v) for v in a.nc0.split(",")])
            for nc0 in cands * a.reps:
                grp.set_knobs(LayerKnobs.for_world(par.world_size, n_comm0=nc0, n_comm1=0, **extra))
                r = grp.measure(iters=a.iters)
                r["n_comm0"] = grp.layers[0].n_comm0(M) if nc0 is None else nc0
                if best is None or r["latency_ms"] < best["latency_ms"]:
                    best = r
            rec = {"knobs": a.knobs, "shape": shape, "E": E, "topk": topk, "N": N, "K": K, "ep": ep, "tp": tp, "M": M, "std": std,
                   "emulated": par.world_size > 1, "latency_ms": round(best["latency_ms"], 4),
                   "hot_rank": best["hot_rank"], "n_comm0": best["n_comm0"],
                   "chained_mean_ms": round(best.get("chained_mean_ms", 0.0), 4),
                   "kernels_ms_hot_rank": {k: round(v, 4) for k, v in best["kernels_ms_hot_rank"].items()},
                   "roofline_ms_burst": round(rf_b.ms, 4), "roofline_ms_sustained": round(rf_s.ms, 4),
                   "roofline_bound": rf_b.bound, "t_nvlink_ms": round(rf_b.t_nvlink_ms, 4),
                   "pct_roofline_burst": round(100 * rf_b.ms / best["latency_ms"], 1),
                   "pct_roofline_sustained": round(100 * rf_s.ms / best["latency_ms"], 1),
                   "peaks": {"burst_tflops": burst, "sustained_tflops": sust, "source": src}}
            rec.update(extra_terms(routing, rec["latency_ms"], hbm))
            try:
                if par.world_size == 1:
                    u = unfused_ms(grp)
                else:  # every rank emulated: all-to-alls as HBM copies (measure.EmulatedUnfused)
                    from paper_2502_19811_b200.measure import EmulatedUnfused
                    u = EmulatedUnfused(grp).measure(iters=a.iters)["latency_ms"]
                    torch.cuda.empty_cache()
                rec["unfused_ms"] = round(u, 4)
                rec["speedup_vs_unfused"] = round(u / best["latency_ms"], 3)
            except Exception as exc:  # report, keep going
                rec["unfused_error"] = repr(exc)[:200]
            grp.close()
            del grp
            torch.cuda.empty_cache()
            rec["wall_s"] = round(time.time() - t0, 1)
            print(json.dumps(rec), flush=True)
            fh.write(json.dumps(rec) + "\n")
            fh.flush()


if __name__ == "__main__":
    main()
