"""Per-rank kernel times of an EP=W layer emulated on one GPU (all ranks'
heaps on this device; NVLink traffic becomes local HBM traffic)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing
from paper_2502_19811_b200.executor import MoELayer, RankWeights, _lib

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nc0 = int(os.environ.get("NC0", 2)); nc1 = int(os.environ.get("NC1", 0)); g0 = int(os.environ.get("G0", 4))
E, topk, N, K, M = 8, 2, 4096, 14336, 8192
model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
par = ParallelSpec(1, W)
r = build_routing(model, par, WorkloadSpec(M=M, seed=0))
g = torch.Generator(device="cuda").manual_seed(0)
layers = []
for rank in range(W):
    e_per = E // W
    w0t = (torch.randn(e_per, K, N, device="cuda", generator=g) / 64).to(torch.bfloat16)
    w1t = (torch.randn(e_per, N, K, device="cuda", generator=g) / 64).to(torch.bfloat16)
    layers.append(MoELayer(model, par, rank, M, RankWeights(w0t, w1t), knobs=LayerKnobs(n_comm0=nc0, n_comm1=nc1)))
_lib.Context.link_local([l.ctx for l in layers])
x = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
ex = torch.from_numpy(r.as_array().copy()).cuda()
ys = []
for l in layers:
    lo, hi = l.token_range(M)
    l.place_tokens(x[lo:hi], M)
    ys.append(torch.empty(hi - lo, N, dtype=torch.bfloat16, device="cuda"))
ev = lambda: torch.cuda.Event(enable_timing=True)
res = {k: [] for k in ("index", "layer0", "layer1", "finish", "total")}
for it in range(6):
    ti = []
    for l in layers:
        a, b = ev(), ev(); a.record(); l.ctx.index_build(ex, M, flags=4); b.record()
        ti.append((a, b))
    t = []
    for l in layers:
        a, b = ev(), ev(); a.record(); l.ctx.layer0(l.weights.w0t, 0, nc0, g0); b.record(); t.append((a, b))
    t1 = []
    for l, y in zip(layers, ys):
        a, b = ev(), ev(); a.record(); l.ctx.layer1(l.weights.w1t, None, y, nc1, 4); b.record(); t1.append((a, b))
    t2 = []
    for l, y in zip(layers, ys):
        a, b = ev(), ev(); a.record(); l.ctx.combine_finish(y); b.record(); t2.append((a, b))
    torch.cuda.synchronize()
    if it >= 2:
        res["index"].append(max(a.elapsed_time(b) for a, b in ti))
        res["layer0"].append(max(a.elapsed_time(b) for a, b in t))
        res["total"].append(max(sum(x[0].elapsed_time(x[1]) for x in xs) for xs in zip(ti, t, t1, t2)))
        res["layer1"].append(max(a.elapsed_time(b) for a, b in t1))
        res["finish"].append(max(a.elapsed_time(b) for a, b in t2))
rows = layers[0].ctx.index_meta()[0]
fl = 2.0 * rows * N * K / W * W  # per rank (tp=1): 2*rows*N*K
print(f"EP={W} rank rows={rows}: forward {statistics.median(res['total']):.3f} ms (index {statistics.median(res['index']):.3f}); layer0 {statistics.median(res['layer0']):.3f} ms, layer1 {statistics.median(res['layer1']):.3f} ms, "
      f"finish {statistics.median(res['finish']):.3f} ms (max over ranks); per-layer TF/s "
      f"{2.0*rows*N*K/statistics.median(res['layer0'])/1e9:.0f} / {2.0*rows*N*K/statistics.median(res['layer1'])/1e9:.0f}")

if os.environ.get("TL"):
    # one more forward with timelines on rank 0: per-role busy and spans
    l0 = layers[0]
    l0.ctx.timeline_enable(256)
    for l in layers:
        l.ctx.index_build(ex, M, flags=4)
    for l in layers:
        l.ctx.layer0(l.weights.w0t, 0, nc0, g0)
    torch.cuda.synchronize()
    for tag in ("layer0", "layer1"):
        if tag == "layer1":
            for l, y in zip(layers, ys):
                l.ctx.layer1(l.weights.w1t, None, y, nc1, 4)
            for l, y in zip(layers, ys):
                l.ctx.combine_finish(y)
            torch.cuda.synchronize()
        recs = l0.ctx.timeline_dump()
        t0 = min(r_[3] for r_ in recs)
        print(f"== rank0 {tag}: span {(max(r_[4] for r_ in recs) - t0)/1e3:.1f} us")
        for role in ("load", "mma", "tmem_wait", "epilogue", "comm"):
            d = [r_ for r_ in recs if r_[1] == role]
            if d:
                print(f"   {role:9s} n={len(d):5d} first start +{(min(x[3] for x in d)-t0)/1e3:8.1f}us last end +{(max(x[4] for x in d)-t0)/1e3:8.1f}us mean {statistics.mean(x[4]-x[3] for x in d)/1e3:7.2f}us")
        if tag == "layer1":
            for x in sorted([r_ for r_ in recs if r_[1] == "comm"], key=lambda x: x[3])[:40]:
                print("     comm cta", x[0], "nb", x[2], f"+{(x[3]-t0)/1e3:.1f} .. +{(x[4]-t0)/1e3:.1f}")
