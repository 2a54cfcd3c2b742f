"""Per-role timeline statistics of the fused layer kernels (one forward)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_19811_b200 import _lib
from paper_2502_19811_b200 import config as C, routing as Rt

E, topk, N, K, M = 8, 2, 4096, 14336, 8192
args = sys.argv[1:]
model = C.ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
r = Rt.build_routing(model, C.ParallelSpec(1, 1), C.WorkloadSpec(M=M, seed=0))
g = torch.Generator(device="cuda").manual_seed(0)
w0t = (torch.randn(E, K, N, device="cuda", generator=g) / N ** 0.5).to(torch.bfloat16)
w1t = (torch.randn(E, N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
ex = torch.from_numpy(r.as_array().copy()).cuda()
ctx = _lib.Context(rank=0, world=1, tp=1, ep=1, device=0, E=E, topk=topk, N=N, K=K, m_cap=M)
ctx.token_buffer()[:M].copy_(torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16))
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
g0 = int(os.environ.get("G0", 16)); w1 = int(os.environ.get("W1", 4))
for _ in range(3):
    ctx.forward(ex, M, w0t, w1t, None, y, n_comm0=0, n_comm1=0, group0=g0, wave1=w1)
torch.cuda.synchronize()
ctx.timeline_enable(256)
for layer in (0, 1):
    ctx.index_build(ex, M)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if layer == 0:
        ctx.layer0(w0t, 0, 0, g0)
    else:
        ctx.layer0(w0t, 0, 0, g0); torch.cuda.synchronize(); ctx.timeline_dump(); s.record()
        ctx.layer1(w1t, None, y, 0, w1)
    e.record(); torch.cuda.synchronize()
    recs = ctx.timeline_dump()
    t0 = min(r[3] for r in recs); t1 = max(r[4] for r in recs)
    print(f"== layer{layer}: kernel(s) {s.elapsed_time(e):.3f} ms, timeline span {(t1-t0)/1e6:.3f} ms, {len(recs)} records")
    for role in ("load", "mma", "tmem_wait", "epilogue"):
        d = [r[4] - r[3] for r in recs if r[1] == role]
        if not d:
            continue
        per_cta = {}
        for r_ in recs:
            if r_[1] == role:
                per_cta[r_[0]] = per_cta.get(r_[0], 0) + r_[4] - r_[3]
        busy = statistics.mean(per_cta.values()) / (t1 - t0)
        print(f"   {role:10s} n={len(d):5d} mean={statistics.mean(d)/1e3:8.2f}us p50={statistics.median(d)/1e3:8.2f}us max={max(d)/1e3:8.2f}us  busy/cta={busy:6.1%}")
    # first start / last end per role
    firsts = sorted(r[3] for r in recs if r[1] == "mma")[:3]
    lasts = sorted(r[4] for r in recs if r[1] == "epilogue")[-3:]
    print(f"   first mma starts at +{(firsts[0]-t0)/1e3:.1f}us; last epilogue ends at +{(lasts[-1]-t0)/1e3:.1f}us")
