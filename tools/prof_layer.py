"""Per-layer timing of the fused kernels at a bench shape (EP=1)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_19811_b200 import _lib
from paper_2502_19811_b200 import config as C, routing as Rt

ap = argparse.ArgumentParser()
ap.add_argument("--E", type=int, default=8); ap.add_argument("--topk", type=int, default=2)
ap.add_argument("--N", type=int, default=4096); ap.add_argument("--K", type=int, default=14336)
ap.add_argument("--M", type=int, default=8192); ap.add_argument("--std", type=float, default=0.0)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--once", action="store_true", help="single forward (for ncu)")
a = ap.parse_args()

model = C.ModelConfig(L=1, E=a.E, topk=a.topk, N=a.N, K=a.K)
r = Rt.build_routing(model, C.ParallelSpec(1, 1), C.WorkloadSpec(M=a.M, seed=0, std=a.std))
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(a.M, a.N, device="cuda", generator=g).to(torch.bfloat16)
w0t = (torch.randn(a.E, a.K, a.N, device="cuda", generator=g) / a.N ** 0.5).to(torch.bfloat16)
w1t = (torch.randn(a.E, a.N, a.K, device="cuda", generator=g) / a.K ** 0.5).to(torch.bfloat16)
ex = torch.from_numpy(r.as_array().copy()).cuda()
ctx = _lib.Context(rank=0, world=1, tp=1, ep=1, device=0, E=a.E, topk=a.topk, N=a.N, K=a.K, m_cap=a.M)
ctx.token_buffer()[:a.M].copy_(x)
y = torch.empty(a.M, a.N, dtype=torch.bfloat16, device="cuda")
flops = 2.0 * a.M * a.topk * a.N * a.K

if a.once:
    ctx.forward(ex, a.M, w0t, w1t, None, y, n_comm0=0, n_comm1=0, group0=8, wave1=4)
    torch.cuda.synchronize()
    sys.exit(0)

def timeit(fn, n=a.iters):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n

ctx.index_build(ex, a.M)
t_idx = timeit(lambda: ctx.index_build(ex, a.M))
configs = [(16, 4, 0)]
if a.sweep:
    configs = [(g0, 4, 0) for g0 in (1, 2, 4, 8, 16, 32, 64)] + [(16, w1, 0) for w1 in (1, 2, 8, 16)]
for g0, w1, nc in configs:
    t0 = timeit(lambda: ctx.layer0(w0t, 0, nc, g0))
    t1 = timeit(lambda: ctx.layer1(w1t, None, y, nc, w1))
    tf = timeit(lambda: ctx.forward(ex, a.M, w0t, w1t, None, y, n_comm0=nc, n_comm1=nc, group0=g0, wave1=w1))
    print(f"group0={g0:3d} wave1={w1:2d} n_comm1={nc}: index {t_idx*1e3:7.1f} us | layer0 {t0:7.3f} ms "
          f"({flops/t0/1e9:6.1f} TF/s) | layer1 {t1:7.3f} ms ({flops/t1/1e9:6.1f} TF/s) | forward {tf:7.3f} ms", flush=True)
# torch reference GEMM rate for this shape (one expert, cuBLAS)
xa = torch.randn(a.M * a.topk // a.E, a.N, device="cuda", dtype=torch.bfloat16)
tb = timeit(lambda: [xa @ w0t[e].t() for e in range(a.E)])
print(f"cuBLAS per-expert loop layer0-shape: {tb:.3f} ms ({flops/tb/1e9:.1f} TF/s)")
