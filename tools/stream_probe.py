"""Timeline of the single-GPU host forwards, Mixtral EP=1: MODE=stream
(comet_forward_host), MODE=zc (comet_forward_zerocopy), MODE=dev (device
resident comet_forward, for comparison)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import rank_weights_random  # noqa: E402
from paper_2502_19811_b200 import LayerKnobs, ModelConfig, MoELayer, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402

M, N = 8192, 4096
model = ModelConfig(L=1, E=8, topk=2, N=N, K=14336)
par = ParallelSpec()
routing = build_routing(model, par, WorkloadSpec(M=M, seed=0))
g0 = int(os.environ.get("G0", 8))
nc = int(os.environ.get("NC0", 32))
layer = MoELayer(model, par, 0, M, rank_weights_random(model, par, 0, torch.device("cuda", 0)),
                 knobs=LayerKnobs(n_comm0=nc, group0=g0, zc_order=int(os.environ.get("ZC_ORDER", 0)) or None))
x_host = torch.randn(M, N).to(torch.bfloat16).pin_memory()
ex_host = torch.from_numpy(routing.as_array().copy()).pin_memory()
y_host = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
mode = os.environ.get("MODE", "stream")
ex_dev = ex_host.cuda()
y_dev = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
x_dev = x_host.cuda()
layer.place_tokens(x_dev, M)
for chunks in ((8, 16) if mode == "stream" else (0,)):
    def run():
        if mode == "stream":
            layer.ctx.forward_host(x_host, ex_host, None, y_host, M, layer.weights.w0t, layer.weights.w1t, 0,
                                   n_comm0=nc, group0=g0, wave1=4, chunks=chunks)
        elif mode == "zc":
            layer.ctx.forward_zerocopy(x_host, ex_host, None, y_host, M, layer.weights.w0t, layer.weights.w1t, 0,
                                       n_comm0=nc, group0=g0, wave1=4)
        else:
            layer.run(ex_dev, M, y_dev)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        run()
    e.record()
    torch.cuda.synchronize()
    print(f"{mode} chunks={chunks}: {s.elapsed_time(e) / 10:.3f} ms per forward")
layer.ctx.timeline_enable(1024)
torch.cuda.synchronize()
t_host = torch.cuda.Event(enable_timing=True)
run()
torch.cuda.synchronize()
recs = layer.ctx.timeline_dump()
life = [r for r in recs if r[1] == "tmem_wait" and r[2] == (1 << 20) - 2]
recs = [r for r in recs if not (r[1] == "tmem_wait" and r[2] == (1 << 20) - 2)]
t0 = min(r[3] for r in recs)
if life:
    print(f"CTA exits: first {(min(r[4] for r in life) - t0) / 1e3:.0f}, last {(max(r[4] for r in life) - t0) / 1e3:.0f} us")
by = {}
for c, role, task, s_, e_ in recs:
    by.setdefault(role, []).append((task, (s_ - t0) / 1e3, (e_ - t0) / 1e3, c))
comm = sorted(by.get("comm", []), key=lambda r: r[2])
print(f"span {max(r[4] for r in recs) / 1e3 - t0 / 1e3:.1f} us")
if comm:
    print(f"dispatch items {len(comm)}: done at 10% {comm[len(comm) // 10][2]:.0f} 50% {comm[len(comm) // 2][2]:.0f} "
          f"100% {comm[-1][2]:.0f} us")
P = int(layer.ctx.index_meta()[3])
U0 = P * 28
ilv = int(os.environ.get("COMET_ZC_ILV", 1)) if mode == "zc" else 0


def seq_layer(g):
    """Sequence index -> layer (the interleaved zero-copy sequence, unit_at)."""
    if ilv <= 0:
        return 0 if g < U0 else 1
    n_g = (P + g0 - 1) // g0
    for k in range(n_g + ilv):
        if k < n_g:
            sz = min(g0, P - k * g0) * 28
            if g < sz:
                return 0
            g -= sz
        if k >= ilv:
            sz = min(g0, P - (k - ilv) * g0) * 8
            if g < sz:
                return 1
            g -= sz
    return 1


mma = by["mma"]
l0 = sorted(e for t, s_, e, c in mma if seq_layer(t) == 0)
l1 = sorted(s_ for t, s_, e, c in mma if seq_layer(t) == 1)
l0s = sorted(s_ for t, s_, e, c in mma if seq_layer(t) == 0)
print(f"layer0 units: first start {l0s[0]:.0f}, 10% started {l0s[len(l0s) // 10]:.0f}")
print(f"layer0 units {len(l0)}: 10% done {l0[len(l0) // 10]:.0f} 50% {l0[len(l0) // 2]:.0f} last {l0[-1]:.0f} us")
print(f"layer1 units {len(l1)}: first start {l1[0]:.0f}, last end {max(e for t, s_, e, c in mma if seq_layer(t) == 1):.0f} us")
ld = {(c, t): s_ for t, s_, e, c in by["load"]}
d0 = [e - max(s_, ld.get((c, t), s_)) for t, s_, e, c in mma if seq_layer(t) == 0]
d1 = [e - max(s_, ld.get((c, t), s_)) for t, s_, e, c in mma if seq_layer(t) == 1]
print(f"MMA compute per unit: L0 {statistics.mean(d0):.1f} us, L1 {statistics.mean(d1):.1f} us")
ep = by["epilogue"]
print(f"epilogue: L0 {statistics.mean(e - s_ for t, s_, e, c in ep if seq_layer(t) == 0):.1f} us, "
      f"L1 {statistics.mean(e - s_ for t, s_, e, c in ep if seq_layer(t) == 1):.1f} us (max {max(e - s_ for t, s_, e, c in ep if seq_layer(t) == 1):.1f})")
