"""Index-build phase timing (globaltimer probes in meta[8..14]) for an EP=W rank."""
import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2502_19811_b200 import _lib, config as C, routing as Rt
W = int(sys.argv[1]) if len(sys.argv) > 1 else 1
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
r = Rt.build_routing(C.ModelConfig(L=1, E=8, topk=2, N=4096, K=14336), C.ParallelSpec(1, W), C.WorkloadSpec(M=8192))
ctxs = [_lib.Context(rank=i, world=W, tp=1, ep=W, device=0, E=8, topk=2, N=4096, K=14336, m_cap=8192) for i in range(W)]
if W > 1:
    _lib.Context.link_local(ctxs)
ctx = ctxs[0]
ex = torch.from_numpy(r.as_array().copy()).cuda()
for i in range(3):
    ctx.index_build(ex, 8192, flags=flags)
    m = ctx.index_meta()
    print("cta0: phase1a %d, 1b %d, barrier %d, phase2 %d | last cta: phase3 start %d end %d" % tuple(m[8:14]))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for i in range(20): ctx.index_build(ex, 8192, flags=flags)
e.record(); torch.cuda.synchronize(); print("per build us", s.elapsed_time(e) / 20 * 1e3)
s.record()
for i in range(20): ctx.signal_tokens_ready()
e.record(); torch.cuda.synchronize(); print("per signal us", s.elapsed_time(e) / 20 * 1e3)
