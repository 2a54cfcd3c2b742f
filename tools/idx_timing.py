import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2502_19811_b200 import _lib, config as C, routing as Rt
r = Rt.build_routing(C.ModelConfig(L=1, E=8, topk=2, N=4096, K=14336), C.ParallelSpec(1, 1), C.WorkloadSpec(M=8192))
ctx = _lib.Context(rank=0, world=1, tp=1, ep=1, device=0, E=8, topk=2, N=4096, K=14336, m_cap=8192)
ex = torch.from_numpy(r.as_array().copy()).cuda()
for i in range(5):
    ctx.index_build(ex, 8192, flags=0)
    m = ctx.index_meta()
    print("hist %d, phase1 %d, end %d | p2 start %d, tiles0 done %d, tiles1 done %d, pairs done %d" % (m[8], m[9], m[10], m[11], m[12], m[13], m[14]))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for i in range(20): ctx.index_build(ex, 8192, flags=0)
e.record(); torch.cuda.synchronize(); print("per build us", s.elapsed_time(e) / 20 * 1e3)
