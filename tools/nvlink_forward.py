"""One process driving EP GPUs (comet_link_local, peer access over NVLink):
the Mixtral MoE layer forward with every rank on its own B200, for ncu's
NVLink counters (tools/ncu_nvlink.sh) and a device-timed latency.

    python tools/nvlink_forward.py [--ep 8] [--M 8192] [--iters 20]

Needs EP visible GPUs (exits with a message otherwise).  Latency = max over
ranks of the rank's CUDA-event time around its forward (index build, layer
kernel, remote-combine finish), all ranks enqueued back to back.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, MoELayer, ParallelSpec, WorkloadSpec, _lib, build_routing  # noqa: E402
from paper_2502_19811_b200.measure import NVLINK_GBS, distinct_remote_pairs, roofline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ep", type=int, default=8)
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--std", type=float, default=0.0)
    a = ap.parse_args()
    if torch.cuda.device_count() < a.ep:
        print(f"needs {a.ep} GPUs, {torch.cuda.device_count()} visible")
        return 0
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import load_peaks, rank_weights_random
    model = ModelConfig(L=1, E=8, topk=2, N=4096, K=14336)
    par = ParallelSpec(1, a.ep)
    routing = build_routing(model, par, WorkloadSpec(M=a.M, seed=0, std=a.std))
    layers = []
    for r in range(a.ep):
        with torch.cuda.device(r):
            layers.append(MoELayer(model, par, r, a.M, rank_weights_random(model, par, r, torch.device("cuda", r)),
                                   device=r, knobs=LayerKnobs.for_world(a.ep)))
    _lib.Context.link_local([l.ctx for l in layers])
    ex, ys = [], []
    for l in layers:
        lo, hi = l.token_range(a.M)
        with torch.cuda.device(l.device):
            g = torch.Generator(device=f"cuda:{l.device}").manual_seed(7 + l.rank)
            l.place_tokens(torch.randn(hi - lo, model.N, device=f"cuda:{l.device}", generator=g).to(torch.bfloat16), a.M)
            ex.append(torch.from_numpy(routing.as_array().copy()).cuda(l.device))
            ys.append(torch.empty(hi - lo, model.N, dtype=torch.bfloat16, device=f"cuda:{l.device}"))

    def forward(events=None):
        for i, l in enumerate(layers):
            with torch.cuda.device(l.device):
                if events:
                    events[i][0].record()
                l.run(ex[i], a.M, ys[i])
                if events:
                    events[i][1].record()

    for _ in range(3):
        forward()
    for l in layers:
        torch.cuda.synchronize(l.device)
    per_rank = [[] for _ in layers]
    for _ in range(a.iters):
        evs = []
        for l in layers:
            with torch.cuda.device(l.device):
                evs.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
        forward(evs)
        for l in layers:
            torch.cuda.synchronize(l.device)
        for i in range(len(layers)):
            per_rank[i].append(evs[i][0].elapsed_time(evs[i][1]))
    lat = max(sorted(t)[len(t) // 2] for t in per_rank)
    burst = load_peaks()[0]
    rf = roofline(routing, burst)
    d_out, d_in = distinct_remote_pairs(routing)
    print(f"EP={a.ep} M={a.M}: latency {lat:.4f} ms (max over ranks, median of {a.iters}); roofline {rf.ms:.4f} ms "
          f"({100 * rf.ms / lat:.1f}%); rank-0 dispatch-in {int(d_in[0]) * 2 * model.N / 1e6:.1f} MB, "
          f"NVLink term {rf.t_nvlink_ms:.4f} ms at {NVLINK_GBS} GB/s")
    for l in layers:
        l.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
