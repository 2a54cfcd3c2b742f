"""Per-pair timeline of one fused (layer0 + layer1) launch of emulated rank 0.

    python tools/fused_timeline.py [--shape MX] [--ep 8] [--tp 1] [--M 8192] [--std 0] [--nc0 8]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19811_b200 import LayerKnobs, ModelConfig, ParallelSpec, WorkloadSpec, build_routing  # noqa: E402
from paper_2502_19811_b200.measure import EmulatedGroup  # noqa: E402

SHAPES = {"MX": (8, 2, 4096, 14336), "PH": (16, 2, 4096, 6400), "QW": (64, 8, 3584, 2560)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="MX")
ap.add_argument("--ep", type=int, default=8)
ap.add_argument("--tp", type=int, default=1)
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--std", type=float, default=0.0)
ap.add_argument("--nc0", type=int, default=8)
ap.add_argument("--g0", type=int, default=4)
ap.add_argument("--wave1", type=int, default=4)
ap.add_argument("--pairs", type=int, default=8, help="pairs to print in detail")
ap.add_argument("--knobs", default="", help="extra LayerKnobs fields, e.g. streamk=0")
a = ap.parse_args()
E, topk, N, K = SHAPES[a.shape]
model = ModelConfig(L=1, E=E, topk=topk, N=N, K=K)
par = ParallelSpec(a.tp, a.ep)
routing = build_routing(model, par, WorkloadSpec(M=a.M, seed=0, std=a.std))
extra = {k: int(v) for k, v in (kv.split("=") for kv in a.knobs.split(",") if kv)}
grp = EmulatedGroup(model, par, routing, knobs=LayerKnobs(n_comm0=a.nc0, n_comm1=0, group0=a.g0, wave1=a.wave1, **extra))
r = grp.measure(iters=5)
print("measured:", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k != "per_rank_ms"})
l0 = grp.layers[0]
l0.ctx.timeline_enable(512)
grp._forward_timed(False)
torch.cuda.synchronize()
recs = l0.ctx.timeline_dump()
meta = l0.ctx.index_meta()
P = int(meta[3])
kl = K // a.tp
NB0 = -(-kl // 512)
NB1 = -(-N // 512)
U0 = P * NB0
split1 = int(os.environ.get("COMET_SPLIT1", 0))
U1 = P * NB1
full1 = U1 - min(U1, split1)
LIFE = (1 << 20) - 2
life = [x for x in recs if x[1] == "tmem_wait" and x[2] == LIFE]
recs = [x for x in recs if not (x[1] == "tmem_wait" and x[2] == LIFE)]
t0 = min(x[3] for x in recs)
span = max(x[4] for x in recs) - t0
print(f"rank0: P={P} NB0={NB0} NB1={NB1} U0={U0} U1={U1} (halves from layer1 unit {full1}); span {span/1e3:.1f} us")


def kind(g):
    if g < U0:
        return "L0"
    return "L1h" if g - U0 >= full1 else "L1"


by_role = {}
for c, role, task, s, e in recs:
    by_role.setdefault(role, []).append((c, task, s - t0, e - t0))
for role, xs in sorted(by_role.items()):
    print(f"  {role:9s} n={len(xs):5d} first +{min(x[2] for x in xs)/1e3:7.1f} last +{max(x[3] for x in xs)/1e3:7.1f}")
mma = by_role.get("mma", [])
for k in ("L0", "L1", "L1h"):
    d = [x[3] - x[2] for x in mma if kind(x[1]) == k]
    if d:
        print(f"  MMA {k:3s}: n={len(d):4d} mean {statistics.mean(d)/1e3:7.2f} us  min {min(d)/1e3:7.2f}  max {max(d)/1e3:7.2f}")
    d = [x[3] - x[2] for x in by_role.get("tmem_wait", []) if kind(x[1]) == k]
    if d:
        print(f"  TMW {k:3s}: n={len(d):4d} mean {statistics.mean(d)/1e3:7.2f} us  max {max(d)/1e3:7.2f}")
    d = [x[3] - x[2] for x in by_role.get("load", []) if kind(x[1]) == k]
    if d:
        print(f"  LD  {k:3s}: n={len(d):4d} mean {statistics.mean(d)/1e3:7.2f} us  max {max(d)/1e3:7.2f}")
    d = [(x[3] - x[2], x[3]) for x in by_role.get("epilogue", []) if kind(x[1]) == k]
    if d:
        print(f"  EPI {k:3s}: n={len(d):4d} mean {statistics.mean(v for v, _ in d)/1e3:7.2f} us  max {max(v for v, _ in d)/1e3:7.2f}"
              f"  last end +{max(e for _, e in d)/1e3:7.1f}")
# per pair (leader CTA) chronology
pairs = {}
for c, task, s, e in mma:
    pairs.setdefault(c, []).append((s, e, task))
loads = {(c, t): (s, e) for c, t, s, e in by_role.get("load", [])}
ends = []
for c in sorted(pairs):
    xs = sorted(pairs[c])
    busy = sum(e - s for s, e, _ in xs)
    ends.append((xs[-1][1], c))
    if c // 2 < a.pairs or c >= 2 * (74 - 4):
        line = " ".join(f"{kind(t)}#{t}[{s/1e3:.0f}-{e/1e3:.0f}|ld{loads.get((c, t), (0, 0))[0]/1e3:.0f}]" for s, e, t in xs)
        print(f"  cta {c:3d}: units {len(xs):2d} busy {busy/1e3:6.1f} us | {line}")
ends.sort()
for e, c in ends[-4:]:
    xs = sorted(pairs[c])
    print(f"  late cta {c:3d}: " + " ".join(f"{kind(t)}[{s/1e3:.0f}-{e2/1e3:.0f}|ld{loads.get((c, t), (0, 0))[0]/1e3:.0f}]"
                                            for s, e2, t in xs))
print("pair end times (us): min %.1f median %.1f max %.1f" % (ends[0][0] / 1e3, ends[len(ends) // 2][0] / 1e3,
                                                            ends[-1][0] / 1e3))
if life:
    print("CTA lifetime: entry first %+.1f last %+.1f us | exit first %+.1f last %+.1f us (rel. to first record)" % (
        (min(x[3] for x in life) - t0) / 1e3, (max(x[3] for x in life) - t0) / 1e3,
        (min(x[4] for x in life) - t0) / 1e3, (max(x[4] for x in life) - t0) / 1e3))
if os.environ.get("TAIL"):
    # the last epilogues: (cta, task, mma start/end, epilogue start/end)
    mm = {(c, t): (s, e) for c, t, s, e in mma}
    epi = sorted(by_role.get("epilogue", []), key=lambda x: x[3])[-int(os.environ["TAIL"]):]
    for c, t, s, e in epi:
        ms, me = mm.get((c & ~1, t), mm.get((c, t), (0, 0)))
        print(f"  tail epi cta {c:3d} {kind(t)}#{t}: mma {ms/1e3:6.1f}-{me/1e3:6.1f}  epi {s/1e3:6.1f}-{e/1e3:6.1f}")
comm = by_role.get("comm", [])
if comm:
    print(f"  dispatch: {len(comm)} tiles, last published +{max(x[3] for x in comm)/1e3:.1f} us")
grp.close()
if comm and os.environ.get("DISP"):
    # dispatch CTAs: items (storer start -> tile publication) per CTA
    per = {}
    for c, task, s, e in comm:
        per.setdefault(c, []).append((s, e, task))
    starts = sorted(min(x[0] for x in v) for v in per.values())
    ends = sorted(max(x[1] for x in v) for v in per.values())
    print(f"  dispatch CTAs {len(per)}: first item start min {starts[0]/1e3:.1f} max {starts[-1]/1e3:.1f} us;"
          f" last publication min {ends[0]/1e3:.1f} median {ends[len(ends)//2]/1e3:.1f} max {ends[-1]/1e3:.1f} us")
    for c in sorted(per)[:4] + sorted(per)[-4:]:
        xs = sorted(per[c])
        print(f"   cta {c:3d}: " + " ".join(f"q{t}[{s/1e3:.1f}-{e/1e3:.1f}]" for s, e, t in xs[:10]))
if os.environ.get("GAPS"):
    # per pair: MMA busy, gaps before each unit (claim / operand / TMEM waits)
    tmw = {(c, t): (s, e) for c, t, s, e in by_role.get("tmem_wait", [])}
    tot_busy = tot_gap = tot_head = tot_tail = 0.0
    span_end = max(e for xs in pairs.values() for _, e, _ in xs)
    for c in sorted(pairs):
        xs = sorted(pairs[c])
        busy = sum(e - s for s, e, _ in xs)
        gaps = sum(xs[i + 1][0] - xs[i][1] for i in range(len(xs) - 1))
        tot_busy += busy; tot_gap += gaps; tot_head += xs[0][0]; tot_tail += span_end - xs[-1][1]
    n = len(pairs)
    print(f"  pairs {n}: mean busy {tot_busy/n/1e3:.1f} us, gaps {tot_gap/n/1e3:.1f}, head {tot_head/n/1e3:.1f}, "
          f"tail to last MMA end {tot_tail/n/1e3:.1f} (span to last MMA end {span_end/1e3:.1f})")
    # MMA intervals include in-loop waits: operand (load) waits show as load start after claim
    for k in ("L0", "L1", "L1h"):
        d = [loads[(c, t)][0] - s for c, xs in pairs.items() for s, e, t in xs if kind(t) == k and (c, t) in loads]
        if d:
            print(f"  {k}: first load after MMA-start mean {statistics.mean(d)/1e3:.2f} us max {max(d)/1e3:.2f}")
