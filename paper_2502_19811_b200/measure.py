"""Measured layer timings and the §8(d) roofline for any (model, EP x TP).

``roofline`` restates SURVEY.md §8(d) / BASELINE.md for one routing:

    FLOPs_r  = 4 * rows_r * N * K/tp            (two expert GEMMs, 2 flop / MAC)
    Bytes_r  = 2 * N * (D_out_r + D_in_r)       bf16 bytes rank r transmits: dispatch
                                                rows it sends + partial rows it pushes back
    T        = max(max_r FLOPs_r / peak_flops, max_r Bytes_r / 900 GB/s)

where rows_r are the (token, expert) rows hosted on r (routing.py:78-84
counts over r's experts, replicated over the TP group) and D are distinct
(token, remote destination rank) pairs (the dedup of the token-slot buffer,
config.py:218-226).

``EmulatedGroup`` runs every rank of a ``ParallelSpec`` on ONE GPU (their
symmetric heaps linked in-process, NVLink traffic becomes HBM traffic) and
times each rank's kernels with CUDA events on the launching stream; a rank's
latency is the sum of its kernel times (index build + layer0 + layer1 +
remote-combine finish) while it has the GPU to itself, and the group latency
is the max over ranks -- the per-GPU time of a real EP deployment minus the
NVLink/HBM bandwidth difference of the dispatched rows (<= 30 MB per rank at
Mixtral EP=8, overlapped by the comm CTAs).
"""

from __future__ import annotations

import math
import statistics
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from .config import ModelConfig, ParallelSpec
from .routing import RoutingTable

NVLINK_GBS = 900.0  # NVLink 5, per direction per GPU


def rows_per_rank(routing: RoutingTable) -> np.ndarray:
    """(token, expert) rows hosted on each rank (TP ranks of a group host the
    same rows)."""
    par, model = routing.parallel, routing.model
    counts = np.asarray(routing.expert_counts, dtype=np.int64)
    e_per = model.E // par.ep
    per_group = counts.reshape(par.ep, e_per).sum(1)
    return np.repeat(per_group, par.tp)


def distinct_remote_pairs(routing: RoutingTable):
    """(D_out[r], D_in[r]): distinct (token, remote destination rank) pairs
    each rank sends / receives in the dispatch (every TP rank of a token's EP
    groups is a destination, routing.py:106-117)."""
    par, model = routing.parallel, routing.model
    W, M = par.world_size, routing.workload.M
    ex = routing.as_array().astype(np.int64)
    d_out = np.zeros(W, np.int64)
    d_in = np.zeros(W, np.int64)
    if M == 0:
        return d_out, d_in
    e_per = model.E // par.ep
    base = M // W
    t = np.arange(M)
    src = np.minimum(t // base, W - 1) if base > 0 else np.full(M, W - 1)
    groups = ex // e_per                                   # [M, topk]
    mask = np.zeros((M, par.ep), bool)
    mask[np.repeat(t, ex.shape[1]), groups.reshape(-1)] = True
    for g in range(par.ep):
        for s in range(par.tp):
            d = g * par.tp + s
            sel = mask[:, g] & (src != d)
            d_in[d] += int(sel.sum())
            np.add.at(d_out, src[sel], 1)
    return d_out, d_in


@dataclass
class Roofline:
    flops_max: float       # max_r FLOPs_r
    bytes_max: float       # max_r Bytes_r (per direction)
    t_flops_ms: float
    t_nvlink_ms: float
    ms: float
    bound: str
    peak_tflops: float


def roofline(routing: RoutingTable, peak_tflops: float, nvlink_gbs: float = NVLINK_GBS) -> Roofline:
    model, par = routing.model, routing.parallel
    rows = rows_per_rank(routing)
    flops = 4.0 * rows.astype(np.float64) * model.N * (model.K // par.tp)
    d_out, d_in = distinct_remote_pairs(routing)
    byts = 2.0 * model.N * (d_out + d_in).astype(np.float64)
    tf = float(flops.max()) / (peak_tflops * 1e12) * 1e3
    tn = float(byts.max()) / (nvlink_gbs * 1e9) * 1e3
    return Roofline(float(flops.max()), float(byts.max()), tf, tn, max(tf, tn),
                    "tensor" if tf >= tn else "nvlink", peak_tflops)


class EmulatedGroup:
    """Every rank of ``parallel`` on one GPU, random-init bf16 weights per rank
    (N(0,1)/sqrt(N), generated on the device), synthetic tokens."""

    def __init__(self, model: ModelConfig, parallel: ParallelSpec, routing: RoutingTable, knobs=None,
                 activation=None, seed: int = 0):
        from . import _lib
        from .executor import LayerKnobs, MoELayer, RankWeights, _ceil
        torch = _lib.require_device()
        self.torch, self.model, self.parallel, self.routing = torch, model, parallel, routing
        self.M = M = routing.workload.M
        W = parallel.world_size
        e_per, kl = model.E // parallel.ep, model.K // parallel.tp
        n_pad, k_pad = _ceil(model.N, 64), _ceil(kl, 64)
        g = torch.Generator(device="cuda").manual_seed(seed)
        s = 1.0 / math.sqrt(model.N)
        self.layers = []
        for r in range(W):
            w0t = torch.zeros(e_per, k_pad, n_pad, dtype=torch.bfloat16, device="cuda")
            w1t = torch.zeros(e_per, n_pad, k_pad, dtype=torch.bfloat16, device="cuda")
            for e in range(e_per):
                w0t[e, :kl, :model.N] = (torch.randn(kl, model.N, device="cuda", generator=g) * s).to(torch.bfloat16)
                w1t[e, :model.N, :kl] = (torch.randn(model.N, kl, device="cuda", generator=g) * s).to(torch.bfloat16)
            self.layers.append(MoELayer(model, parallel, r, max(1, M), RankWeights(w0t, w1t),
                                        activation=activation, knobs=knobs or LayerKnobs.for_world(W)))
        if W > 1:
            _lib.Context.link_local([l.ctx for l in self.layers])
        x = torch.randn(M, model.N, device="cuda", generator=g).to(torch.bfloat16)
        self.ex = torch.from_numpy(routing.as_array().copy()).cuda()
        self.ys = []
        for l in self.layers:
            lo, hi = l.token_range(M)
            l.place_tokens(x[lo:hi], M)
            self.ys.append(torch.empty(hi - lo, n_pad, dtype=torch.bfloat16, device="cuda"))

    def set_knobs(self, knobs) -> None:
        for l in self.layers:
            l.knobs = knobs

    def _forward_timed(self, record: bool):
        """One forward, phase-ordered over the emulated ranks (ranks share a
        device, so each in-kernel wait is on work enqueued before it)."""
        from .executor import index_flags
        torch = self.torch
        W = self.parallel.world_size
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if record else (lambda: None)
        fused = self.layers[0].knobs.is_fused(W)
        rec = {k: [] for k in (("index", "layers", "finish") if fused else ("index", "layer0", "layer1", "finish"))}

        def timed(key, fn):
            a, b = ev(), ev()
            if a is not None:
                a.record()
            fn()
            if b is not None:
                b.record()
            rec[key].append((a, b))

        for l in self.layers:
            timed("index", lambda l=l: l.ctx.index_build(self.ex, self.M, flags=index_flags(W, l.n_comm1())))
        if fused:
            for l, y in zip(self.layers, self.ys):
                k = l.knobs
                timed("layers", lambda l=l, y=y, k=k: l.ctx.layers(l.weights.w0t, l.weights.w1t, None, y, l.act,
                                                                   l.n_comm0(self.M), l.group0(self.M), k.wave1))
        else:
            for l in self.layers:
                k = l.knobs
                timed("layer0", lambda l=l, k=k: l.ctx.layer0(l.weights.w0t, l.act, l.n_comm0(self.M),
                                                              l.group0(self.M)))
            for l, y in zip(self.layers, self.ys):
                timed("layer1", lambda l=l, y=y: l.ctx.layer1(l.weights.w1t, None, y, l.n_comm1(), l.knobs.wave1))
        for l, y in zip(self.layers, self.ys):
            timed("finish", lambda l=l, y=y: l.ctx.combine_finish(y))
        return rec

    def measure(self, iters: int = 10, warmup: int = 3) -> Dict[str, object]:
        """Median over ``iters`` forwards of each rank's kernel times (ms);
        ``latency_ms`` = max over ranks of the per-rank sum."""
        torch = self.torch
        for _ in range(warmup):
            self._forward_timed(False)
        torch.cuda.synchronize()
        per_iter = []
        for _ in range(iters):
            # give the host a head start: every launch of the phase-ordered
            # forward is enqueued while the GPU spins, so no event interval
            # contains host (Python / ctypes) enqueue time
            torch.cuda._sleep(3_000_000)
            rec = self._forward_timed(True)
            torch.cuda.synchronize()
            per_iter.append({k: [a.elapsed_time(b) for a, b in v] for k, v in rec.items()})
        W = self.parallel.world_size
        med = {k: [statistics.median(it[k][r] for it in per_iter) for r in range(W)] for k in per_iter[0]}
        per_rank = [sum(med[k][r] for k in med) for r in range(W)]
        hot = int(np.argmax(per_rank))
        # the same forwards without events between the kernels (PDL chains
        # intact): whole phase-ordered forward / ranks -- a mean over ranks,
        # so it hides imbalance; the per-rank event sums above pay ~4 us of
        # broken launch overlap per kernel boundary (reported alongside)
        whole = []
        for _ in range(max(3, iters // 2)):
            torch.cuda._sleep(3_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            self._forward_timed(False)
            b.record()
            torch.cuda.synchronize()
            whole.append(a.elapsed_time(b))
        return {"latency_ms": max(per_rank), "hot_rank": hot, "per_rank_ms": per_rank,
                "kernels_ms_hot_rank": {k: med[k][hot] for k in med},
                "kernels_ms_max": {k: max(med[k]) for k in med},
                "chained_mean_ms": statistics.median(whole) / W}

    def close(self) -> None:
        for l in self.layers:
            l.close()
        self.layers = []


class EmulatedUnfused:
    """The unfused comparison path (``unfused.UnfusedLayer``: gather,
    all-to-all, cuBLAS grouped GEMMs, all-to-all back, top-k reduce) for
    every rank of an ``EmulatedGroup``, on the same GPU, weights and tokens,
    timed the way the fused group is: each rank's own phases with CUDA
    events, the all-to-all as the receiving rank's copies of its rows from
    the senders' buffers (HBM copies: the NVLink transfer of a real
    deployment is slower), host split-size synchronisation outside the
    timed intervals (a real ``all_to_all_single`` pays it).  Latency = max
    over ranks of the rank's summed phases.  ``forward`` returns the rank
    outputs (checked against the oracle by tests)."""

    def __init__(self, grp: "EmulatedGroup", activation: Optional[str] = None):
        from .unfused import UnfusedLayer
        torch = grp.torch
        self.torch, self.grp = torch, grp
        self.M = grp.M
        self.layers = []
        for r, l in enumerate(grp.layers):
            w0 = l.weights.w0t.transpose(1, 2).contiguous()  # [E_r, N, K/tp], row-major like the reference
            w1 = l.weights.w1t.transpose(1, 2).contiguous()  # [E_r, K/tp, N]
            self.layers.append(UnfusedLayer(grp.model, grp.parallel, r, w0, w1, activation=activation))
        self.xs = []
        for l in grp.layers:
            lo, hi = l.token_range(self.M)
            self.xs.append(l.ctx.token_buffer()[lo:hi])

    def forward(self, combine_w=None, record: bool = False):
        torch = self.torch
        W = self.grp.parallel.world_size
        M, topk = self.M, self.grp.ex.shape[1]
        times = [[] for _ in range(W)]

        def timed(r, fn):
            a = torch.cuda.Event(enable_timing=True) if record else None
            b = torch.cuda.Event(enable_timing=True) if record else None
            if a is not None:
                a.record()
            out = fn()
            if b is not None:
                b.record()
                times[r].append((a, b))
            return out

        # 1. per source rank: send order and the gathered rows
        plans = []
        for r, ul in enumerate(self.layers):
            lo, hi = self.grp.layers[r].token_range(M)
            ex_r = self.grp.ex[lo:hi]
            plans.append(timed(r, lambda ul=ul, ex_r=ex_r, r=r: (
                lambda p: (p, self.xs[r][p[1] // topk], p[3].int()))(ul._plan(ex_r))))
        counts = [p[0][2].tolist() for p in plans]  # split sizes on the host (untimed)
        offs = [np.concatenate([[0], np.cumsum(c)]) for c in counts]
        # 2. all-to-all: receiver d copies its rows from every sender
        recv = []
        for d in range(W):
            recv.append(timed(d, lambda d=d: (
                torch.cat([plans[r][1][offs[r][d]:offs[r][d + 1]] for r in range(W)]),
                torch.cat([plans[r][2][offs[r][d]:offs[r][d + 1]] for r in range(W)]))))
        # 3. expert GEMMs on every rank
        backs = [timed(d, lambda d=d: self.layers[d]._experts(*recv[d])) for d in range(W)]
        # 4. all-to-all back: source r copies its rows from every expert rank
        roff = [np.concatenate([[0], np.cumsum([counts[r][d] for r in range(W)])]) for d in range(W)]
        rets = [timed(r, lambda r=r: torch.cat([backs[d][roff[d][r]:roff[d][r + 1]] for d in range(W)]))
                for r in range(W)]
        # 5. top-k (weighted) reduce at the source
        outs = []
        for r in range(W):
            lo, hi = self.grp.layers[r].token_range(M)
            src_row = plans[r][0][1]

            def red(r=r, lo=lo, hi=hi, src_row=src_row):
                rows = torch.zeros((hi - lo) * topk, rets[r].shape[1], dtype=torch.float32, device=rets[r].device)
                rows.index_add_(0, src_row, rets[r].float())
                rows = rows.view(hi - lo, topk, -1)
                if combine_w is not None:
                    rows = rows * combine_w[lo:hi].float().unsqueeze(-1)
                return rows.sum(1).to(torch.bfloat16)
            outs.append(timed(r, red))
        return outs, times

    def measure(self, iters: int = 5, warmup: int = 2) -> Dict[str, object]:
        torch = self.torch
        for _ in range(warmup):
            self.forward()
        torch.cuda.synchronize()
        per_iter = []
        for _ in range(iters):
            _, times = self.forward(record=True)
            torch.cuda.synchronize()
            per_iter.append([sum(a.elapsed_time(b) for a, b in t) for t in times])
        per_rank = [statistics.median(it[r] for it in per_iter) for r in range(len(per_iter[0]))]
        return {"latency_ms": max(per_rank), "per_rank_ms": per_rank, "hot_rank": int(np.argmax(per_rank))}
