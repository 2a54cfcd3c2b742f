"""Unfused comparison paths: NCCL all-to-all + GroupGEMM (library calls).

These are the baselines the north star measures the fused kernels against
(BASELINE.md section 4), NOT the product:

* ``UnfusedLayer.forward(..., chunks=1)`` -- the unfused path: routing-driven
  permutation with torch ops, ``dist.all_to_all_single`` dispatch of every
  (token, expert) row to the ranks hosting the expert (every TP rank of the
  EP group, ref routing.py:106-117 ``transfer_counts``), cuBLAS grouped
  GEMMs (``torch._grouped_mm`` when available, else one cuBLAS GEMM per
  expert), activation, second grouped GEMM, ``all_to_all_single`` combine,
  and the top-k (weighted) reduce at the source (TP partials summed there,
  executor.py:221-246).
* ``chunks=k > 1`` -- the coarse-grained pipelined baseline (the analogue of
  the reference's ``simulate_coarse``, simulator.py:624-743; Tutel /
  FasterMoE style): the rank's tokens are cut into k chunks
  and chunk c's dispatch all-to-all (communication stream) overlaps chunk
  c-1's GEMMs (compute stream), whose combine all-to-all overlaps chunk c+1's
  GEMMs.  The per-chunk sizes are exchanged once up front.

Same inputs and outputs as ``MoELayer.forward``.  Works on CPU tensors with
the gloo backend (the multi-process tests) and on GPUs with NCCL.
"""

from __future__ import annotations

import contextlib
from typing import Optional

from .config import ModelConfig, ParallelSpec


class UnfusedLayer:
    """Per-rank unfused layer.  ``w0``: [E_r, N, K/tp], ``w1``: [E_r, K/tp, N]
    (this rank's experts and K shard, row-major like the reference)."""

    def __init__(self, model: ModelConfig, parallel: ParallelSpec, rank: int, w0, w1, device=None,
                 activation: Optional[str] = None):
        import torch
        self.torch = torch
        self.model, self.parallel, self.rank = model, parallel, rank
        self.e_per = model.E // parallel.ep
        self.e_lo = parallel.ep_group_of_rank(rank) * self.e_per
        self.w0 = w0.contiguous()
        self.w1 = w1.contiguous()
        self.activation = activation
        self.grouped = hasattr(torch, "_grouped_mm") and self.w0.is_cuda
        self._comm = None

    # -- local expert compute -------------------------------------------------
    def _gemm(self, x, w, offs):
        torch = self.torch
        if self.grouped and x.shape[0] > 0:
            try:
                return torch._grouped_mm(x, w, offs=offs)
            except Exception:  # noqa: BLE001 -- older builds: per-expert GEMMs
                self.grouped = False
        outs, start = [], 0
        for e, stop in enumerate(offs.tolist()):
            outs.append(x[start:stop] @ w[e])
            start = stop
        return torch.cat(outs) if outs else x.new_zeros((0, w.shape[-1]))

    def _experts(self, rows, eids):
        """Grouped GEMM pair over this rank's experts for rows with global
        expert ids ``eids``; returns bf16 rows in the input order."""
        torch = self.torch
        le = eids.long() - self.e_lo
        perm = torch.argsort(le, stable=True)
        xs = rows[perm]
        offs = torch.cumsum(torch.bincount(le, minlength=self.e_per), 0).int()
        h = self._gemm(xs, self.w0, offs)
        if self.activation == "silu":
            h = torch.nn.functional.silu(h.float())
        elif self.activation == "tanh":
            h = torch.tanh(h.float())
        elif self.activation == "relu":
            h = torch.relu(h)
        y = self._gemm(h.to(torch.bfloat16), self.w1, offs).to(torch.bfloat16)
        back = torch.empty_like(y)
        back[perm] = y
        return back

    # -- routing of one token range ---------------------------------------------
    def _plan(self, experts_rows):
        """Send order for tokens ``experts_rows`` [m, topk]: every (token,
        slot) row goes to each TP rank of its expert's EP group.  Returns
        (order of the replicated rows by destination, source (token, slot)
        row of each, destination counts, expert id of each)."""
        torch = self.torch
        tp, W = self.parallel.tp, self.parallel.world_size
        m, topk = experts_rows.shape
        flat_e = experts_rows.reshape(-1).long()
        rep_e = flat_e.repeat_interleave(tp)                     # [m*topk*tp]
        shard = torch.arange(tp, device=flat_e.device).repeat(m * topk)
        dest = (rep_e // self.e_per) * tp + shard
        order = torch.argsort(dest * self.model.E + rep_e, stable=True)
        counts = torch.bincount(dest, minlength=W)
        return order, order // tp, counts, rep_e[order]

    @contextlib.contextmanager
    def _on(self, stream):
        if stream is None:
            yield
        else:
            with self.torch.cuda.stream(stream):
                yield

    def forward(self, x_local, experts, combine_w=None, M: Optional[int] = None, chunks: int = 1):
        import torch.distributed as dist
        torch = self.torch
        W = self.parallel.world_size
        tp = self.parallel.tp
        M = experts.shape[0] if M is None else M
        base = M // W
        lo = self.rank * base
        hi = M if self.rank == W - 1 else lo + base
        m_r = hi - lo
        topk = experts.shape[1]
        N = x_local.shape[1]
        dist_on = W > 1
        C = max(1, min(int(chunks), max(m_r, 1)))
        bounds = [m_r * c // C for c in range(C + 1)]
        plans = [self._plan(experts[lo + bounds[c]:lo + bounds[c + 1]]) for c in range(C)]
        # every chunk's send counts exchanged once: [W dest, C] -> [W src, C]
        send_cnt = torch.stack([p[2] for p in plans], 1).contiguous() if C else None
        if dist_on:
            recv_cnt = torch.empty_like(send_cnt)
            dist.all_to_all_single(recv_cnt, send_cnt)
            sc_all, rc_all = send_cnt.t().tolist(), recv_cnt.t().tolist()
        else:
            sc_all = rc_all = send_cnt.t().tolist()
        cuda = x_local.is_cuda
        comp = torch.cuda.current_stream(x_local.device) if cuda else None
        comm = None
        if cuda and dist_on and C > 1:
            if self._comm is None:
                self._comm = torch.cuda.Stream(x_local.device)
            comm = self._comm
        out = torch.zeros(m_r, N, dtype=torch.float32, device=x_local.device)

        def record(stream):
            if stream is None:
                return None
            ev = torch.cuda.Event()
            ev.record(stream)
            return ev

        def dispatch(c):
            """Gather chunk c's rows (compute stream), all-to-all them and
            their expert ids (communication stream)."""
            _, src_row, _, eids = plans[c]
            sc, rc = sc_all[c], rc_all[c]
            send_rows = x_local[bounds[c] + src_row // topk].to(torch.bfloat16)
            if not dist_on:
                return send_rows, eids, None
            if comm is not None:
                comm.wait_stream(comp)
            with self._on(comm):
                recv_rows = send_rows.new_empty((sum(rc), N))
                dist.all_to_all_single(recv_rows, send_rows, rc, sc)
                send_e = eids.int()
                recv_e = send_e.new_empty(sum(rc))
                dist.all_to_all_single(recv_e, send_e, rc, sc)
            if comm is not None:  # allocated on the comm stream, read on the compute stream
                recv_rows.record_stream(comp)
                recv_e.record_stream(comp)
            return recv_rows, recv_e, record(comm)

        def send_back(c, back, ready):
            """Return chunk c's expert rows to their source ranks."""
            sc, rc = sc_all[c], rc_all[c]
            if not dist_on:
                return back, None
            if comm is not None:
                comm.wait_event(ready)
            with self._on(comm):
                ret = back.new_empty((sum(sc), N))
                dist.all_to_all_single(ret, back, sc, rc)
            if comm is not None:
                back.record_stream(comm)
                ret.record_stream(comp)
            return ret, record(comm)

        def reduce(c, ret, ready):
            """Top-k (weighted) reduce of chunk c at the source; TP partials
            of one (token, slot) are summed first."""
            _, src_row, _, _ = plans[c]
            if ready is not None:
                comp.wait_event(ready)
            n_c = bounds[c + 1] - bounds[c]
            rows = torch.zeros(n_c * topk, N, dtype=torch.float32, device=ret.device)
            rows.index_add_(0, src_row, ret.float())
            rows = rows.view(n_c, topk, N)
            if combine_w is not None:
                rows = rows * combine_w[lo + bounds[c]:lo + bounds[c + 1]].float().unsqueeze(-1)
            out[bounds[c]:bounds[c + 1]] = rows.sum(1)

        # software pipeline (depth 1): dispatch(c+1) is issued before the
        # GEMMs of chunk c, whose return all-to-all runs under the GEMMs of
        # chunk c+1; the reduce of chunk c-1 follows the GEMMs of chunk c
        nxt = dispatch(0) if C else None
        back_of = [None] * C
        for c in range(C):
            recv_rows, recv_e, ev = nxt
            if c + 1 < C:
                nxt = dispatch(c + 1)
            if ev is not None:
                comp.wait_event(ev)
            back = self._experts(recv_rows, recv_e)
            back_of[c] = send_back(c, back, record(comp))
            if c > 0:
                reduce(c - 1, *back_of[c - 1])
                back_of[c - 1] = None
        if C:
            reduce(C - 1, *back_of[C - 1])
        return out.to(torch.bfloat16)
