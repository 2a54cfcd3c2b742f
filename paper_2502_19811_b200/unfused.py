"""Unfused comparison path: NCCL all-to-all + GroupGEMM (library calls).

This is the baseline the north star measures the fused kernels against
(BASELINE.md section 4), NOT the product: routing-driven permutation with
torch ops, ``dist.all_to_all_single`` dispatch, cuBLAS grouped GEMMs
(``torch._grouped_mm`` when available, else one cuBLAS GEMM per expert),
activation, second grouped GEMM, ``all_to_all_single`` combine and an
index-add top-k reduce.  Same inputs and outputs as ``MoELayer.forward``.
"""

from __future__ import annotations

from typing import Optional

from .config import ModelConfig, ParallelSpec


class UnfusedLayer:
    """Per-rank unfused layer (tp must be 1)."""

    def __init__(self, model: ModelConfig, parallel: ParallelSpec, rank: int, w0, w1, device=None):
        import torch
        if parallel.tp != 1:
            raise ValueError("the unfused baseline covers tp == 1")
        self.torch = torch
        self.model, self.parallel, self.rank = model, parallel, rank
        self.e_per = model.E // parallel.ep
        self.e_lo = rank * self.e_per
        # w0: [E_r, N, K], w1: [E_r, K, N] bf16 (row-major like the reference)
        self.w0 = w0.contiguous()
        self.w1 = w1.contiguous()
        self.grouped = hasattr(torch, "_grouped_mm")

    def _gemm(self, x, w, offs):
        torch = self.torch
        if self.grouped and x.shape[0] > 0:
            try:
                return torch._grouped_mm(x, w, offs=offs)
            except Exception:
                self.grouped = False
        outs, start = [], 0
        for e, stop in enumerate(offs.tolist()):
            outs.append(x[start:stop] @ w[e])
            start = stop
        return torch.cat(outs) if outs else x.new_zeros((0, w.shape[-1]))

    def forward(self, x_local, experts, combine_w=None, M: Optional[int] = None):
        import torch.distributed as dist
        torch = self.torch
        world = self.parallel.world_size
        M = experts.shape[0] if M is None else M
        base = M // world
        lo = self.rank * base
        hi = M if self.rank == world - 1 else lo + base
        ex_local = experts[lo:hi].long()                      # [M_r, topk]
        topk = ex_local.shape[1]
        flat_e = ex_local.reshape(-1)
        dest = flat_e // self.e_per                           # destination rank of each (token, slot)
        order = torch.argsort(dest * self.model.E + flat_e, stable=True)
        send_rows = x_local[order // topk]                    # permuted token rows
        send_counts = torch.bincount(dest, minlength=world)
        if world > 1:
            recv_counts = torch.empty_like(send_counts)
            dist.all_to_all_single(recv_counts, send_counts)
            sc, rc = send_counts.tolist(), recv_counts.tolist()
            recv_rows = send_rows.new_empty((sum(rc), send_rows.shape[1]))
            dist.all_to_all_single(recv_rows, send_rows, rc, sc)
            send_e = flat_e[order].int()
            recv_e = send_e.new_empty(sum(rc))
            dist.all_to_all_single(recv_e, send_e, rc, sc)
        else:
            rc, sc = [send_rows.shape[0]], [send_rows.shape[0]]
            recv_rows, recv_e = send_rows, flat_e[order]
        # local grouped GEMMs over this rank's experts
        le = recv_e.long() - self.e_lo
        perm = torch.argsort(le, stable=True)
        xs = recv_rows[perm]
        offs = torch.cumsum(torch.bincount(le, minlength=self.e_per), 0).int()
        h = self._gemm(xs, self.w0, offs)
        y = self._gemm(h.to(torch.bfloat16), self.w1, offs).to(torch.bfloat16)
        back = torch.empty_like(y)
        back[perm] = y
        if world > 1:
            ret = back.new_empty((sum(sc), back.shape[1]))
            dist.all_to_all_single(ret, back, sc, rc)
        else:
            ret = back
        rows = torch.empty_like(ret)
        rows[order] = ret                                     # back to (token, slot) order
        rows = rows.view(hi - lo, topk, -1).float()
        if combine_w is not None:
            rows = rows * combine_w[lo:hi].unsqueeze(-1)
        return rows.sum(1).to(torch.bfloat16)
