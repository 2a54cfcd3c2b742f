"""B200 cost model fitted to measured per-CTA timelines.

The reference's ``CostModel`` (simulator.py:66-139) is a parametric timing of
tiles and messages per thread block, driving a discrete-event simulation of
the fused kernel (``simulate_fine``, simulator.py:447-575) whose n_c curve
feeds the split chooser.  Here the same parameters are FITTED to what the
B200 kernels actually did (``comet_timeline_*`` records: the MMA interval of
every work unit, the interval of every dispatch item), and the simulation
replays the real kernel's scheduling -- one persistent launch, dynamic unit
claims in sequence order over 2-CTA pairs, layer0 units gated on their
tiles' dispatch, layer1 units gated on their H tiles, dispatch CTAs that
join the GEMMs when done -- so ``predict_split`` can answer shapes that were
never profiled instead of ``select_split`` raising ``UnprofiledConfigError``
(assigner.py:260-292).

Units of the model: ``compute_flops_per_s`` is per 2-CTA PAIR (the unit of
work here), ``intra_node_bytes_per_s`` per dispatch CTA (NVLink pulls),
``alpha_tile_s`` the fixed cost of a work unit (pipeline fill + epilogue
tail), ``alpha_msg_s`` the fixed cost of a 32-row dispatch item, and
``fixed_s`` the per-forward cost outside the layer kernel (index build,
local dispatch, combine, launches).  ``epilogue_s`` / ``fold_row_s``: a
unit's accumulator drain (the next unit's MMAs wait for it: both 256-column
TMEM halves are in use) and, in the fused combine at world > 1, the extra
time per earlier hosted row a token's last row folds in (top-8 shapes: the
folder units read up to 7 rows and end layer1).  Host-only (numpy): the
routing gives the pair structure and fold counts without the GPU index
build.
"""

from __future__ import annotations

import heapq
import json
import math
import os
from dataclasses import asdict, dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from .assigner import SplitKey, SplitRecord, candidate_ncs, record_from_curve
from .config import ConfigurationError, ModelConfig, ParallelSpec, WorkloadSpec
from .routing import RoutingTable, build_routing

PAIR_ROWS = 256
BLOCK_N = 512
HALF_N = 256
HALF_COST = 1.35  # a 256-column half unit's time per FLOP vs a full unit (64 vs 48 B/cycle/SM of operands)
ITEM_ROWS = 32
PRESET_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "costmodel_b200.json")


@dataclass(frozen=True)
class CostModel:
    """Reference field names (simulator.py:66-96) + ``fixed_s``; see module doc."""

    compute_flops_per_s: float
    alpha_tile_s: float
    alpha_msg_s: float
    local_bytes_per_s: float
    intra_node_bytes_per_s: float
    chunk_overhead_s: float = 0.0
    blocks: int = 148
    fixed_s: float = 0.0
    epilogue_s: float = 0.0
    fold_row_s: float = 0.0

    def __post_init__(self) -> None:
        if self.compute_flops_per_s <= 0 or self.intra_node_bytes_per_s <= 0 or self.local_bytes_per_s <= 0:
            raise ConfigurationError("rates must be > 0")
        if min(self.alpha_tile_s, self.alpha_msg_s, self.chunk_overhead_s, self.fixed_s, self.epilogue_s,
               self.fold_row_s) < 0:
            raise ConfigurationError("fixed overheads must be >= 0")
        if self.blocks < 4:
            raise ConfigurationError("need at least two 2-CTA pairs")

    def unit_s(self, flops: float) -> float:
        return self.alpha_tile_s + flops / self.compute_flops_per_s

    def item_s(self, nbytes: float) -> float:
        return self.alpha_msg_s + nbytes / self.intra_node_bytes_per_s

    def to_json_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_json_dict(cls, data: dict) -> "CostModel":
        return cls(**{k: (int(v) if k == "blocks" else float(v)) for k, v in data.items()})


def preset() -> CostModel:
    """The committed fit (costmodel_b200.json, written by ``fit`` on a B200)."""
    with open(PRESET_PATH) as fh:
        return CostModel.from_json_dict(json.load(fh)["model"])


# ---------------------------------------------------------------------------
# Pair structure of one rank (host, from the routing counts)
# ---------------------------------------------------------------------------

@dataclass
class RankShape:
    pairs: List[Tuple[int, int, int]]   # (expert_local, valid_rows, remote_rows) per pair, claim order
    k_local: int
    n_embed: int
    folds: List[float] = None           # per pair: max over its two 128-row tiles of the mean rows folded per row


def rank_shape(routing: RoutingTable, rank: int) -> RankShape:
    """Pairs of 256 rows per hosted expert (local rows first, resolver.py:
    171-195), in the layer0 claim order (fewer remote rows first,
    resolver.py:206-252), with each pair's fused-combine fold load: a token's
    row in its LAST hosted expert folds its rows in the other hosted experts
    (moe_layers.cu epilogue)."""
    model, par = routing.model, routing.parallel
    M, W = routing.workload.M, par.world_size
    ex = routing.as_array().astype(np.int64)
    e_per = model.E // par.ep
    e_lo = (rank // par.tp) * e_per
    base = M // W
    lo = rank * base if base else 0
    hi = (M if rank == W - 1 else lo + base) if base else (M if rank == W - 1 else 0)
    hosted = (ex >= e_lo) & (ex < e_lo + e_per)
    n_host = hosted.sum(axis=1)
    last_host = np.where(n_host > 0, np.max(np.where(hosted, ex - e_lo, -1), axis=1), -1)
    tok = np.arange(M)
    src = np.minimum(tok // base, W - 1) if base else np.full(M, W - 1)
    pairs, keys, folds = [], [], []
    for j in range(e_per):
        hit = (ex == e_lo + j).any(axis=1)
        t_j = tok[hit]
        order = np.lexsort((t_j, (src[hit] - rank) % W))  # rows: ((src - rank) mod W, token)
        t_j = t_j[order]
        fold_row = np.where(last_host[t_j] == j, n_host[t_j] - 1, 0).astype(float)
        cnt = int(hit.sum())
        loc = int(hit[lo:hi].sum())
        for k in range(0, cnt, PAIR_ROWS):
            rows = min(PAIR_ROWS, cnt - k)
            loc_in = max(0, min(rows, loc - k))
            pairs.append((j, rows, rows - loc_in))
            # claim key = reference key of the pair's last 128-row tile:
            # (remote rows, expert, row start)  (index_build.cu pair_of)
            h0 = 128 if rows > 128 else 0
            half = rows - h0
            keys.append((half - max(0, min(half, loc_in - h0)), j, k + h0))
            f = fold_row[k:k + rows]
            folds.append(max(float(f[:128].mean()), float(f[128:].mean()) if rows > 128 else 0.0))
    order = sorted(range(len(pairs)), key=lambda i: keys[i])
    return RankShape([pairs[i] for i in order], model.K // par.tp, model.N, [folds[i] for i in order])


# ---------------------------------------------------------------------------
# Simulation of one launch (the kernel's scheduling, moe_layers.cu)
# ---------------------------------------------------------------------------

def _halves(seq, n_split):
    """The last ``n_split`` units of a layer's sequence as two 256-column
    halves each, after the full units (sched.cuh make_sched / unit_at)."""
    full = len(seq) - max(0, min(len(seq), n_split))
    out = seq[:full]
    for layer, p, cols, _, _ in seq[full:]:
        out += [(layer, p, min(cols, HALF_N), 1, 0), (layer, p, max(0, cols - HALF_N), 1, 0)]
    return out


def _ksplit(tiles: int, k_blocks: int, n_pairs: int) -> int:
    """K slices per output tile (sched.cuh ksplit_for, COMET_KSPLIT=8)."""
    return max(1, min(8, k_blocks // 4, n_pairs // tiles)) if tiles else 1


def _sliced(seq, S):
    """Every unit as S consecutive K-slice claims (no halves then)."""
    return [(layer, p, cols, S, ks) for layer, p, cols, _, _ in seq for ks in range(S)]


def _units(shape: RankShape, group: int, wave: int, split1: int = 0, n_pairs: int = 74):
    """(layer, pair, columns, K slices) in claim-sequence order: layer0 pair
    groups x n-blocks (raster 0; a mostly idle last round as halves), then
    layer1 pair groups x waves x n-blocks (raster 2; the last ``split1`` units
    as halves); split-K when a layer has fewer tiles than pairs -- sched.cuh
    make_sched / layer0_split / ksplit_for / unit_at."""
    P = len(shape.pairs)
    seq = []
    nb0 = -(-shape.k_local // BLOCK_N)
    nb1 = -(-shape.n_embed // BLOCK_N)
    for g0 in range(0, P, group):
        ge = min(group, P - g0)
        for nb in range(nb0):
            for p in range(g0, g0 + ge):
                seq.append((0, p, min(BLOCK_N, shape.k_local - nb * BLOCK_N), 1, 0))
    S0 = _ksplit(len(seq), shape.n_embed // 64, n_pairs)
    if S0 > 1:
        seq = _sliced(seq, S0)
    else:
        rem = len(seq) % n_pairs
        seq = _halves(seq, rem if 0 < rem and 2 * rem <= n_pairs else 0)
    seq1 = []
    for g0 in range(0, P, group):
        ge = min(group, P - g0)
        for w0 in range(0, nb1, wave):
            for nb in range(w0, min(nb1, w0 + wave)):
                for p in range(g0, g0 + ge):
                    seq1.append((1, p, min(BLOCK_N, shape.n_embed - nb * BLOCK_N), 1, 0))
    S1 = _ksplit(len(seq1), shape.k_local // 64, n_pairs)
    if split1 < 0:  # automatic (sched.cuh seq_total): a 1-4 round layer1 ends its last 16 units in halves
        split1 = 16 if n_pairs < len(seq1) < 4 * n_pairs else 0
    seq1 = _sliced(seq1, S1) if S1 > 1 else _halves(seq1, split1)
    return seq + seq1, nb0


def default_split1(routing: RoutingTable, blocks: int) -> int:
    """The kernel's default layer1 tail halves (capi.cu layer1_args): 3/4 of
    the pairs when fold chains are long (world > 1, top-k >= 4, >= 4 hosted
    experts), else automatic (-1: 16 units when layer1 is 1-4 rounds)."""
    par, model = routing.parallel, routing.model
    long_folds = par.world_size > 1 and model.topk >= 4 and model.E // par.ep >= 4
    return 3 * (blocks // 2) // 4 if long_folds else -1  # -1: by the round count (_units)


def simulate(routing: RoutingTable, rank: int, cm: CostModel, n_c: int, group: int = 4, wave: int = 4) -> float:
    """Predicted forward latency (seconds) of ``rank`` with ``n_c`` dispatch CTAs."""
    shape = rank_shape(routing, rank)
    P = len(shape.pairs)
    row_bytes = 2 * shape.n_embed
    n_pairs = cm.blocks // 2
    fused = routing.parallel.world_size > 1  # the combine folds in layer1's epilogue
    n_c = max(0, min(n_c, cm.blocks - 2)) if routing.parallel.world_size > 1 else 0
    # dispatch: 32-row items of each pair's remote rows, round-robin over n_c CTAs
    tile_ready = [0.0] * P
    cta_t = [0.0] * max(1, n_c)
    if n_c:
        item = 0
        for p, (_, _, remote) in enumerate(shape.pairs):
            for r0 in range(0, remote, ITEM_ROWS):
                c = item % n_c
                cta_t[c] += cm.item_s(min(ITEM_ROWS, remote - r0) * row_bytes)
                tile_ready[p] = max(tile_ready[p], cta_t[c])
                item += 1
    # pairs free at: compute pairs 0, dispatch pairs when both CTAs are done
    free = [0.0] * (n_pairs - n_c // 2) + [max(cta_t[2 * i], cta_t[2 * i + 1]) for i in range(n_c // 2)]
    heapq.heapify(free)
    seq, nb0 = _units(shape, group, wave, default_split1(routing, cm.blocks), n_pairs)
    h_done = [0.0] * P
    end = 0.0
    for layer, p, cols, S, ks in seq:
        if cols <= 0:  # half 1 of a narrow last block: no columns
            continue
        t = heapq.heappop(free)
        rows = PAIR_ROWS
        k = shape.n_embed if layer == 0 else shape.k_local
        eff_cols = HALF_N if cols <= HALF_N else BLOCK_N
        cost_cols = HALF_N * HALF_COST if cols <= HALF_N else BLOCK_N
        dur = cm.unit_s(2.0 * rows * cost_cols * k / S) + cm.epilogue_s * eff_cols / BLOCK_N
        if S > 1:  # fp32 partial store (2x the bytes); the last slice reduces all S
            dur += cm.epilogue_s * (1 + (S if ks == S - 1 else 0))
        if layer == 1 and fused:
            dur += shape.folds[p] * cm.fold_row_s * eff_cols / BLOCK_N
        start = max(t, tile_ready[p] if layer == 0 else h_done[p])
        stop = start + dur
        if layer == 0:
            h_done[p] = max(h_done[p], stop)
        heapq.heappush(free, stop)
        end = max(end, stop)
    return end + cm.fixed_s


def predict_split(model: ModelConfig, parallel: ParallelSpec, workload: WorkloadSpec,
                  cm: Optional[CostModel] = None, rank: Optional[int] = None, stride: int = 8,
                  max_nc: int = 96) -> SplitRecord:
    """The n_c curve predicted by the fitted model (max over ranks unless
    ``rank``), as a SplitRecord with cost "b200-model" (assigner.py schema)."""
    cm = cm or preset()
    routing = build_routing(model, parallel, workload)
    ranks = [rank] if rank is not None else list(range(parallel.world_size))
    pts = []
    for nc in candidate_ncs(cm.blocks, stride, max_nc):
        ns = max(simulate(routing, r, cm, nc) for r in ranks)
        pts.append((nc, int(round(ns * 1e9))))
    key = SplitKey.for_config(model, parallel, workload.M, "b200-model", cm.blocks)
    return record_from_curve(key, pts)


# ---------------------------------------------------------------------------
# Fit from measured timelines
# ---------------------------------------------------------------------------

def fit(samples: Sequence[dict], blocks: int = 148) -> CostModel:
    """``samples``: dicts with ``unit_flops`` / ``unit_s`` (per measured MMA
    interval), ``cta_rates`` (dispatch bytes/s of each dispatch CTA) and
    ``fixed_s`` (forward latency minus the layer kernel's span).  Least
    squares for (alpha, 1/rate) of units; medians for the rest."""
    uf = np.concatenate([np.asarray(s["unit_flops"], float) for s in samples])
    us = np.concatenate([np.asarray(s["unit_s"], float) for s in samples])
    A = np.stack([np.ones_like(uf), uf], 1)
    (a_t, inv_r), *_ = np.linalg.lstsq(A, us, rcond=None)
    # dispatch: a CTA's items overlap in its copy pipeline, so the rate is the
    # CTA's bytes over its busy span (median over CTAs); no per-item constant
    rates = np.concatenate([np.asarray(s.get("cta_rates", []), float) for s in samples])
    a_m, inv_b = 0.0, 1.0 / (float(np.median(rates)) if len(rates) else 20e9)
    fixed = float(np.median([s["fixed_s"] for s in samples]))
    # epilogue: median drain of units without folds; fold cost per folded
    # row: least squares through the origin of the excess over that median
    # (epi_folds and epi_scale: a half unit drains half the columns)
    epi = np.concatenate([np.asarray(s.get("epi_s", []), float) for s in samples])
    efold = np.concatenate([np.asarray(s.get("epi_folds", []), float) for s in samples])
    escale = np.concatenate([np.asarray(s.get("epi_scale", np.ones(len(s.get("epi_s", [])))), float)
                             for s in samples])
    base = (efold == 0) & (escale == 1)
    epi_s = float(np.median(epi[base])) if np.any(base) else 0.0
    m = efold > 0
    fold_s = (float(np.sum(efold[m] * (epi[m] - epi_s * escale[m])) / np.sum(efold[m] ** 2))
              if np.any(m) else 0.0)
    return CostModel(compute_flops_per_s=float(1.0 / max(inv_r, 1e-18)), alpha_tile_s=max(0.0, float(a_t)),
                     alpha_msg_s=max(0.0, float(a_m)), local_bytes_per_s=float(1.0 / max(inv_b, 1e-15) * 4),
                     intra_node_bytes_per_s=float(1.0 / max(inv_b, 1e-15)), blocks=blocks, fixed_s=max(0.0, fixed),
                     epilogue_s=max(0.0, epi_s), fold_row_s=max(0.0, fold_s))


def sample_from_timeline(records: Iterable[Tuple[int, str, int, int, int]], routing: RoutingTable, rank: int,
                         latency_s: float, group: int = 4, wave: int = 4, split1: Optional[int] = None,
                         blocks: int = 148) -> dict:
    """Turn one launch's timeline (``Context.timeline_dump``) into a fit
    sample: every full MMA interval with its unit's FLOPs, every dispatch
    item with its bytes (32 rows; a tile's last item may be shorter)."""
    shape = rank_shape(routing, rank)
    seq, _ = _units(shape, group, wave, default_split1(routing, blocks) if split1 is None else split1, blocks // 2)
    recs = list(records)
    mma = [(t, s, e) for c, r, t, s, e in recs if r == "mma"]
    load = {(c, t): s for c, r, t, s, e in recs if r == "load"}
    uf, us = [], []
    for c, r, t, s, e in recs:
        if r != "mma" or t >= len(seq):
            continue
        layer, p, cols, S, _ = seq[t]
        if cols <= 0:
            continue
        k = shape.n_embed if layer == 0 else shape.k_local
        eff = HALF_N * HALF_COST if cols <= HALF_N else BLOCK_N
        s0 = max(s, load.get((c, t), s))  # dependency waits excluded
        uf.append(2.0 * PAIR_ROWS * eff * k / S)
        us.append((e - s0) * 1e-9)
    row_bytes = 2 * shape.n_embed
    per_cta: Dict[int, List[Tuple[int, int]]] = {}
    for c, r, t, s, e in recs:
        if r == "comm":
            per_cta.setdefault(c, []).append((s, e))
    rates = []
    for ivs in per_cta.values():  # items of 32 rows (a tile's last one may be shorter: upper bound)
        span = (max(e for _, e in ivs) - min(s for s, _ in ivs)) * 1e-9
        if span > 0:
            rates.append(len(ivs) * ITEM_ROWS * row_bytes / span)
    # epilogue drains (leader CTAs' records) with the unit's fold load
    fused = routing.parallel.world_size > 1
    epi_s, epi_folds, epi_scale = [], [], []
    for c, r, t, s, e in recs:
        if r != "epilogue" or t >= len(seq) or c % 2:
            continue
        layer, p, cols, S, _ = seq[t]
        if cols <= 0 or S > 1:
            continue
        scale = (HALF_N if cols <= HALF_N else BLOCK_N) / BLOCK_N
        epi_s.append((e - s) * 1e-9)
        epi_scale.append(scale)
        epi_folds.append(scale * shape.folds[p] if (layer == 1 and fused) else 0.0)
    span = (max(e for *_, e in recs) - min(s for _, _, _, s, _ in recs)) * 1e-9 if recs else 0.0
    return {"unit_flops": uf, "unit_s": us, "cta_rates": rates, "fixed_s": max(0.0, latency_s - span),
            "epi_s": epi_s, "epi_folds": epi_folds, "epi_scale": epi_scale}
