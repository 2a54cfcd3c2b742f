"""Shared-tensor decomposition and tile rescheduling, built on the GPU.

Mirror of `pkg/src/moepipe/resolver.py`: the same dataclasses
(``SharedTensorMeta``, ``Tile``, ``ReduceChunk``, ``TileSchedule``,
``Violation``), JSON form and error behaviour.  The integer work -- the
per-expert sorted layout (resolver.py:171-195), the locality-first layer0
order (206-252) and the column-wave layer1 order with its reduce chunks
(255-309) -- is produced by the CUDA index builder (``moe_index_build`` in
``csrc/index_build.cu``, bit-exact with the reference) and only wrapped into
Python objects here.  ``validate_schedule`` compares a schedule against a
GPU-built cover with the reference's violation codes (342-441).

No GPU -> these functions raise ``NativeUnavailable``; there is no host
fallback.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from .config import ConfigurationError, ModelConfig, WorkloadSpec, canonical_json
from .routing import RoutingTable

M_DIM = "M"
N_DIM = "N"

DEFAULT_TILE_ROWS = 128


def default_tile_cols(n_embed: int) -> int:
    """>= four column waves when possible (ref resolver.py:35-39)."""
    return 128 if n_embed >= 512 else max(1, n_embed // 4)


@dataclass(frozen=True)
class SharedTensorMeta:
    """The (M*topk, N) buffer between a pipeline's two operators and how it is
    tiled (ref resolver.py:42-70)."""

    global_rows: int
    cols: int
    decomposed_dim: str
    tile_rows: int = DEFAULT_TILE_ROWS
    tile_cols: int = 0

    def __post_init__(self) -> None:
        if self.decomposed_dim not in (M_DIM, N_DIM):
            raise ConfigurationError(
                f"decomposed_dim must be {M_DIM!r} or {N_DIM!r}, got {self.decomposed_dim!r}")
        if self.global_rows < 0 or self.cols < 1:
            raise ConfigurationError("invalid shared tensor shape")
        if self.tile_rows < 1:
            raise ConfigurationError(f"tile_rows must be >= 1, got {self.tile_rows}")
        if self.decomposed_dim == N_DIM and not 1 <= self.tile_cols <= self.cols:
            raise ConfigurationError(f"tile_cols must be in [1, {self.cols}], got {self.tile_cols}")

    def col_blocks(self) -> int:
        return -(-self.cols // self.tile_cols) if self.decomposed_dim == N_DIM else 1


def meta_for_layer0(model: ModelConfig, workload: WorkloadSpec,
                    tile_rows: int = DEFAULT_TILE_ROWS) -> SharedTensorMeta:
    return SharedTensorMeta(global_rows=workload.M * model.topk, cols=model.N,
                            decomposed_dim=M_DIM, tile_rows=tile_rows)


def meta_for_layer1(model: ModelConfig, workload: WorkloadSpec,
                    tile_rows: int = DEFAULT_TILE_ROWS,
                    tile_cols: Optional[int] = None) -> SharedTensorMeta:
    return SharedTensorMeta(global_rows=workload.M * model.topk, cols=model.N,
                            decomposed_dim=N_DIM, tile_rows=tile_rows,
                            tile_cols=default_tile_cols(model.N) if tile_cols is None else tile_cols)


@dataclass(frozen=True)
class Tile:
    """GEMM work over a contiguous row slice of one expert's block
    (ref resolver.py:99-117)."""

    tile_id: int
    layer: int
    expert: int
    row_start: int
    row_stop: int
    rows: Tuple[Tuple[int, int], ...]
    deps: frozenset
    col_start: int = 0
    col_stop: int = 0


@dataclass(frozen=True)
class ReduceChunk:
    """Column block of the combine and the tiles it waits for
    (ref resolver.py:120-127)."""

    chunk_id: int
    col_start: int
    col_stop: int
    prereq_tile_ids: frozenset


@dataclass(frozen=True)
class TileSchedule:
    """Ordered tiles (and layer1 reduce chunks) of one rank
    (ref resolver.py:130-168)."""

    rank: int
    layer: int
    meta: SharedTensorMeta
    tiles: Tuple[Tile, ...]
    reduce_chunks: Tuple[ReduceChunk, ...] = ()
    layout: Dict[int, Tuple[Tuple[int, int], ...]] = field(default_factory=dict)

    def to_json_dict(self) -> dict:
        return {
            "rank": self.rank,
            "layer": self.layer,
            "tile_rows": self.meta.tile_rows,
            "tile_cols": self.meta.tile_cols,
            "tiles": [{
                "tile_id": t.tile_id,
                "expert": t.expert,
                "rows": [t.row_start, t.row_stop],
                "cols": [t.col_start, t.col_stop] if self.layer == 1 else None,
                "deps": sorted(list(d) for d in t.deps),
            } for t in self.tiles],
            "reduce_chunks": [{
                "chunk_id": c.chunk_id,
                "cols": [c.col_start, c.col_stop],
                "prereq_tile_ids": sorted(c.prereq_tile_ids),
            } for c in self.reduce_chunks],
        }

    def to_json_str(self) -> str:
        return canonical_json(self.to_json_dict())


@dataclass(frozen=True)
class Violation:
    """One schedule defect (ref resolver.py:312-318)."""

    code: str
    subject: Optional[int]
    message: str


# ---------------------------------------------------------------------------
# Device index access (one cached index-only context per shape and rank).
# ---------------------------------------------------------------------------

_CTX_LOCK = threading.Lock()
_CTX_CACHE: Dict[tuple, object] = {}


def _index_context(routing: RoutingTable, rank: int):
    from . import _lib
    _lib.require_device()
    model, par = routing.model, routing.parallel
    m_cap = max(1, routing.workload.M)
    key = (model.E, model.topk, model.N, model.K, par.tp, par.ep, rank, m_cap)
    with _CTX_LOCK:
        ctx = _CTX_CACHE.get(key)
        if ctx is None:
            if len(_CTX_CACHE) > 32:
                for old in _CTX_CACHE.values():
                    old.close()
                _CTX_CACHE.clear()
            ctx = _lib.Context(rank=rank, world=par.world_size, tp=par.tp, ep=par.ep, device=0,
                               E=model.E, topk=model.topk, N=model.N, K=model.K, m_cap=m_cap)
            _CTX_CACHE[key] = ctx
    return ctx


def device_index(routing: RoutingTable, rank: int, tile_rows: int = DEFAULT_TILE_ROWS,
                 tile_cols: Optional[int] = None) -> Dict[str, np.ndarray]:
    """Run ``moe_index_build`` for ``rank`` and return the host copy of the
    index (flat arrays; see include/comet_b200.h, comet_index_host)."""
    routing.parallel._check_rank(rank)
    ctx = _index_context(routing, rank)
    torch = ctx.torch
    tc = default_tile_cols(routing.model.N) if tile_cols is None else tile_cols
    m = routing.workload.M
    experts = torch.from_numpy(routing.as_array().copy())
    dev = ctx.routing_buffer()[: m * routing.model.topk]
    if m:
        dev.copy_(experts.reshape(-1))
    ctx.index_build(dev, m, tile_rows, tc)
    return ctx.download_index()


def _layout_from_index(idx: Dict[str, np.ndarray], routing: RoutingTable, rank: int
                       ) -> Dict[int, Tuple[Tuple[int, int], ...]]:
    from .config import experts_on_rank
    hosted = experts_on_rank(routing.model, routing.parallel, rank)
    off = idx["row_offsets"]
    tok, src = idx["row_token"].tolist(), idx["row_src"].tolist()
    return {e: tuple(zip(tok[off[j]:off[j + 1]], src[off[j]:off[j + 1]])) for j, e in enumerate(hosted)}


def sort_tokens_by_source(routing: RoutingTable, rank: int) -> Dict[int, Tuple[Tuple[int, int], ...]]:
    """Per hosted expert, (token, src) rows ordered by ((src - rank) mod W,
    token): local rows first (ref resolver.py:171-195).  Built on the GPU."""
    return _layout_from_index(device_index(routing, rank), routing, rank)


def _tile(tile_id, layer, e, rs, re, layout, rank, c0=0, c1=0) -> Tile:
    rows = layout[e][rs:re]
    deps = frozenset(r for r in rows if r[1] != rank)
    return Tile(tile_id=tile_id, layer=layer, expert=e, row_start=rs, row_stop=re,
                rows=rows, deps=deps, col_start=c0, col_stop=c1)


def resolve_layer0(routing: RoutingTable, rank: int, meta: SharedTensorMeta) -> TileSchedule:
    """Row-decomposed dispatch->GEMM schedule, locality-first
    (ref resolver.py:206-252)."""
    if meta.decomposed_dim != M_DIM:
        raise ConfigurationError(
            "the dispatch->GEMM pipeline can only be decomposed along the token "
            "rows; column decomposition is not feasible for a GEMM input")
    idx = device_index(routing, rank, meta.tile_rows, default_tile_cols(routing.model.N))
    layout = _layout_from_index(idx, routing, rank)
    tiles = tuple(_tile(i, 0, int(e), int(rs), int(re), layout, rank)
                  for i, (e, rs, re, _nd) in enumerate(idx["tiles0"].tolist()))
    return TileSchedule(rank=rank, layer=0, meta=meta, tiles=tiles, layout=layout)


def resolve_layer1(routing: RoutingTable, rank: int, meta: SharedTensorMeta) -> TileSchedule:
    """Column-decomposed GEMM->combine schedule in column waves with one
    reduce chunk per column block (ref resolver.py:255-309)."""
    if meta.decomposed_dim != N_DIM:
        raise ConfigurationError(
            "the GEMM->combine pipeline can only be decomposed along the "
            "embedding columns; token rows are coupled by the topk reduction")
    idx = device_index(routing, rank, meta.tile_rows, meta.tile_cols)
    layout = _layout_from_index(idx, routing, rank)
    tiles = tuple(_tile(i, 1, int(e), int(rs), int(re), layout, rank, int(c0), int(c1))
                  for i, (e, rs, re, c0, c1, _nd) in enumerate(idx["tiles1"].tolist()))
    chunks = tuple(ReduceChunk(chunk_id=c, col_start=int(c0), col_stop=int(c1),
                               prereq_tile_ids=frozenset(range(int(first), int(first) + int(n))))
                   for c, (c0, c1, first, n) in enumerate(idx["chunks"].tolist()))
    return TileSchedule(rank=rank, layer=1, meta=meta, tiles=tiles, reduce_chunks=chunks, layout=layout)


def _col_ranges(cols: int, step: int) -> List[Tuple[int, int]]:
    return [(s, min(s + step, cols)) for s in range(0, cols, step)]


def validate_schedule(schedule: TileSchedule, routing: RoutingTable,
                      rank: Optional[int] = None) -> List[Violation]:
    """Defects of ``schedule`` against the routing; [] when clean
    (ref resolver.py:342-441, same codes).  The expected cover comes from the
    GPU index build."""
    rank = schedule.rank if rank is None else rank
    if rank != schedule.rank:
        return [Violation("rank-mismatch", None,
                          f"schedule built for rank {schedule.rank}, validated against {rank}")]
    meta = schedule.meta
    idx = device_index(routing, rank, meta.tile_rows,
                       meta.tile_cols if meta.decomposed_dim == N_DIM else default_tile_cols(routing.model.N))
    layout = _layout_from_index(idx, routing, rank)
    cols = _col_ranges(meta.cols, meta.tile_cols) if meta.decomposed_dim == N_DIM else [(0, 0)]
    expected = {}
    for e in sorted(layout):
        rows = layout[e]
        for rs in range(0, len(rows), meta.tile_rows):
            re = min(rs + meta.tile_rows, len(rows))
            chunk = rows[rs:re]
            deps = frozenset(r for r in chunk if r[1] != rank)
            for c0, c1 in cols:
                expected[(e, rs, re, c0, c1)] = (chunk, deps)
    out: List[Violation] = []
    seen: Dict[tuple, int] = {}
    routed = routing.as_array()
    for tile in schedule.tiles:
        key = (tile.expert, tile.row_start, tile.row_stop, tile.col_start, tile.col_stop)
        if key in seen:
            out.append(Violation("duplicate-tile", tile.tile_id, f"tile {key} appears more than once"))
            continue
        seen[key] = tile.tile_id
        if key not in expected:
            out.append(Violation("unexpected-tile", tile.tile_id, f"tile {key} not part of the cover"))
            continue
        rows, deps = expected[key]
        if tile.rows != rows:
            out.append(Violation("bad-rows", tile.tile_id, f"tile {key} rows disagree with the sorted layout"))
        if tile.deps != deps:
            out.append(Violation("bad-deps", tile.tile_id,
                                 f"tile {key} dependency set is not exactly its remote rows"))
        for t, _src in tile.deps:
            if not (0 <= t < routing.workload.M and (routed[t] == tile.expert).any()):
                out.append(Violation("unrouted-dep", tile.tile_id,
                                     f"token {t} is not routed to expert {tile.expert}"))
    for key in expected:
        if key not in seen:
            out.append(Violation("missing-tile", None, f"tile {key} missing from the schedule"))
    if schedule.layer == 1 or schedule.reduce_chunks:
        ranges = _col_ranges(meta.cols, meta.tile_cols)
        by_id = {t.tile_id for t in schedule.tiles}
        if len(schedule.reduce_chunks) != len(ranges):
            out.append(Violation("bad-reduce-count", None,
                                 f"expected {len(ranges)} reduce chunks, got {len(schedule.reduce_chunks)}"))
        last = -1
        for ch in schedule.reduce_chunks:
            if ch.chunk_id <= last:
                out.append(Violation("reduce-order", ch.chunk_id,
                                     "reduce chunks not emitted in ascending column order"))
            last = ch.chunk_id
            members = {t.tile_id for t in schedule.tiles if (t.col_start, t.col_stop) == (ch.col_start, ch.col_stop)}
            if not members >= ch.prereq_tile_ids:
                out.append(Violation("alien-prereq", ch.chunk_id,
                                     "reduce chunk lists a prerequisite outside its column block"))
            if not ch.prereq_tile_ids >= members:
                out.append(Violation("premature-reduce", ch.chunk_id,
                                     "reduce chunk would fire before all of its column's tiles complete"))
            for tid in ch.prereq_tile_ids:
                if tid not in by_id:
                    out.append(Violation("unknown-prereq", ch.chunk_id,
                                         f"prerequisite tile {tid} not in schedule"))
    return out
