"""CPU oracle for the fused MoE layer path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker or the timed CPU arm.  The product package
(``paper_2502_19811_b200``) never imports it: its index build and layer
arithmetic run in the sm_100a kernels of ``libcomet_b200.so`` and fail loudly
when that library is missing.

What it restates (numpy, vectorised), each function citing the reference
line range it follows under ``/root/reference/pkg/src/moepipe/``:

* integer path, bit-exact targets for the CUDA index builder:
  ``expert_counts`` / ``transfer_counts`` (routing.py:78-117),
  ``sort_layout`` (resolver.py:171-195), ``layer0_tiles`` (resolver.py:206-252),
  ``layer1_tiles`` (resolver.py:255-309);
* router front-end: ``router_topk`` -- gate logits ->
  top-k expert ids stored ascending (the RoutingTable.experts_per_token
  layout, routing.py:146-163) + softmax combine weights in the same slot
  order (executor.py:102-120).  The reference has no router
  (``build_routing``, routing.py:283-307, synthesises counts), so this one
  is **parity unpinned** against the reference: it is defined here as a
  stable descending argsort and pinned by construction-level checks only;
* float path: ``layer_forward`` = ``execute_naive`` (executor.py:132-148) with
  ``_hidden_row`` (86-90), ``_output_columns`` (93-99) and ``_combine``
  (102-120) folded into one GEMM pair per expert; ``layer_forward_tp`` =
  ``execute_tp_sharded`` (executor.py:221-246); ``execute_naive_literal`` =
  the reference's loop nest itself (one dot per (token, expert) hidden row
  and per output column), the literal CPU arm at Config 1.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
``tests/golden/*`` -- fixtures produced by running the reference package
itself (``tests/golden/make_golden.py``, committed) -- and against the
reference's own known-answer tests (test_resolver.py:131-141, 163-168,
186-195, 208-222; test_routing.py:128-149).  The float path is pinned to the
literal fp64 ``execute_naive`` output at Config 1 to <= 1e-12 relative.
"""

from __future__ import annotations

from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

Activation = Optional[Callable[[np.ndarray], np.ndarray]]


# ---------------------------------------------------------------------------
# Integer path
# ---------------------------------------------------------------------------

def source_ranks(m_tokens: int, world: int) -> np.ndarray:
    """src rank of every token (routing.py:86-95)."""
    t = np.arange(m_tokens, dtype=np.int64)
    base = m_tokens // world
    if base == 0:
        return np.full(m_tokens, world - 1, dtype=np.int64)
    return np.minimum(t // base, world - 1)


def expert_counts(experts: np.ndarray, E: int) -> np.ndarray:
    """Tokens per expert (routing.py:78-84)."""
    return np.bincount(experts.ravel().astype(np.int64), minlength=E)[:E]


def transfer_counts(experts: np.ndarray, E: int, tp: int, ep: int) -> np.ndarray:
    """[src][dst] received rows; one per TP rank of the owning group
    (routing.py:106-117)."""
    world = tp * ep
    m = experts.shape[0]
    src = source_ranks(m, world)
    per_group = E // ep
    mat = np.zeros((world, world), dtype=np.int64)
    grp = experts.astype(np.int64) // per_group          # [M, topk]
    for g in range(ep):
        n_rows = np.bincount(src, weights=(grp == g).sum(axis=1), minlength=world)
        for d in range(g * tp, (g + 1) * tp):
            mat[:, d] += n_rows.astype(np.int64)
    return mat


def sort_layout(experts: np.ndarray, E: int, tp: int, ep: int, rank: int
                ) -> Dict[int, np.ndarray]:
    """Per hosted expert, rows (token, src) ordered by ((src - rank) mod W,
    token) -- local rows first (resolver.py:171-195).  Returns
    {expert: int64[n_rows, 2]}."""
    world = tp * ep
    m = experts.shape[0]
    src = source_ranks(m, world)
    per_group = E // ep
    g = rank // tp
    out: Dict[int, np.ndarray] = {}
    ring = (src - rank) % world
    for e in range(g * per_group, (g + 1) * per_group):
        toks = np.flatnonzero((experts == e).any(axis=1))
        order = np.lexsort((toks, ring[toks]))
        toks = toks[order]
        out[e] = np.stack([toks, src[toks]], axis=1) if toks.size else np.zeros((0, 2), np.int64)
    return out


def _row_chunks(n: int, step: int) -> List[Tuple[int, int]]:
    return [(s, min(s + step, n)) for s in range(0, n, step)]


def layer0_tiles(layout: Dict[int, np.ndarray], rank: int, tile_rows: int) -> np.ndarray:
    """Tiles (expert, row_start, row_stop, n_deps) sorted by
    (n_deps, expert, row_start) (resolver.py:206-252)."""
    recs = []
    for e in sorted(layout):
        rows = layout[e]
        remote = rows[:, 1] != rank
        for lo, hi in _row_chunks(len(rows), tile_rows):
            recs.append((e, lo, hi, int(remote[lo:hi].sum())))
    arr = np.array(recs, dtype=np.int64).reshape(-1, 4)
    if len(arr):
        arr = arr[np.lexsort((arr[:, 1], arr[:, 0], arr[:, 3]))]
    return arr


def layer1_tiles(layout: Dict[int, np.ndarray], rank: int, tile_rows: int,
                 tile_cols: int, n_embed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Column-wave tiles (expert, row_start, row_stop, col_start, col_stop,
    n_deps) in tile_id order, and reduce chunks (col_start, col_stop,
    first_tile_id, n_tiles): chunk c waits for exactly its column's tiles
    (resolver.py:255-309)."""
    per_col = []
    for e in sorted(layout):
        rows = layout[e]
        remote = rows[:, 1] != rank
        for lo, hi in _row_chunks(len(rows), tile_rows):
            per_col.append((e, lo, hi, int(remote[lo:hi].sum())))
    tiles, chunks = [], []
    for c0, c1 in _row_chunks(n_embed, tile_cols):
        chunks.append((c0, c1, len(tiles), len(per_col)))
        for e, lo, hi, nd in per_col:
            tiles.append((e, lo, hi, c0, c1, nd))
    return (np.array(tiles, dtype=np.int64).reshape(-1, 6),
            np.array(chunks, dtype=np.int64).reshape(-1, 4))


def index_for_rank(experts: np.ndarray, E: int, tp: int, ep: int, rank: int,
                   tile_rows: int, tile_cols: int, n_embed: int) -> dict:
    """Everything ``moe_index_build`` emits for one rank, in the flat integer
    form the C-ABI returns (see include/comet_b200.h, struct comet_index_host)."""
    lay = sort_layout(experts, E, tp, ep, rank)
    hosted = sorted(lay)
    counts_h = np.array([len(lay[e]) for e in hosted], dtype=np.int64)
    rows = (np.concatenate([lay[e] for e in hosted]) if counts_h.sum()
            else np.zeros((0, 2), np.int64))
    n_local = np.array([int((lay[e][:, 1] == rank).sum()) for e in hosted], dtype=np.int64)
    t1, ch = layer1_tiles(lay, rank, tile_rows, tile_cols, n_embed)
    return {
        "expert_counts": expert_counts(experts, E),
        "transfer_counts": transfer_counts(experts, E, tp, ep),
        "row_offsets": np.concatenate([[0], np.cumsum(counts_h)]).astype(np.int64),
        "row_token": rows[:, 0],
        "row_src": rows[:, 1],
        "n_local": n_local,
        "tiles0": layer0_tiles(lay, rank, tile_rows),
        "tiles1": t1,
        "chunks": ch,
    }


# ---------------------------------------------------------------------------
# Float path
# ---------------------------------------------------------------------------

def _fold_combine(experts: np.ndarray, rows_by_expert: Dict[int, np.ndarray],
                  pos: Dict[int, np.ndarray], combine_weights: Optional[np.ndarray],
                  out_dtype) -> np.ndarray:
    """out[t] = left fold over t's experts in ascending order, row *
    weight[t, slot] when weights are given (executor.py:102-120)."""
    m, topk = experts.shape
    n = next(iter(rows_by_expert.values())).shape[1] if rows_by_expert else 0
    out = np.zeros((m, n), dtype=out_dtype)
    for slot in range(topk):
        e_col = experts[:, slot]
        contrib = np.empty((m, n), dtype=out_dtype)
        for e in np.unique(e_col):
            toks = np.flatnonzero(e_col == e)
            contrib[toks] = rows_by_expert[int(e)][pos[int(e)][toks]]
        if combine_weights is not None:
            contrib = contrib * combine_weights[:, slot:slot + 1].astype(out_dtype)
        out = contrib if slot == 0 else out + contrib
    return out


def _expert_rows(experts: np.ndarray, E: int):
    toks_of, pos = {}, {}
    for e in range(E):
        toks = np.flatnonzero((experts == e).any(axis=1))
        toks_of[e] = toks
        p = np.full(experts.shape[0], -1, dtype=np.int64)
        p[toks] = np.arange(toks.size)
        pos[e] = p
    return toks_of, pos


def layer_forward(x: np.ndarray, w0: np.ndarray, w1: np.ndarray, experts: np.ndarray,
                  activation: Activation = None,
                  combine_weights: Optional[np.ndarray] = None,
                  dtype=np.float64) -> np.ndarray:
    """Vectorised ``execute_naive`` (executor.py:132-148): per expert
    h = act(x[rows] @ w0[e]) (86-90), y = h @ w1[e] (93-99), then the
    ascending-slot combine (102-120).  ``dtype`` float64 reproduces the
    reference; float32 is the fast CPU arm."""
    E = w0.shape[0]
    toks_of, pos = _expert_rows(experts, E)
    x = np.asarray(x, dtype=dtype)
    rows = {}
    for e in range(E):
        if toks_of[e].size == 0:
            continue
        h = x[toks_of[e]] @ np.asarray(w0[e], dtype=dtype)
        if activation is not None:
            h = activation(h)
        rows[e] = h @ np.asarray(w1[e], dtype=dtype)
    if experts.shape[0] == 0:
        return np.zeros((0, x.shape[1]), dtype=dtype)
    return _fold_combine(experts, rows, pos, combine_weights, dtype)


def execute_naive_literal(x: np.ndarray, w0: np.ndarray, w1: np.ndarray, experts: np.ndarray,
                          activation: Activation = None,
                          combine_weights: Optional[np.ndarray] = None) -> np.ndarray:
    """The reference's ``execute_naive`` loop nest restated literally
    (executor.py:132-148): token-major, per (token, expert) ``_hidden_row``
    = one ``np.dot`` of the token row with w0[e] (86-90), ``_output_columns``
    = one ``np.dot`` per output column (93-99), and ``_combine``'s
    ascending-slot fold (102-120).  Same float64 operations in the same
    order, so it reproduces the reference output bitwise; it is the CPU
    timing arm at Config 1 (524K dot calls, seconds)."""
    x = np.asarray(x, dtype=np.float64)
    m, n = x.shape
    out = np.zeros((m, n), dtype=np.float64)
    for t in range(m):
        acc = None
        for slot, e in enumerate(experts[t]):
            h = np.dot(x[t], w0[e])
            if activation is not None:
                h = activation(h)
            w1_e = w1[e]
            row = np.array([np.dot(h, w1_e[:, j]) for j in range(n)], dtype=np.float64)
            if combine_weights is not None:
                row = row * combine_weights[t, slot]
            acc = row.copy() if acc is None else acc + row
        if acc is not None:
            out[t] = acc
    return out


def layer_forward_tp(x, w0, w1, experts, tp: int, activation: Activation = None,
                     combine_weights=None, dtype=np.float64) -> np.ndarray:
    """``execute_tp_sharded`` (executor.py:221-246): K cut into tp contiguous
    shards, per-(token, expert) partials summed shard-ascending, then combine."""
    E, N, K = w0.shape
    ks = K // tp
    toks_of, pos = _expert_rows(experts, E)
    x = np.asarray(x, dtype=dtype)
    rows = {}
    for e in range(E):
        if toks_of[e].size == 0:
            continue
        xe = x[toks_of[e]]
        acc = np.zeros((xe.shape[0], N), dtype=dtype)
        for s in range(tp):
            h = xe @ np.asarray(w0[e][:, s * ks:(s + 1) * ks], dtype=dtype)
            if activation is not None:
                h = activation(h)
            acc = acc + h @ np.asarray(w1[e][s * ks:(s + 1) * ks, :], dtype=dtype)
        rows[e] = acc
    if experts.shape[0] == 0:
        return np.zeros((0, N), dtype=dtype)
    return _fold_combine(experts, rows, pos, combine_weights, dtype)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    u = a32.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32)


def relative_error(got: np.ndarray, ref: np.ndarray) -> Tuple[float, float]:
    """(max|d| / max|ref|, ||d||_F / ||ref||_F): the tolerance metric stated
    in SURVEY.md section 8(c) (elementwise relative error is unusable: many
    outputs are near zero)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = got - ref
    mx = float(np.abs(ref).max()) if ref.size else 0.0
    fr = float(np.linalg.norm(ref)) if ref.size else 0.0
    return (float(np.abs(d).max()) / mx if mx else float(np.abs(d).max() if d.size else 0.0),
            float(np.linalg.norm(d)) / fr if fr else float(np.linalg.norm(d)))


# ---------------------------------------------------------------------------
# Router front-end (no reference counterpart: parity unpinned)
# ---------------------------------------------------------------------------

def router_topk(logits: np.ndarray, topk: int, norm: str = "topk") -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """Top-k experts per token, stored ascending (routing.py:146-163 layout).

    Selection = stable descending argsort of the logits: larger logit first,
    ties -> smaller expert id; -0.0 ties +0.0; NaN ranks below -inf.
    Weights (float64) in ascending-expert slot order: ``"topk"`` softmax over
    the selected logits, ``"all"`` softmax over all E logits (selected
    entries), ``None`` no weights."""
    lg = np.asarray(logits, dtype=np.float64)
    M, E = lg.shape
    key = np.where(np.isnan(lg), -np.inf, lg)
    # rank NaN strictly below -inf: sort by (isnan, -key, id)
    order = np.lexsort((np.broadcast_to(np.arange(E), (M, E)), -key, np.isnan(lg)), axis=1)
    sel = order[:, :topk]
    experts = np.sort(sel, axis=1).astype(np.int32)
    if norm is None:
        return experts, None
    chosen = np.take_along_axis(lg, experts.astype(np.int64), axis=1)
    if norm == "topk":
        mx = chosen.max(axis=1, keepdims=True) if topk else 0.0
        ex = np.exp(chosen - mx)
        w = ex / ex.sum(axis=1, keepdims=True)
    elif norm == "all":
        mx = lg.max(axis=1, keepdims=True)
        w = np.exp(chosen - mx) / np.exp(lg - mx).sum(axis=1, keepdims=True)
    else:
        raise ValueError(f"unknown norm {norm!r}")
    return experts, w

