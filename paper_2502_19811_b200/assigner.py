"""Adaptive compute/communication block split, chosen from measured timings.

Mirror of `pkg/src/moepipe/assigner.py` (the split knob of
`simulator.py:45-65`).  ``KernelSplit``, ``split_for``, ``SplitKey``,
``SplitRecord``, ``SplitMetadata``, ``select_split`` and
``UnprofiledConfigError`` keep the reference's semantics and JSON schema
(assigner.py:44-292): argmin over the sweep curve with ties to the smaller
n_c, exact-key lookup else the nearest log2 token bucket (ties to the
smaller M), refusal when nothing compatible was profiled.

What changes on B200: ``sweep_split`` times the real fused layer kernels on
this GPU (CUDA events, median over repeats) instead of running the
discrete-event simulator, and records ``cost="b200"`` with ``blocks`` = the
device's SM count.  n_c is the number of communication CTAs of the fused
layer kernels (layer1's combine CTAs; layer0's NVLink dispatch CTAs when the
layer has remote rows).
"""

from __future__ import annotations

import json
import math
import os
import tempfile
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

from .config import ConfigurationError, ModelConfig, ParallelSpec, WorkloadSpec, canonical_json


class UnprofiledConfigError(ConfigurationError):
    """No profiled record is compatible with the query (ref assigner.py:40-41)."""


@dataclass(frozen=True)
class KernelSplit:
    """n thread blocks = n_p compute + n_c communication (ref simulator.py:45-61)."""

    n: int
    n_p: int
    n_c: int

    def __post_init__(self) -> None:
        if self.n_p < 1 or self.n_c < 1:
            raise ConfigurationError(
                f"both block pools need at least one block, got n_p={self.n_p}, n_c={self.n_c}")
        if self.n_p + self.n_c != self.n:
            raise ConfigurationError(f"n_p + n_c must equal n: {self.n_p} + {self.n_c} != {self.n}")


def split_for(n: int, n_c: int) -> KernelSplit:
    return KernelSplit(n=n, n_p=n - n_c, n_c=n_c)


_KEY_FIELDS = ("m", "tp", "ep", "experts", "topk", "embed", "hidden", "cost", "blocks")


@dataclass(frozen=True)
class SplitKey:
    """One profiled configuration; ``m`` is the token bucket (ref 44-117)."""

    m: int
    tp: int
    ep: int
    experts: int
    topk: int
    embed: int
    hidden: int
    cost: str
    blocks: int

    def compatible(self, other: "SplitKey") -> bool:
        return all(getattr(self, f) == getattr(other, f) for f in _KEY_FIELDS if f != "m")

    def to_json_dict(self) -> dict:
        return {f: getattr(self, f) for f in _KEY_FIELDS}

    @classmethod
    def from_json_dict(cls, data: dict) -> "SplitKey":
        vals = {f: (str(data[f]) if f == "cost" else int(data[f])) for f in _KEY_FIELDS}
        return cls(**vals)

    @classmethod
    def for_config(cls, model: ModelConfig, parallel: ParallelSpec, m_tokens: int,
                   cost_name: str, blocks: int) -> "SplitKey":
        return cls(m=m_tokens, tp=parallel.tp, ep=parallel.ep, experts=model.E, topk=model.topk,
                   embed=model.N, hidden=model.K, cost=cost_name, blocks=blocks)


@dataclass(frozen=True)
class SplitRecord:
    """Sweep curve and its argmin (ref 120-153)."""

    key: SplitKey
    optimal_nc: int
    latency_ns: int
    curve: Tuple[Tuple[int, int], ...]
    # B200 extension (absent from the reference schema, optional in the
    # JSON): the layer0 pair-group size the curve was measured at, chosen
    # jointly with n_c by the sweep (the curve is the one at this group)
    group0: Optional[int] = None

    def __post_init__(self) -> None:
        if not self.curve:
            raise ConfigurationError("sweep curve is empty")
        best = min(self.curve, key=lambda pt: (pt[1], pt[0]))
        if (self.optimal_nc, self.latency_ns) != best:
            raise ConfigurationError("stored optimum is not the argmin of the stored curve")

    def to_json_dict(self) -> dict:
        out = {"key": self.key.to_json_dict(), "optimal_nc": self.optimal_nc,
               "latency_ns": self.latency_ns, "curve": [list(pt) for pt in self.curve]}
        if self.group0 is not None:
            out["group0"] = self.group0
        return out

    @classmethod
    def from_json_dict(cls, data: dict) -> "SplitRecord":
        return cls(key=SplitKey.from_json_dict(data["key"]), optimal_nc=int(data["optimal_nc"]),
                   latency_ns=int(data["latency_ns"]),
                   curve=tuple((int(a), int(b)) for a, b in data["curve"]),
                   group0=int(data["group0"]) if data.get("group0") is not None else None)


@dataclass
class SplitMetadata:
    """Flat store of records persisted as one JSON file (ref 156-197)."""

    records: List[SplitRecord]

    def add(self, record: SplitRecord) -> None:
        self.records = [r for r in self.records if r.key != record.key] + [record]

    def to_json_str(self) -> str:
        ordered = sorted(self.records, key=lambda r: tuple(sorted(r.key.to_json_dict().items())))
        return canonical_json({"records": [r.to_json_dict() for r in ordered]})

    @classmethod
    def from_json_str(cls, text: str) -> "SplitMetadata":
        return cls(records=[SplitRecord.from_json_dict(r) for r in json.loads(text).get("records", [])])

    def save(self, path: str) -> None:
        """Whole-file atomic replace."""
        fd, tmp = tempfile.mkstemp(dir=os.path.dirname(os.path.abspath(path)), suffix=".tmp")
        try:
            with os.fdopen(fd, "w") as fh:
                fh.write(self.to_json_str())
            os.replace(tmp, path)
        except BaseException:
            if os.path.exists(tmp):
                os.unlink(tmp)
            raise

    @classmethod
    def load(cls, path: str) -> "SplitMetadata":
        with open(path) as fh:
            return cls.from_json_str(fh.read())


def candidate_ncs(blocks: int, stride: int = 2, max_nc: Optional[int] = None) -> List[int]:
    """Even n_c candidates (2-CTA clusters) from 2 to ``max_nc``."""
    if stride < 1:
        raise ConfigurationError(f"stride must be >= 1, got {stride}")
    hi = min(blocks - 2, max_nc if max_nc is not None else blocks - 2)
    out = list(range(2, hi + 1, max(2, stride + (stride & 1))))
    if not out:
        raise ConfigurationError("no candidate split")
    return out


def record_from_curve(key: SplitKey, points: Sequence[Tuple[int, int]], group0: Optional[int] = None) -> SplitRecord:
    curve = tuple(sorted((int(a), int(b)) for a, b in points))
    nc, ns = min(curve, key=lambda pt: (pt[1], pt[0]))
    return SplitRecord(key=key, optimal_nc=nc, latency_ns=ns, curve=curve, group0=group0)


def sweep_split(model: ModelConfig, parallel: ParallelSpec, workload: WorkloadSpec,
                cost=None, cost_name: str = "b200", blocks: Optional[int] = None,
                stride: int = 2, rank: int = 0, max_nc: int = 16, repeats: int = 5,
                measure: Optional[Callable[..., float]] = None,
                candidates: Optional[Sequence[int]] = None,
                groups: Optional[Sequence[int]] = None, passes: int = 1) -> SplitRecord:
    """Measure the fused layer at each candidate n_c and record the argmin.

    ``measure(n_c) -> seconds`` defaults to timing the layer on this GPU with
    synthetic tokens and random weights of the model's shape, every rank of
    ``parallel`` emulated on the device (``measure.EmulatedGroup``: latency =
    max over ranks of the rank's kernel time, the other knobs at the product
    defaults of ``LayerKnobs.for_world``).  ``candidates`` overrides the
    even grid ``candidate_ncs(blocks, stride, max_nc)``.  ``cost`` is
    accepted for signature compatibility with the reference and ignored.
    ``groups`` (B200 extension): layer0 pair-group sizes swept jointly with
    n_c (``measure(n_c, group0)``); the record keeps the curve of the best
    group and that group in ``group0``.  ``passes`` > 1 measures the whole
    grid that many times round-robin and keeps each point's minimum (robust
    to slow drift of the clock between points of a flat curve).
    """
    if blocks is None:
        from . import _lib
        blocks = _lib.device_info(0)["sms"]
    if measure is None:
        measure = _default_measure(model, parallel, workload, repeats)
    cands = list(candidates) if candidates is not None else candidate_ncs(blocks, stride, max_nc)
    key = SplitKey.for_config(model, parallel, workload.M, cost_name, blocks)
    if not groups:
        lat = {nc: min(measure(nc) for _ in range(max(1, passes))) for nc in cands}
        return record_from_curve(key, [(nc, int(round(lat[nc] * 1e9))) for nc in cands])
    lat = {}
    for _ in range(max(1, passes)):
        for g in groups:
            for nc in cands:
                t = measure(nc, g)
                lat[(g, nc)] = min(t, lat.get((g, nc), t))
    curves = {g: [(nc, int(round(lat[(g, nc)] * 1e9))) for nc in cands] for g in groups}
    best = min(groups, key=lambda g: (min(ns for _, ns in curves[g]), g))
    return record_from_curve(key, curves[best], group0=best)


def _default_measure(model, parallel, workload, repeats):
    import dataclasses
    from .executor import LayerKnobs
    from .measure import EmulatedGroup
    from .routing import build_routing
    routing = build_routing(model, parallel, workload)
    grp = EmulatedGroup(model, parallel, routing, seed=workload.seed + 2)
    base = LayerKnobs.for_world(parallel.world_size)

    def measure(nc, group0=None):
        grp.set_knobs(dataclasses.replace(base, n_comm0=nc, group0=group0))
        return grp.measure(iters=repeats)["latency_ms"] * 1e-3
    return measure


def select_split(metadata: SplitMetadata, query: SplitKey) -> KernelSplit:
    """Exact key, else nearest log2 token bucket (ties -> smaller M), else
    ``UnprofiledConfigError`` (ref assigner.py:260-292)."""
    chosen = select_record(metadata, query)
    return split_for(chosen.key.blocks, chosen.optimal_nc)


def select_record(metadata: SplitMetadata, query: SplitKey) -> SplitRecord:
    """The record ``select_split`` picks (same lookup rules)."""
    if not metadata.records:
        raise UnprofiledConfigError("split metadata is empty")
    compatible = [r for r in metadata.records if r.key.compatible(query)]
    if not compatible:
        raise UnprofiledConfigError(
            f"unprofiled configuration: no record matches {query.to_json_dict()} "
            "in every field but the token count")
    exact = [r for r in compatible if r.key.m == query.m]
    if exact:
        chosen = exact[0]
    else:
        if query.m < 1:
            raise UnprofiledConfigError(f"cannot bucket a token count of {query.m}; profile it explicitly")
        chosen = min(compatible, key=lambda r: (abs(math.log2(query.m) - math.log2(r.key.m)), r.key.m))
    return chosen


# ---------------------------------------------------------------------------
# The product path's chooser (paper section 3.3: n_c from measured timings)
# ---------------------------------------------------------------------------

DEFAULT_METADATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "split_b200.json")
_default_meta: Optional[SplitMetadata] = None


def default_metadata() -> SplitMetadata:
    """The committed n_c sweep measured on B200 (tools/sweep_b200.py ->
    ``split_b200.json``, the reference's SplitMetadata schema, cost "b200")."""
    global _default_meta
    if _default_meta is None:
        _default_meta = SplitMetadata.load(DEFAULT_METADATA) if os.path.exists(DEFAULT_METADATA) \
            else SplitMetadata(records=[])
    return _default_meta


def choose_split(model: ModelConfig, parallel: ParallelSpec, m_tokens: int, blocks: int,
                 metadata: Optional[SplitMetadata] = None) -> Tuple[KernelSplit, str]:
    """Communication blocks n_c of the fused layer for ``m_tokens`` tokens, as
    the reference's cli picks them (cli.py:228-235): ``select_split`` on the
    measured metadata (exact key, else the nearest log2 token bucket,
    assigner.py:260-292); for an unprofiled shape the fitted b200 cost model
    (costmodel.predict_split) instead of ``UnprofiledConfigError``.  Returns
    (split, "measured" | "model")."""
    split, src, _ = choose_knobs(model, parallel, m_tokens, blocks, metadata)
    return split, src


def default_group0(world: int) -> int:
    """Layer0 pair-group size without a measured record: 8
    pairs at EP = 1 and EP >= 8, 4 at EP = 2/4."""
    return 8 if world == 1 or world >= 8 else 4


def choose_knobs(model: ModelConfig, parallel: ParallelSpec, m_tokens: int, blocks: int,
                 metadata: Optional[SplitMetadata] = None) -> Tuple[KernelSplit, str, int]:
    """``choose_split`` plus the layer0 pair-group size measured with it
    (the record's ``group0``; ``default_group0`` when the record has none or
    the cost model answered)."""
    meta = metadata if metadata is not None else default_metadata()
    try:
        rec = select_record(meta, SplitKey.for_config(model, parallel, m_tokens, "b200", blocks))
        g0 = rec.group0 if rec.group0 is not None else default_group0(parallel.world_size)
        return split_for(rec.key.blocks, rec.optimal_nc), "measured", g0
    except UnprofiledConfigError:
        from .costmodel import predict_split
        rec = predict_split(model, parallel, WorkloadSpec(M=max(1, m_tokens), seed=0))
        return split_for(blocks, min(rec.optimal_nc, blocks - 2)), "model", default_group0(parallel.world_size)
