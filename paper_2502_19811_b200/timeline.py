"""Measured per-CTA timelines, scored and audited like the reference's
simulated ones.

The fused kernels stamp ``%globaltimer`` intervals per CTA and role
(``comet_timeline_enable``/``comet_timeline_dump``).  This module converts
them to the reference simulator's ``Interval`` / timeline CSV schema
(``block_id,block_kind,task_id,start_ns,end_ns``, simulator.py:175-245) and
computes the same overlap metrics as ``_finalize`` (simulator.py:578-617):
union of communication busy time, union of compute busy time, exposed
communication (comm active while no compute block is busy) and the hidden
fraction ``1 - exposed / comm_union``.  ``audit`` checks the measured
dependency order the reference's ``audit_timeline`` (simulator.py:791-879)
checks on simulated runs: per-block interval exclusivity, and no compute
task starting before the communication it depends on finished.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, List, Sequence, Tuple


@dataclass(frozen=True)
class Interval:
    """One busy slot on one CTA (ref simulator.py:175-185)."""

    block_id: int
    block_kind: str  # "compute" | "comm"
    task_id: int
    start_ns: int
    end_ns: int


COMPUTE_ROLES = ("mma",)
COMM_ROLES = ("comm",)


def from_records(records: Iterable[Tuple[int, str, int, int, int]], t0: int = None) -> List[Interval]:
    """(cta, role, task, start, end) records -> Intervals (MMA = compute,
    comm-CTA jobs = comm), times rebased to the earliest record."""
    recs = [r for r in records if r[1] in COMPUTE_ROLES + COMM_ROLES]
    if not recs:
        return []
    base = min(r[3] for r in recs) if t0 is None else t0
    return [Interval(c, "compute" if role in COMPUTE_ROLES else "comm", task, s - base, e - base)
            for c, role, task, s, e in recs]


def timeline_csv(intervals: Sequence[Interval]) -> str:
    """Reference CSV schema and ordering (simulator.py:235-245)."""
    lines = ["block_id,block_kind,task_id,start_ns,end_ns"]
    for iv in sorted(intervals, key=lambda iv: (iv.start_ns, iv.block_id, iv.end_ns, iv.task_id)):
        lines.append(f"{iv.block_id},{iv.block_kind},{iv.task_id},{iv.start_ns},{iv.end_ns}")
    return "\n".join(lines) + "\n"


def _union(spans: List[Tuple[int, int]]) -> int:
    total, end = 0, -1
    for s, e in sorted(spans):
        if s > end:
            total += e - s
            end = e
        elif e > end:
            total += e - end
            end = e
    return total


def _exposed(spans: List[Tuple[int, int]], cover: List[Tuple[int, int]]) -> int:
    ev = [(s, 0, 1) for s, e in spans if s < e] + [(e, 0, -1) for s, e in spans if s < e]
    ev += [(s, 1, 1) for s, e in cover if s < e] + [(e, 1, -1) for s, e in cover if s < e]
    ev.sort()
    exposed = active = covered = 0
    prev = 0
    for pos, which, delta in ev:
        if active > 0 and covered == 0:
            exposed += pos - prev
        prev = pos
        if which == 0:
            active += delta
        else:
            covered += delta
    return exposed


def metrics(intervals: Sequence[Interval]) -> Dict[str, float]:
    """The reference's _finalize metrics on a measured timeline."""
    comm = [(iv.start_ns, iv.end_ns) for iv in intervals if iv.block_kind == "comm"]
    comp = [(iv.start_ns, iv.end_ns) for iv in intervals if iv.block_kind == "compute"]
    latency = max((iv.end_ns for iv in intervals), default=0)
    cu = _union(comm)
    exp = _exposed(comm, comp)
    busy: Dict[int, int] = {}
    for iv in intervals:
        if iv.block_kind == "compute":
            busy[iv.block_id] = busy.get(iv.block_id, 0) + iv.end_ns - iv.start_ns
    return {"total_latency_ns": latency, "comm_busy_ns": cu, "compute_busy_ns": _union(comp),
            "exposed_comm_ns": exp, "hidden_fraction": 1.0 if cu == 0 else 1.0 - exp / cu,
            "mean_compute_bubble_ns": (sum(latency - b for b in busy.values()) / len(busy)) if busy else 0.0}


def audit(intervals: Sequence[Interval], deps: Dict[int, List[int]] = None) -> List[str]:
    """Per-block exclusivity, plus: compute task ``t`` must not start before
    every comm task in ``deps[t]`` ended (measured dependency safety)."""
    problems: List[str] = []
    per: Dict[int, List[Interval]] = {}
    for iv in intervals:
        per.setdefault(iv.block_id, []).append(iv)
        if iv.end_ns < iv.start_ns:
            problems.append(f"block {iv.block_id}: negative interval for task {iv.task_id}")
    for b, ivs in sorted(per.items()):
        ivs = sorted(ivs, key=lambda iv: iv.start_ns)
        for a, c in zip(ivs, ivs[1:]):
            if c.start_ns < a.end_ns and a.block_kind == c.block_kind:
                problems.append(f"block {b}: [{a.start_ns},{a.end_ns}) overlaps [{c.start_ns},{c.end_ns})")
    if deps:
        comm_end: Dict[int, int] = {}  # a task split over several intervals ends with its last
        for iv in intervals:
            if iv.block_kind == "comm":
                comm_end[iv.task_id] = max(comm_end.get(iv.task_id, iv.end_ns), iv.end_ns)
        for iv in intervals:
            if iv.block_kind != "compute":
                continue
            for d in deps.get(iv.task_id, ()):
                if d in comm_end and comm_end[d] > iv.start_ns:
                    problems.append(f"compute task {iv.task_id} started before comm task {d} ended")
    return problems
