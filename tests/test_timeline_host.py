"""Timeline scoring/audit host logic (reference _finalize / audit_timeline
semantics, simulator.py:578-617, 791-879) on synthetic intervals."""

from paper_2502_19811_b200.timeline import Interval, audit, from_records, metrics, timeline_csv


def test_metrics_hidden_fraction_and_csv():
    ivs = [Interval(0, "compute", 0, 0, 100), Interval(1, "comm", 5, 50, 150), Interval(1, "comm", 6, 150, 160)]
    m = metrics(ivs)
    assert m["comm_busy_ns"] == 110 and m["compute_busy_ns"] == 100
    assert m["exposed_comm_ns"] == 60
    assert abs(m["hidden_fraction"] - (1 - 60 / 110)) < 1e-12
    assert m["total_latency_ns"] == 160
    csv = timeline_csv(ivs).splitlines()
    assert csv[0] == "block_id,block_kind,task_id,start_ns,end_ns"
    assert csv[1] == "0,compute,0,0,100"


def test_audit_detects_overlap_and_early_start():
    ivs = [Interval(0, "compute", 1, 0, 10), Interval(0, "compute", 2, 5, 20), Interval(3, "comm", 7, 0, 12)]
    probs = audit(ivs, deps={1: [7]})
    assert any("overlaps" in p for p in probs)
    assert any("before comm task 7" in p for p in probs)
    assert audit([Interval(0, "compute", 1, 20, 30), Interval(3, "comm", 7, 0, 12)], deps={1: [7]}) == []


def test_from_records_rebases_and_filters_roles():
    recs = [(0, "mma", 3, 1000, 1100), (5, "comm", 9, 990, 1010), (0, "epilogue", 3, 1100, 1150)]
    ivs = from_records(recs)
    assert [iv.block_kind for iv in ivs] == ["compute", "comm"]
    assert min(iv.start_ns for iv in ivs) == 0
