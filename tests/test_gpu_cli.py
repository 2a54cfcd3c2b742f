"""CLI run / compare / verify on the GPU: measured timeline in the
reference CSV schema, result.json with the reference SimResult fields,
compare.csv over the B200 modes, and the bitwise verify suite."""

import json

import pytest

from paper_2502_19811_b200.cli import main

pytestmark = pytest.mark.gpu
SMALL = ["--model", "mixtral-8x7b", "--tokens", "2048", "--std", "0.032"]


def test_run_writes_measured_result_and_timeline(tmp_path):
    rc = main(["run", "--ep", "4", "--rank", "1", "--nc", "16", "--dump-schedule", "--out-dir", str(tmp_path)] + SMALL)
    assert rc == 0
    res = json.loads((tmp_path / "result.json").read_text())["result"]
    for k in ("mode", "n_p", "n_c", "total_latency_ns", "comm_busy_ns", "compute_busy_ns", "exposed_comm_ns",
              "hidden_fraction", "comm_work_ns", "compute_work_ns", "bubble_ns"):
        assert k in res
    assert res["mode"] == "fine" and res["n_c"] == 16 and res["total_latency_ns"] > 0
    assert 0.0 <= res["hidden_fraction"] <= 1.0 and res["comm_busy_ns"] > 0  # EP=4: NVLink dispatch recorded
    csv = (tmp_path / "timeline.csv").read_text().splitlines()
    assert csv[0] == "block_id,block_kind,task_id,start_ns,end_ns" and len(csv) > 10
    assert (tmp_path / "schedule_layer0.json").exists() and (tmp_path / "schedule_layer1.json").exists()


def test_compare_modes(tmp_path):
    rc = main(["compare", "--ep", "8", "--modes", "fine,sequential,coarse:2", "--out-dir", str(tmp_path)] + SMALL)
    assert rc == 0
    rows = (tmp_path / "compare.csv").read_text().splitlines()
    assert rows[0].startswith("mode,total_latency_ns")
    lat = {r.split(",")[0]: int(r.split(",")[1]) for r in rows[1:]}
    assert set(lat) == {"fine", "sequential", "coarse:2"} and all(v > 0 for v in lat.values())
    rc = main(["compare", "--modes", "fine,unfused", "--out-dir", str(tmp_path)] + SMALL)
    assert rc == 0


def test_verify_bitwise_and_sweep(tmp_path):
    assert main(["verify", "--instances", "3", "--ep", "2"]) == 0
    assert main(["sweep", "--ep", "2", "--tokens", "1024", "--max-nc", "18", "--out-dir", str(tmp_path)]
                + ["--model", "mixtral-8x7b"]) == 0
    md = json.loads((tmp_path / "metadata.json").read_text())
    assert md["records"][0]["key"]["cost"] == "b200"
    assert main(["run", "--ep", "2", "--tokens", "1024", "--auto-split", "--out-dir", str(tmp_path),
                 "--model", "mixtral-8x7b"]) == 0


def test_fuzz_is_detected_exit_1(capsys):
    """A corrupted schedule must be caught by the validator (exit 1)."""
    assert main(["verify", "--fuzz", "--tokens", "24"]) == 1
    out = capsys.readouterr()
    assert "injected corruption detected" in out.out
    assert "verification failed" in out.err
