"""CLI parity (ref pkg/src/moepipe/cli.py) -- host-only subcommands and
error behaviour: routing.json identical to build_routing's, flags > config
file > defaults, exit code 2 on invalid config (the --fuzz check needs the
GPU resolver: tests/test_gpu_cli.py)."""

import json

from paper_2502_19811_b200 import ModelConfig, ParallelSpec, WorkloadSpec, build_routing, model_preset
from paper_2502_19811_b200.cli import _build_experiment, build_parser, main


def test_route_writes_reference_routing(tmp_path):
    rc = main(["route", "--model", "mixtral-8x7b", "--ep", "8", "--tokens", "512", "--std", "0.032",
               "--out-dir", str(tmp_path)])
    assert rc == 0
    text = (tmp_path / "routing.json").read_text()
    ref = build_routing(model_preset("mixtral-8x7b"), ParallelSpec(1, 8), WorkloadSpec(M=512, seed=0, std=0.032))
    assert text == ref.to_json_str()


def test_flags_override_config_file(tmp_path):
    cfg = tmp_path / "exp.json"
    cfg.write_text(json.dumps({"model": {"L": 1, "E": 16, "topk": 2, "N": 256, "K": 512, "dtype_bytes": 2},
                               "parallel": {"tp": 2, "ep": 4}, "workload": {"M": 1000, "seed": 3, "std": 0.0},
                               "sim": {"n_c": 32, "mode": "sequential", "rank": 3}}))
    args = build_parser().parse_args(["run", "--config", str(cfg), "--ep", "2", "--tokens", "640"])
    exp = _build_experiment(args)
    assert exp.model == ModelConfig(L=1, E=16, topk=2, N=256, K=512)
    assert exp.parallel == ParallelSpec(tp=2, ep=2)           # flag wins
    assert exp.workload == WorkloadSpec(M=640, seed=3, std=0.0)
    assert exp.n_c == 32 and exp.mode == "sequential"


def test_invalid_configs_exit_2(tmp_path, capsys):
    assert main(["route", "--model", "no-such-model", "--out-dir", str(tmp_path)]) == 2
    assert main(["run", "--mode", "zigzag", "--out-dir", str(tmp_path)]) == 2
    assert main(["run", "--mode", "coarse:0", "--out-dir", str(tmp_path)]) == 2
    assert main(["run", "--cost", "h800", "--out-dir", str(tmp_path)]) == 2
    assert main(["run", "--ep", "2", "--rank", "5", "--out-dir", str(tmp_path)]) == 2
    assert "error:" in capsys.readouterr().err
