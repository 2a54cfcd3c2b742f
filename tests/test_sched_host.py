"""The layer kernel's unit schedule (csrc/sched.cuh, host+device code),
checked on the CPU: tests/sched_harness.cu enumerates the fused launch's
claim sequence for 4000 random shapes / knob sets (rasters, layer0 tail
halves, layer1 split halves, split-K, narrow blocks, the zero-copy
interleave) and asserts coverage, H-before-layer1 and per-n-block fold
ordering (see the harness header)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_unit_schedule_properties(tmp_path):
    exe = tmp_path / "sched_harness"
    b = subprocess.run(["nvcc", "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                        os.path.join(ROOT, "tests", "sched_harness.cu")], capture_output=True, text=True, timeout=300)
    assert b.returncode == 0, b.stderr[-3000:]
    r = subprocess.run([str(exe), "4000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout[-2000:] + r.stderr[-2000:]
