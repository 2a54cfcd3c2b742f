"""The multi-rank protocol with real processes: one process (own CUDA
context and symmetric heap) per rank, IPC-mapped peer heaps, forwards running
concurrently -- on a single-GPU box every rank shares GPU 0 with the SMs split
between the ranks' persistent kernels (LayerKnobs.grid)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tp,ep,topk", [(1, 2, 2), (2, 1, 2), (1, 2, 3), (1, 4, 2), (2, 2, 2), (1, 8, 2)])
def test_processes_share_the_protocol(tp, ep, topk):
    import torch
    world = tp * ep
    grid = torch.cuda.get_device_properties(0).multi_processor_count // world // 2 * 2
    env = dict(os.environ, COMET_SAME_DEVICE="1", COMET_TEST_GRID=str(grid), MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + tp * 100 + ep * 10 + topk),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(tp), str(ep), str(topk)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "MP_OK" in r.stdout, r.stdout[-2000:]
