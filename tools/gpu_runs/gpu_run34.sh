cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy or streamed or forward_host" > gpurun_out/pytest_zc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zc.log
tail -3 gpurun_out/pytest_zc.log; grep -E "^E " gpurun_out/pytest_zc.log | head -8
timeout 300 python tools/e2e_probe.py 2>&1 | tail -22
