cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy" > gpurun_out/pytest_zc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zc.log
tail -1 gpurun_out/pytest_zc.log
COMET_ZC_ORDER=1 timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy" > gpurun_out/pytest_zc1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zc1.log
tail -1 gpurun_out/pytest_zc1.log; grep -E "^E " gpurun_out/pytest_zc1.log | head -5
for O in 0 1; do for L in 2 3 5; do echo "== ORDER=$O ILV=$L"; COMET_ZC_ORDER=$O COMET_ZC_ILV=$L MODE=zc NC0=16 timeout 120 python tools/stream_probe.py 2>&1 | tail -10; done; done
