cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy" > gpurun_out/pytest_zc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zc.log
tail -3 gpurun_out/pytest_zc.log; grep -E "^E " gpurun_out/pytest_zc.log | head -8
for L in 0 2 3; do for D in 8 16; do echo "== ILV=$L DL=$D"; COMET_ZC_DL=$D COMET_ZC_ILV=$L MODE=zc NC0=16 timeout 120 python tools/stream_probe.py 2>&1 | tail -8 | head -1; done; done
for D in 4 8; do echo "== ILV=2 NC0=32 DL=$D"; COMET_ZC_DL=$D COMET_ZC_ILV=2 MODE=zc NC0=32 timeout 120 python tools/stream_probe.py 2>&1 | tail -8 | head -1; done
