cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -k "streamed or forward_host" 2>&1 | tail -3
timeout 400 python tools/e2e_probe.py 2>&1 | grep -E "H2D|D2H|device forward:|chunks=None|chunks=3"
