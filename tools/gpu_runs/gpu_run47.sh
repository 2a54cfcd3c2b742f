cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "dedup" 2>&1 | tail -3
