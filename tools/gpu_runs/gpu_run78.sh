cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -k "zerocopy_unweighted" 2>&1 | tail -3
