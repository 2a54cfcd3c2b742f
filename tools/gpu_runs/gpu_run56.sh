cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -m gpu 2>&1 | tail -15
