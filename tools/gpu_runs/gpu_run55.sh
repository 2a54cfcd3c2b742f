cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_failure.py -q -x -m gpu 2>&1 | tail -15
nvidia-smi --query-gpu=name,utilization.gpu --format=csv
timeout 120 python -m pytest tests/test_gpu_layer.py -q -x -m gpu -k "launch_modes" 2>&1 | tail -2
