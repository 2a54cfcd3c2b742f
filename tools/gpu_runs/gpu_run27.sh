cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_multiproc.py -x -q 2>&1 | tail -30
COMET_SAME_DEVICE=1 COMET_GRID=74 COMET_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-unfused 2>&1 | tail -3
