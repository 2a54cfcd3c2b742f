cd $GRAFT_REPO_ROOT
COMET_SAME_DEVICE=1 COMET_GRID=36 COMET_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-unfused > gpurun_out/n4.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/n4.log | cut -c1-250; grep -E "Error" gpurun_out/n4.log | head -3
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | cut -c1-120
