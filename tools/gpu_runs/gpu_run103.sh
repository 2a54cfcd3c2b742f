cd $GRAFT_REPO_ROOT
COMET_SAME_DEVICE=1 COMET_GRID=18 COMET_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu-baseline --no-unfused > gpurun_out/n8.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/n8.log | cut -c1-250; grep -E "Error" gpurun_out/n8.log | head -3
