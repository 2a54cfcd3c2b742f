cd $GRAFT_REPO_ROOT
COMET_SAME_DEVICE=1 COMET_GRID=36 COMET_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-unfused > gpurun_out/n4.log 2>&1; echo "rc=$?"
grep -v "^\s*$" gpurun_out/n4.log | grep -iE "error|Traceback|exception|value" | head -20
COMET_SAME_DEVICE=1 COMET_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 2>&1 | tail -1 | cut -c1-200
