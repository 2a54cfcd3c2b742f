cd $GRAFT_REPO_ROOT
COMET_SAME_DEVICE=1 COMET_GRID=74 COMET_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n2u.log 2>&1; echo "rc=$?"
tail -1 gpurun_out/n2u.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('unfused_ms'), d.get('unfused_error'))"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('unfused_ms'), d.get('unfused_error'))"
