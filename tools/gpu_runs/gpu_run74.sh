cd $GRAFT_REPO_ROOT
for f in 0 1 0 1 0 1; do echo -n "FUSE1=$f: "; COMET_FUSE1=$f timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['clocks']['sm_mhz'])"; done
