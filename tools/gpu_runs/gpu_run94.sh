cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -m gpu -k "zerocopy or full_size" 2>&1 | tail -2
timeout 900 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
