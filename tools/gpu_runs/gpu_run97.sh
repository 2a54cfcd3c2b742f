cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for g in 8 16; do
echo -n "group0=$g: "; timeout 300 python bench.py --steps 40 --warmup 5 --group0 $g --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['clocks']['sm_mhz'])"
done; done
