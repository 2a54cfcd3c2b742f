cd $GRAFT_REPO_ROOT
for i in 1 2; do
echo -n "new defaults: "; timeout 900 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
echo -n "old (G0=8 ILV=3): "; COMET_ZC_G0=8 COMET_ZC_ILV=3 timeout 900 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
