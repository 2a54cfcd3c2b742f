cd $GRAFT_REPO_ROOT
for cfg in "8 4" "16 4" "4 4" "8 8" "8 2" "8 4" "16 8"; do set -- $cfg
echo -n "G1=$1 wave1=$2: "; COMET_G1=$1 timeout 300 python bench.py --steps 40 --warmup 5 --wave1 $2 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['clocks']['sm_mhz'])"
done
