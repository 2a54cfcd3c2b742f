cd $GRAFT_REPO_ROOT
for i in 1 2; do for dbg in 0 131072; do
for cfg in "MX 8 1 64" "PH 4 2 64" "QW 8 1 64"; do set -- $cfg
echo -n "DEBUG=$dbg $1 ep$2: "; COMET_DEBUG=$dbg timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done; done
for dbg in 0 131072; do echo -n "bench DEBUG=$dbg: "; COMET_DEBUG=$dbg timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-unfused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['clocks']['sm_mhz'])"; done
