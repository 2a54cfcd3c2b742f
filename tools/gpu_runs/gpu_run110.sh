cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -m gpu -k "emulated or golden or fold or narrow or modes or dedup" 2>&1 | tail -1
for i in 1 2; do
echo -n "MX EP8: "; timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured" | sed "s/.*'finish': //" | cut -c1-40
echo -n "PH: "; timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.*'finish': //" | cut -c1-40
done
