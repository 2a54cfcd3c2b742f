cd $GRAFT_REPO_ROOT
for i in 1 2; do for b in 8 2 1; do
echo -n "BPS=$b: "; COMET_FINISH_BPS=$b timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured" | sed "s/.*'finish': //" | cut -c1-40
done; done
