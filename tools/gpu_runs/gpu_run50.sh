cd $GRAFT_REPO_ROOT
for nc in 16 32 64; do for g in 2 4 8; do
echo "== MX EP8 nc0=$nc g0=$g"; timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 $nc --g0 $g --pairs 0 2>&1 | grep -E "measured|EPI L0|span" | sed "s/.kernels_ms_max.*//" | sed "s/'kernels_ms_hot_rank'//"
done; done
