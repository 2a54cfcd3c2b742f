cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for g in 4 8; do
for cfg in "2 32" "4 32" "8 64"; do set -- $cfg
echo -n "g0=$g MX ep$1: "; timeout 300 python tools/fused_timeline.py --ep $1 --M 8192 --nc0 $2 --g0 $g --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done; done
