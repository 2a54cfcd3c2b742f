cd $GRAFT_REPO_ROOT
for i in 1 2; do
for cfg in "2 16" "2 64" "4 32" "4 64"; do set -- $cfg
echo -n "MX ep$1 nc0=$2: "; timeout 300 python tools/fused_timeline.py --ep $1 --M 8192 --nc0 $2 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done
