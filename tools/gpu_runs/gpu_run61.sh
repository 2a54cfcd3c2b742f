cd $GRAFT_REPO_ROOT
for dbg in 0 512 1024 1536; do
echo "== DEBUG=$dbg QW EP8"; COMET_DEBUG=$dbg TAIL=2 timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI|tail" | sed "s/.kernels_ms_max.*//"
done
