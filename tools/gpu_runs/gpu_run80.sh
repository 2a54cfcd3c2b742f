cd $GRAFT_REPO_ROOT
for dbg in 0 64 128; do echo "== DEBUG=$dbg"; COMET_DEBUG=$dbg timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|EPI|MMA" | sed "s/.kernels_ms_max.*//"; done
