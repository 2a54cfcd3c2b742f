cd $GRAFT_REPO_ROOT
for dbg in 0 32768 65536 98304 4096; do echo -n "DEBUG=$dbg: "; COMET_DEBUG=$dbg timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|EPI L0|MMA L0" | sed "s/.kernels_ms_hot_rank.*//" | tr '\n' ' '; echo; done
