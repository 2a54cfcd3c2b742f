cd $GRAFT_REPO_ROOT
for fo in 1 0; do echo "== FOLD_ORDER=$fo QW EP8"; COMET_FOLD_ORDER=$fo TAIL=30 timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI|tail"; done
