cd $GRAFT_REPO_ROOT
for g in 1 2 4; do echo "== MX EP8 g0=$g"; timeout 300 python tools/fused_timeline.py --M 8192 --nc0 64 --g0 $g --pairs 0 2>&1 | grep -E "measured|span|pair end|dispatch" | sed "s/.kernels_ms_max.*//"; done
for nc in 32 64 96; do echo "== QW EP8 nc0=$nc"; timeout 300 python tools/fused_timeline.py --shape QW --M 8192 --nc0 $nc --g0 4 --pairs 3 2>&1 | grep -E "measured|span|pair end|dispatch|MMA|EPI|cta|lifetime" | sed "s/.kernels_ms_max.*//"; done
