cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -m gpu 2>&1 | tail -2
for i in 1 2; do
echo "== QW EP8"; TAIL=2 timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI|tail" | sed "s/.kernels_ms_max.*//"
echo "== MX EP8"; timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
echo "== PH"; timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
done
