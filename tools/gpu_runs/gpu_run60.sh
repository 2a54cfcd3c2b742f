cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -m gpu 2>&1 | tail -2
for dbg in 256 0; do
echo "== DEBUG=$dbg QW EP8"; COMET_DEBUG=$dbg TAIL=3 timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI|tail" | sed "s/.kernels_ms_max.*//"
echo "== DEBUG=$dbg MX EP8"; COMET_DEBUG=$dbg timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
echo "== DEBUG=$dbg PH"; COMET_DEBUG=$dbg timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
done
