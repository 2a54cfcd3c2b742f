cd $GRAFT_REPO_ROOT
COMET_DEDUP=1 timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multiproc.py -m gpu -q -x 2>&1 | tail -3
for d in 0 1; do
echo "== DEDUP=$d QW EP8"; COMET_DEDUP=$d timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$d MX EP8"; COMET_DEDUP=$d timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$d MX EP4"; COMET_DEDUP=$d timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$d PH"; COMET_DEDUP=$d timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|dispatch" | sed "s/.kernels_ms_max.*//"
done
