cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
for dd in 0 1; do
echo "== DEDUP=$dd QW"; COMET_DEDUP=$dd timeout 300 python tools/fused_timeline.py --shape QW --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$dd PH"; COMET_DEDUP=$dd timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$dd MX EP4"; COMET_DEDUP=$dd timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|dispatch" | sed "s/.kernels_ms_max.*//"
echo "== DEDUP=$dd MX EP8"; COMET_DEDUP=$dd timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|dispatch" | sed "s/.kernels_ms_max.*//"
done
