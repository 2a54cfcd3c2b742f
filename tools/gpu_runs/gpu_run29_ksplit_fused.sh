cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
for kf in 0 1; do
echo "== KSPLIT_FUSED=$kf MX EP8"; COMET_KSPLIT_FUSED=$kf timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|pair end|EPI" | sed "s/.kernels_ms_max.*//"
echo "== KSPLIT_FUSED=$kf MX EP4"; COMET_KSPLIT_FUSED=$kf timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
echo "== KSPLIT_FUSED=$kf MX EP8 std.05"; COMET_KSPLIT_FUSED=$kf timeout 300 python tools/fused_timeline.py --ep 8 --std 0.05 --M 8192 --nc0 16 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
done
