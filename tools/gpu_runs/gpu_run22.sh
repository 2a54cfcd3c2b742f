cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
echo "== QW EP8"; timeout 300 python tools/fused_timeline.py --shape QW --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|pair end|EPI" | sed "s/.kernels_ms_max.*//"
echo "== MX EP4"; timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|pair end|EPI" | sed "s/.kernels_ms_max.*//"
echo "== MX EP8"; timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|pair end|EPI" | sed "s/.kernels_ms_max.*//"
