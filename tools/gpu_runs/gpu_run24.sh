cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
echo "== QW EP8"; timeout 300 python tools/fused_timeline.py --shape QW --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|pair end|EPI" | sed "s/.kernels_ms_max.*//"
echo "== MX EP4"; timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
echo "== MX EP8"; timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
echo "== PH"; timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
for f in 0 1; do echo "== EP1 FUSE1=$f"; COMET_FUSE1=$f timeout 300 python tools/fused_timeline.py --ep 1 --nc0 0 --g0 8 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_max.*//"; done
timeout 300 python tools/stream_probe.py 2>&1 | tail -9
