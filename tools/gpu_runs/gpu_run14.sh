cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for g in 2 4 8 16; do for w in 2 4 8; do echo "== EP1 g0=$g wave1=$w"; timeout 300 python tools/fused_timeline.py --ep 1 --nc0 0 --g0 $g --wave1 $w --pairs 0 2>&1 | grep -E "measured" | sed 's/.kernels_ms_max.*//'; done; done
echo "== PH"; timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --nc0 64 --pairs 0 2>&1 | grep -E "measured" | sed 's/.kernels_ms_max.*//'
