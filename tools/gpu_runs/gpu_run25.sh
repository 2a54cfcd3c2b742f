cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for pl in 0 1; do echo "== MX EP8 pull_local=$pl"; COMET_PULL_LOCAL=$pl timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|dispatch" | sed "s/.kernels_ms_max.*//"; done
echo "== MX EP4"; timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
echo "== QW EP8"; timeout 300 python tools/fused_timeline.py --shape QW --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
python tools/idx_timing.py 8 4 2>&1 | tail -3
