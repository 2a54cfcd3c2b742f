cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log; grep -E "^E " gpurun_out/pytest_gpu.log | head -5
for cfg in "MX 8 1 64 0" "PH 4 2 64 0" "QW 8 1 64 0" "QW 8 1 64 0.032"; do set -- $cfg
echo -n "$1 ep$2 tp$3 std$5: "; timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --std $5 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done
