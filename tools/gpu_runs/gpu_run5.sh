cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for g in 1 2 4; do for nc in 16 32; do echo "== g0=$g nc0=$nc"; timeout 300 python tools/fused_timeline.py --nc0 $nc --g0 $g --pairs 0 2>&1 | grep -E "measured|MMA|pair end|dispatch"; done; done
timeout 300 python tools/fused_timeline.py --nc0 32 --g0 1 --pairs 6 2>&1 | grep "cta" | head -12
