cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for nc in 8 16 32; do timeout 300 python tools/fused_timeline.py --nc0 $nc --pairs 3 2>&1 | grep -v "^  cta" | tail -14; done
timeout 300 python tools/fused_timeline.py --nc0 16 --pairs 8 2>&1 | grep "cta" | head -12
