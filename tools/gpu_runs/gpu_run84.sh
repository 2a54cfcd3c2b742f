cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
