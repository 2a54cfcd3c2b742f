cd $GRAFT_REPO_ROOT
timeout 1500 python tools/matrix.py --out gpurun_out/matrix.jsonl > gpurun_out/matrix.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/matrix.log; wc -l gpurun_out/matrix.jsonl
