cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python tools/matrix.py --quick --out gpurun_out/matrix_fused.jsonl > gpurun_out/matrix_fused.log 2>&1; echo "matrix rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/matrix_fused.jsonl'):
    r=json.loads(l); print(r['shape'],r['ep'],r['tp'],r['M'],r['std'],r['latency_ms'],r['kernels_ms_hot_rank'],r['pct_roofline_burst'],r.get('unfused_ms'),r['n_comm0'])
PY
