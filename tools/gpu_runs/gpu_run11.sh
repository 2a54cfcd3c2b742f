cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for f in 0 1; do for g1 in 4 8; do echo "== EP1 fused=$f g1=$g1"; COMET_FUSED=$f COMET_G1=$g1 timeout 300 python tools/fused_timeline.py --ep 1 --nc0 0 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed 's/.kernels_ms_max.*//'; done; done
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 900 python tools/matrix.py --quick --out gpurun_out/matrix_q.jsonl > /dev/null 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/matrix_q.jsonl'):
    r=json.loads(l); print(r['shape'],r['ep'],r['tp'],r['M'],r['std'],r['latency_ms'],r['kernels_ms_hot_rank'],r['pct_roofline_burst'],r.get('unfused_ms'),r['n_comm0'])
PY
