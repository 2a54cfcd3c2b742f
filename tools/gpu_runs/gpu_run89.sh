cd $GRAFT_REPO_ROOT
timeout 1500 python tools/matrix.py --out gpurun_out/matrix.jsonl > gpurun_out/matrix.log 2>&1; echo "rc=$?"; wc -l gpurun_out/matrix.jsonl
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['pct_of_roofline'], d['pct_of_roofline_spec_2250tf'], d['roofline']['frac'], d.get('clocks'))"
