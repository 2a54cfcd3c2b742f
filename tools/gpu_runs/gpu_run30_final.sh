cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-unfused > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"moe_layer|index_build|dispatch_local|combine_local" -c 4 \
   -o gpurun_out/prof_fused -f python tools/prof_layer.py --once > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 1800 python tools/matrix.py > gpurun_out/matrix.log 2>&1; echo "matrix rc=$?"
timeout 600 python -m paper_2502_19811_b200.cli compare --ep 8 --tokens 8192 --modes fine,sequential,coarse:2 --out-dir gpurun_out/cli_ep8 > gpurun_out/cli.log 2>&1
timeout 600 python -m paper_2502_19811_b200.cli compare --ep 1 --tokens 8192 --modes fine,sequential,unfused --out-dir gpurun_out/cli_ep1 >> gpurun_out/cli.log 2>&1
timeout 600 python -m paper_2502_19811_b200.cli run --ep 8 --tokens 8192 --out-dir gpurun_out/cli_run_ep8 >> gpurun_out/cli.log 2>&1
tail -12 gpurun_out/cli.log
