# matrix + launch list + ncu full capture at HEAD
cd $GRAFT_REPO_ROOT
timeout 1500 python tools/matrix.py > gpurun_out/matrix.log 2>&1; echo "matrix rc=$?" >> gpurun_out/matrix.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-unfused > gpurun_out/launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"moe_layer|index_build|dispatch_local|combine_local" -c 8 \
   -o gpurun_out/prof_layer -f python tools/prof_layer.py --once > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/matrix.log; tail -3 gpurun_out/ncu_full.log
