cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/r1_layer_final python tools/prof_layer.py --once > gpurun_out/ncu_final.log 2>&1
tail -2 gpurun_out/ncu_final.log
python tools/ncu_summary.py gpurun_out/r1_layer_final.ncu-rep gpurun_out/ncu_layer_summary.json index,dispatch_local,layers,combine_local 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-unfused > /dev/null 2>&1; wc -l gpurun_out/launches.csv
