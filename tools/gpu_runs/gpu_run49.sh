cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:moe_layer_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/zc_layer python tools/zc_once.py > gpurun_out/zc_ncu.log 2>&1
tail -3 gpurun_out/zc_ncu.log
ncu -i gpurun_out/zc_layer.ncu-rep --page raw --csv > gpurun_out/zc_layer_raw.csv 2>&1; wc -c gpurun_out/zc_layer_raw.csv
