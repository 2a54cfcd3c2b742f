cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_layer -s 16 -c 1 -o gpurun_out/prof_ep8 -f python tools/ep_ncu.py 8 > gpurun_out/ncu_ep8.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_ep8.log
python tools/ncu_summary.py gpurun_out/prof_ep8.ncu-rep gpurun_out/ncu_ep8_layer_summary.json layers_ep8_rank0 2>&1 | tail -16
