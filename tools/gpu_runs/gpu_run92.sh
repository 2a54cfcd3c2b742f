cd $GRAFT_REPO_ROOT
timeout 600 python -m paper_2502_19811_b200.cli compare --ep 8 --tokens 8192 --modes fine,sequential,coarse:2 --out-dir gpurun_out/cli_ep8 > gpurun_out/cli.log 2>&1
timeout 600 python -m paper_2502_19811_b200.cli compare --ep 1 --tokens 8192 --modes fine,sequential,unfused --out-dir gpurun_out/cli_ep1 >> gpurun_out/cli.log 2>&1
timeout 600 python -m paper_2502_19811_b200.cli run --ep 8 --tokens 8192 --out-dir gpurun_out/cli_run_ep8 >> gpurun_out/cli.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/cli.log; ls gpurun_out/cli_ep8 gpurun_out/cli_ep1 gpurun_out/cli_run_ep8
