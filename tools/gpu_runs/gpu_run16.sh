cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for M in 1024 2048 4096 8192; do for ks in 0 8; do echo "== EP8 M=$M ksplit=$ks"; COMET_KSPLIT=$ks timeout 300 python tools/fused_timeline.py --M $M --nc0 64 --pairs 0 2>&1 | grep -E "measured" | sed 's/.kernels_ms_max.*//'; done; done
for ks in 0 8; do echo "== EP1 M=1024 ksplit=$ks"; COMET_KSPLIT=$ks timeout 300 python tools/fused_timeline.py --ep 1 --M 1024 --nc0 0 --g0 8 --pairs 0 2>&1 | grep -E "measured" | sed 's/.kernels_ms_max.*//'; done
timeout 800 python tools/fit_costmodel.py 2>&1 | tail -13
