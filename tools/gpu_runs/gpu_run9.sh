cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for g in 1 2 4; do for sp in 0 16 32; do for s0 in 0 1; do echo "== g0=$g split1=$sp split0=$s0"; COMET_SPLIT0=$s0 COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --nc0 64 --g0 $g --pairs 0 2>&1 | grep -E "measured|span|pair end" | sed 's/.kernels_ms_max.*//'; done; done; done
