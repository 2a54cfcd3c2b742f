cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -k "split_k or modes or narrow" 2>&1 | tail -2
for M in 1024 2048 4096; do for ks in 0 2 4 8; do echo "== EP8 M=$M ksplit=$ks"; COMET_KSPLIT=$ks timeout 300 python tools/fused_timeline.py --M $M --nc0 64 --pairs 2 2>&1 | grep -E "measured|cta   [02]:" | sed 's/.kernels_ms_max.*//'; done; done
