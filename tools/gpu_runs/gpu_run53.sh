cd $GRAFT_REPO_ROOT
COMET_W1_PULL=16 COMET_DEDUP=1 timeout 300 python -m pytest tests/test_gpu_layer.py -q -x -m gpu -k "full_size or modes" 2>&1 | tail -2
for cfg in "0 0" "8 0" "16 0" "16 1" "32 1"; do set -- $cfg
echo "== W1_PULL=$1 DEDUP=$2"; COMET_W1_PULL=$1 COMET_DEDUP=$2 timeout 300 python tools/fused_timeline.py --ep 1 --M 8192 --nc0 64 --g0 8 --pairs 0 2>&1 | grep -E "measured|span|CTA lifetime|dispatch" | sed "s/.kernels_ms_max.*//"
done
