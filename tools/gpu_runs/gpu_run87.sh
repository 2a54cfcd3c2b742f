cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x -m gpu 2>&1 | tail -2
for i in 1 2; do
for cfg in "MX 8 1 64" "MX 1 1 0" "PH 4 2 64" "QW 8 1 64"; do set -- $cfg
echo -n "$1 ep$2 tp$3: "; timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured|MMA L0" | sed "s/.kernels_ms_hot_rank.*//" | tr '\n' ' '; echo
done; done
