cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for a in 1 0; do
for cfg in "MX 2 1 32" "MX 4 1 32" "PH 4 2 64"; do set -- $cfg
echo -n "AUTO=$a $1 ep$2: "; COMET_SPLIT1_AUTO=$a timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done; done
