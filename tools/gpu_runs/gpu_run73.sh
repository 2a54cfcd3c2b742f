cd $GRAFT_REPO_ROOT
for i in 1 2; do for sp in 0 8 16; do
for cfg in "MX 1 1 0" "MX 2 1 16" "MX 4 1 32" "MX 8 1 64"; do set -- $cfg
echo -n "$1 ep$2 SPLIT1=$sp: "; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done; done
