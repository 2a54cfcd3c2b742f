cd $GRAFT_REPO_ROOT
for sp in 0 37 74; do
echo "== SPLIT1=$sp"
for cfg in "MX 1 1 0" "MX 2 1 16" "MX 4 1 32" "MX 8 1 64" "PH 4 2 64" "QW 8 1 64"; do set -- $cfg
echo -n "$1 ep$2 tp$3: "; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape $1 --ep $2 --tp $3 --M 8192 --nc0 $4 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done
