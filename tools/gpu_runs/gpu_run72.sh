cd $GRAFT_REPO_ROOT
for i in 1 2; do for sp in 0 8 16 24 32; do
echo -n "PH SPLIT1=$sp: "; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"
done; done
for sp in 0 16; do echo -n "MX EP4 SPLIT1=$sp: "; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --ep 4 --M 8192 --nc0 32 --g0 4 --pairs 0 2>&1 | grep -E "measured" | sed "s/.kernels_ms_hot_rank.*//"; done
