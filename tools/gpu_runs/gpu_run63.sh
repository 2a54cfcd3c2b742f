cd $GRAFT_REPO_ROOT
for sp in 0 28 56 74; do
echo "== SPLIT1=$sp QW EP8"; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span|EPI" | sed "s/.kernels_ms_max.*//"
done
for sp in 0 16; do
echo "== SPLIT1=$sp PH"; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape PH --ep 4 --tp 2 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
echo "== SPLIT1=$sp QW std"; COMET_SPLIT1=$sp timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --std 0.032 --nc0 64 --g0 4 --pairs 0 2>&1 | grep -E "measured|span" | sed "s/.kernels_ms_max.*//"
done
