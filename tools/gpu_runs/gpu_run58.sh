cd $GRAFT_REPO_ROOT
for d in 0 1; do echo "== DEDUP=$d QW EP8"; COMET_DEDUP=$d timeout 300 python tools/fused_timeline.py --shape QW --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 2 2>&1 | tail -22; done
