cd $GRAFT_REPO_ROOT
for f in 0 1; do echo "== fused=$f"; COMET_FUSED=$f timeout 300 python tools/fused_timeline.py --ep 1 --M 2048 --nc0 0 --g0 4 --pairs 4 2>&1 | tail -16; done
