cd $GRAFT_REPO_ROOT
COMET_KSPLIT1_FORCE=2 timeout 300 python tools/fused_timeline.py --ep 8 --M 8192 --nc0 64 --g0 4 --pairs 0 2>&1 | tail -8
