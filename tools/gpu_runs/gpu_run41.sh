cd $GRAFT_REPO_ROOT
for L in 0 3; do echo "== ILV=$L DL=8"; COMET_ZC_DL=8 COMET_ZC_ILV=$L MODE=zc NC0=16 timeout 120 python tools/stream_probe.py 2>&1 | tail -10; done
