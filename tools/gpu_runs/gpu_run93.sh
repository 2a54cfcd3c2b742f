cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for cfg in "8 3" "16 1" "16 2" "24 1"; do set -- $cfg
echo -n "G0=$1 ILV=$2: "; G0=$1 COMET_ZC_ILV=$2 MODE=zc NC0=16 timeout 120 python tools/stream_probe.py 2>&1 | grep "per forward"; done; done
