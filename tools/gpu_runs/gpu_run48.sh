cd $GRAFT_REPO_ROOT
for cfg in "8 3" "4 1" "4 2" "4 4" "2 1" "2 2" "2 4" "16 1"; do set -- $cfg
echo "== G0=$1 ILV=$2"; G0=$1 COMET_ZC_ILV=$2 MODE=zc NC0=16 timeout 120 python tools/stream_probe.py 2>&1 | tail -10 | grep -E "per forward|layer|CTA exits"; done
