cd $GRAFT_REPO_ROOT
for cfg in "16 8" "16 4" "16 12" "12 8" "24 8" "20 8" "16 8"; do set -- $cfg
echo -n "NC0=$1 DL=$2: "; G0=16 NC0=$1 COMET_ZC_DL=$2 MODE=zc timeout 120 python tools/stream_probe.py 2>&1 | grep "per forward"; done
