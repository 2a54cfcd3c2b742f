run() { echo "== $*"; env "$@" timeout -s KILL 60 python tools/prof_layer.py --iters 5 2>&1 | grep -v cuBLAS; }
run COMET_DEBUG=1
run COMET_DEBUG=1 COMET_L2PROMO=0
run COMET_DEBUG=1 COMET_L2PROMO=2
run COMET_DEBUG=1 COMET_GRID=128
run COMET_DEBUG=1 COMET_GRID=96
run COMET_DEBUG=1 COMET_GRID=64
run COMET_DEBUG=1 COMET_GRID=32
