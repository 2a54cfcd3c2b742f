timeout -s KILL 120 python tools/prof_layer.py --sweep --iters 10
for d in 16 8; do echo "== COMET_DEBUG=$d"; COMET_DEBUG=$d timeout -s KILL 60 python tools/prof_layer.py --iters 10 2>&1 | grep -v cuBLAS; done
