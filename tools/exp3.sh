for d in 0 64 128 16 80 144 8 72 136; do echo "== COMET_DEBUG=$d"; COMET_DEBUG=$d timeout -s KILL 60 python tools/prof_layer.py --iters 10 2>&1 | grep -v cuBLAS; done
