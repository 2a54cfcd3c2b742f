for d in 0 64; do echo "== COMET_DEBUG=$d"; COMET_DEBUG=$d timeout -s KILL 60 python tools/prof_layer.py --iters 10 2>&1 | grep -v cuBLAS; done
timeout -s KILL 60 python tools/gpu_check.py small2 mx
