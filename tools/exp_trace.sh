for d in 15 0; do echo "== debug=$d"; RSR_B200_DEBUG=$d RSR_B200_TRACE=1 python tools/prof_multiply.py --iters 1 2>&1 | grep trace | head -15; done
