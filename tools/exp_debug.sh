for d in 0 1 2 3; do RSR_B200_DEBUG=$d python tools/prof_multiply.py --iters 3 | sed "s/^/debug=$d /"; done
python tools/prof_multiply.py --iters 3 --variant rsr | sed "s/^/rsr /"
