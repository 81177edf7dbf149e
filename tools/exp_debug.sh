python tools/prof_multiply.py --iters 3
RSR_B200_PDL=0 python tools/prof_multiply.py --iters 3
