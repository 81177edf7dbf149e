timeout 60 python tools/prof_multiply.py --iters 3
timeout 60 python tools/prof_multiply.py --iters 3 --form scatter --dtype float32
timeout 60 python tools/prof_multiply.py --iters 3 --form gather --dtype float32
