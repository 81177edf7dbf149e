timeout 60 python tools/prof_multiply.py --iters 3
timeout 60 python tools/prof_multiply.py --iters 3 --variant rsr
for c in llama4096 llama14336x4096; do timeout 60 python tools/prof_multiply.py --iters 3 --config $c; done
