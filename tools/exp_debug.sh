python tools/prof_multiply.py --iters 3
python tools/prof_multiply.py --iters 3 --variant rsr
for c in llama4096 llama4096x14336 llama14336x4096; do python tools/prof_multiply.py --iters 3 --config $c; done
