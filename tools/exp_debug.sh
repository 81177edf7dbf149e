for c in llama4096x14336 ternary16384 llama4096; do
timeout 60 python tools/prof_multiply.py --iters 3 --config $c
RSR_B200_NOSCHED=1 timeout 60 python tools/prof_multiply.py --iters 3 --config $c | sed 's/^/nosched /'
done
