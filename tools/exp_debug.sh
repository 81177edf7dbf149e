timeout 60 python tools/prof_multiply.py --iters 3
for dt in float32 int32 float64; do timeout 60 python tools/prof_multiply.py --iters 3 --form gather --dtype $dt; done
timeout 60 python tools/prof_multiply.py --iters 3 --form gather --dtype float32 --variant rsr
