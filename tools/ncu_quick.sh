#!/bin/bash
# ncu --set full of one launch of kernel regex $1 under command "${@:2}" -> gpurun_out/$1.ncu-rep
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 -s 1 -c 1 -o gpurun_out/$1 -f "${@:2}" > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"
