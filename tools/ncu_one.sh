#!/bin/bash
# ncu --set full of one SpMM launch of the bench workload. Usage: bash tools/ncu_one.sh <layout> <tag>
L=${1:-tc}; TAG=${2:-$L}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_spmm -s 3 -c 1 -o gpurun_out/prof_$TAG -f \
  python bench.py --steps 1 --warmup 3 --layout $L --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
