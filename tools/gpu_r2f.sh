#!/bin/bash
set -u
O=gpurun_out/r2f; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_spmm_k8r3 -s 3 -c 1 -o $O/prof_r3 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
