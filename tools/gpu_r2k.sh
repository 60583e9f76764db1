#!/bin/bash
# Same-box A/B of fragment layout v1 (build/ab/libcim_v1.so, the previous commit) vs v2 (in-tree library).
set -u
O=gpurun_out/r2k; mkdir -p $O
for rep in 1 2 3; do
  CIM_B200_LIB=build/ab/libcim_v1.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/v1_$rep.json 2> $O/v1_$rep.err
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/v2_$rep.json 2> $O/v2_$rep.err
done
CIM_B200_LIB=build/ab/libcim_v1.so timeout 300 python bench.py --steps 10 --warmup 3 --k 16 --no-cpu-baseline --e2e-steps 1 > $O/v1_k16.json 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 --k 16 --no-cpu-baseline --e2e-steps 1 > $O/v2_k16.json 2>/dev/null
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks']['reasons'])"; done
