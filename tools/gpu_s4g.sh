#!/bin/bash
# C1 (n = 65,536, L2 flushed per step): three-ring vs two-ring FFMA2 kernel vs the tcgen05 kernel.
set -u
O=gpurun_out/s4g; mkdir -p $O
for rep in 1 2; do for v in r3 r2 tc; do
  unset CIM_K8_RINGS; L=""
  case $v in r2) export CIM_K8_RINGS=2;; tc) L="--layout tc";; esac
  timeout 300 python bench.py --n 65536 --tiles-per-gpu 6268 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 $L > $O/c1.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/c1.json').read().strip().splitlines()[-1]);print('$v C1 kernel us', round(1e3*d['roofline']['kernel_ms'],1), 'frac', round(d['roofline']['frac'],3))"
done; done
