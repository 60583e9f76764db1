#!/bin/bash
set -u
O=gpurun_out/r2j; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -x > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/c2_$rep.json 2> $O/c2_$rep.err
  timeout 300 python bench.py --steps 10 --warmup 3 --k 16 --no-cpu-baseline --e2e-steps 1 > $O/k16_$rep.json 2> /dev/null
done
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/c2_100.json 2>/dev/null
tail -2 $O/pytest_gpu.txt
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'kern', round(d['roofline']['kernel_ms'],4), round(d['value']), d['clocks']['reasons'])"; done
