#!/bin/bash
# A/B: three-ring wide kernel (default) vs the two-ring kernel (CIM_K8_RINGS=2), C2 k=8 f32 / k=4 f64; parity tests.
set -u
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x > $O/pytest_parity.txt 2>&1; echo "pytest exit $?" >> $O/pytest_parity.txt
for rep in 1 2; do
for rings in 3 2; do
  CIM_K8_RINGS=$rings timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/c2_r${rings}_$rep.json 2> $O/c2_r${rings}_$rep.err
  CIM_K8_RINGS=$rings timeout 300 python bench.py --steps 20 --warmup 3 --k 4 --dtype f64 --no-cpu-baseline --e2e-steps 1 > $O/f64k4_r${rings}_$rep.json 2>/dev/null
done
done
CIM_K8_RINGS=3 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/c2_r3_100.json 2>/dev/null
tail -2 $O/pytest_parity.txt
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks']['reasons'])"; done
