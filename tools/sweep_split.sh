#!/bin/bash
# Tuning sweep of the vector split (KV x NG) for the default bench workload.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_quick.txt 2>&1; tail -2 gpurun_out/pytest_quick.txt
for s in ${SPLITS:-8x1 4x2}; do
  CIM_SPLIT=$s timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/split_$s.json 2> gpurun_out/split_$s.err
  python -c "import json;d=json.load(open('gpurun_out/split_$s.json'));print('$s', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],4), d['clocks'])"
done
