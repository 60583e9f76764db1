#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/k_sweep_tc.jsonl
for K in 8 16 32; do
  timeout 300 python bench.py --steps 20 --warmup 3 --k $K --layout tc --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/ktc_$K.json 2> gpurun_out/ktc_$K.err && cat gpurun_out/ktc_$K.json >> gpurun_out/k_sweep_tc.jsonl
  python -c "import json;d=json.load(open('gpurun_out/ktc_$K.json'));print('tc f32 k=$K', round(d['ms_per_step'],3),'ms', round(d['value']),'GFLOP/s', d['clocks']['reasons'])" || tail -3 gpurun_out/ktc_$K.err
done
timeout 600 python -m pytest tests/test_lobpcg.py -q -m gpu 2>&1 | tail -3
