#!/bin/bash
# BASELINE config C4: vector-count sweep on the C2 matrix, f32 and f64, 1 GPU.
mkdir -p gpurun_out
: > gpurun_out/k_sweep.jsonl
for DT in f32 f64; do
  for K in 1 4 8 16 32; do
    timeout 300 python bench.py --steps 20 --warmup 3 --k $K --dtype $DT --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/k_${DT}_${K}.json 2> gpurun_out/k_${DT}_${K}.err && cat gpurun_out/k_${DT}_${K}.json >> gpurun_out/k_sweep.jsonl
    python -c "import json;d=json.load(open('gpurun_out/k_${DT}_${K}.json'));print('$DT k=$K', round(d['ms_per_step'],3),'ms', round(d['value']),'GFLOP/s', round(d['roofline']['achieved']),'GB/s', d['clocks']['reasons'])" || tail -3 gpurun_out/k_${DT}_${K}.err
  done
done
