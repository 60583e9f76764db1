#!/bin/bash
# BASELINE config C4: vector-count sweep on the C2 matrix, f32 and f64, 1 GPU.
# f32 runs every width on both tile layouts (frag = FFMA2 kernel, tc = split-TF32
# tensor-core kernel, k a multiple of 8); the library's guidance is
# the faster one per width.
mkdir -p gpurun_out
: > gpurun_out/k_sweep.jsonl
run() {  # DT K LAYOUT
  timeout 300 python bench.py --steps 20 --warmup 3 --k $2 --dtype $1 --layout $3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/k_$1_$2_$3.json 2> gpurun_out/k_$1_$2_$3.err && cat gpurun_out/k_$1_$2_$3.json >> gpurun_out/k_sweep.jsonl
  python -c "import json;d=json.load(open('gpurun_out/k_$1_$2_$3.json'));print('$1 k=$2 $3', round(d['ms_per_step'],3),'ms', round(d['value']),'GFLOP/s', round(d['roofline']['achieved']),'GB/s', d['clocks']['reasons'])" || tail -3 gpurun_out/k_$1_$2_$3.err
}
for K in 1 4 8 16 32 64; do run f32 $K frag; done
for K in 8 16 32 64; do run f32 $K tc; done
for K in 1 4 8 16 32; do run f64 $K frag; done
for K in 8 16 24 32; do run f64 $K tc; done
