#!/bin/bash
# Bring-up check of the tensor-core path: one guarded test first, then the rest.
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_config and tc" > gpurun_out/tc_first.txt 2>&1; echo "first exit $?" >> gpurun_out/tc_first.txt
tail -15 gpurun_out/tc_first.txt
if grep -q "1 passed" gpurun_out/tc_first.txt; then
  timeout 900 python -m pytest tests -q -m gpu --timeout 120 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
  tail -25 gpurun_out/pytest_gpu.txt
  for L in tc frag; do
    timeout 300 python bench.py --steps 50 --warmup 5 --layout $L --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$L.json 2> gpurun_out/bench_$L.err
    python -c "import json;d=json.load(open('gpurun_out/bench_$L.json'));print('$L', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],4), d['clocks'])" || tail -5 gpurun_out/bench_$L.err
  done
fi
timeout 300 python tools/tc_profile.py 2>&1 | tail -4
