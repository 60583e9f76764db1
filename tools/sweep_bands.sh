#!/bin/bash
# Column-band sweep of the tile order on the default bench workload.
mkdir -p gpurun_out
for b in ${BANDS:-1 2 4 8 1}; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 --bands $b > gpurun_out/bands_$b.json 2> gpurun_out/bands_$b.err
  python -c "import json;d=json.load(open('gpurun_out/bands_$b.json'));print('bands $b', round(d['roofline']['kernel_ms'],4), 'ms', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/bands_$b.err
done
