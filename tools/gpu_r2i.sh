#!/bin/bash
# A/B: paired passes on the two-ring kernel (f64 multi-pass widths), paired vs per-pass launches.
set -u
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x -k "k_sweep or multipass or host_batch or chunked" > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
for k in 16 32 12; do
for pp in 1 0; do
  CIM_K8_PAIRED=$pp timeout 300 python bench.py --steps 10 --warmup 3 --k $k --dtype f64 --no-cpu-baseline --e2e-steps 1 > $O/f64k${k}_p${pp}.json 2> $O/f64k${k}_p${pp}.err
done
done
tail -2 $O/pytest.txt
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'GFLOP/s', round(d['value']), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks']['reasons'])" || tail -2 ${f%.json}.err; done
