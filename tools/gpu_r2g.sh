#!/bin/bash
# A/B: f32 k = 16/24/32/64 as paired passes on the three-ring kernel (default) vs the old kernels (CIM_K8_PAIRED=0).
set -u
O=gpurun_out/r2g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x -k "k_sweep_f32 or multipass or host_batch or chunked" > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
for k in 16 32 24 64; do
for paired in 1 0; do
  CIM_K8_PAIRED=$paired timeout 300 python bench.py --steps 10 --warmup 3 --k $k --no-cpu-baseline --e2e-steps 1 > $O/k${k}_p${paired}.json 2> $O/k${k}_p${paired}.err
done
done
tail -2 $O/pytest.txt
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'GFLOP/s', round(d['value']), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks']['reasons'])" || tail -2 ${f%.json}.err; done
