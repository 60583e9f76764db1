#!/bin/bash
# A/B: f64 k = 8/16/32 as paired 4-vector passes on the three-ring kernel vs the two-ring kernels.
set -u
O=gpurun_out/r2h; mkdir -p $O
CIM_K8_PAIRED_F64=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x -k "k_sweep_f64 or multipass or host_batch" > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
for k in 8 16 32 12; do
for pf in 1 0; do
  CIM_K8_PAIRED_F64=$pf timeout 300 python bench.py --steps 10 --warmup 3 --k $k --dtype f64 --no-cpu-baseline --e2e-steps 1 > $O/k${k}_pf${pf}.json 2> $O/k${k}_pf${pf}.err
done
done
tail -2 $O/pytest.txt
for f in $O/*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'GFLOP/s', round(d['value']), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks']['reasons'])" || tail -2 ${f%.json}.err; done
