#!/bin/bash
# e2e leg: 16 vs 64 host blocks through sym_spmm_host_batch; the PCIe ceiling probe.
set -u
O=gpurun_out/s4i; mkdir -p $O
timeout 120 python tools/probe_pcie.py
for rep in 1 2; do for s in 16 64 128; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps $s > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);e=d['e2e'];print('e2e_steps=$s', round(e['value']/1e3,2), 'TFLOP/s', 'kernel frac', round(d['roofline']['frac'],3))"
done; done
