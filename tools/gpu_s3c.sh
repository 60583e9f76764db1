#!/bin/bash
# Sustained (100-step) C2 k=8: FFMA2 (frag) vs tcgen05 (tc) on the same box, alternating; power and clocks.
set -u
O=gpurun_out/s3c; mkdir -p $O
for rep in 1 2; do for L in frag tc; do
timeout 300 python bench.py --layout $L --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/$L.$rep.json 2>/dev/null
python -c "
import json;d=json.load(open('$O/$L.$rep.json'));r=d['roofline'];c=d['clocks'];print('$L 100 steps', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac'],4), c['sm_mhz'], c.get('power_w_median'), c['reasons'])"
done; done
