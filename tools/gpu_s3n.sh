#!/bin/bash
# Sustained (power-capped) behaviour: power limits, then frag vs tc layout at k=8 over 300 steps, alternating.
set -u
O=gpurun_out/s3n; mkdir -p $O
nvidia-smi -q -d POWER > $O/power.txt 2>&1; grep -i "limit\|draw" $O/power.txt | head -12
for rep in 1 2; do for lay in frag tc; do
  timeout 600 python bench.py --layout $lay --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/b_$lay.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b_$lay.json').read().strip().splitlines()[-1]);c=d['clocks'];print('$lay', d['ms_per_step'], round(d['roofline']['frac'],3), c['sm_mhz'], c['reasons'], c.get('power_w_median'))"
  sleep 20
done; done
