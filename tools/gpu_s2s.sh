#!/bin/bash
# L2 policies of the tc kernel at k = 16 / 32: X copies (evict_last / first / normal) x Y bulk reductions (none / first / last).
set -u
O=gpurun_out/s2s; mkdir -p $O
for k in 16 32; do for xp in 0 1 2; do for yp in 0 2; do
CIM_TC_XPOL=$xp CIM_TC_YPOL=$yp timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/k${k}_x${xp}_y${yp}.json 2>/dev/null
python -c "
import json;d=json.load(open('$O/k${k}_x${xp}_y${yp}.json'));r=d['roofline'];print('k=$k xpol=$xp ypol=$yp', round(r['kernel_ms'],3))" 2>/dev/null || echo "k=$k $xp $yp failed"
done; done; done
