#!/bin/bash
# ncu (with source) of the staged sparse kernel at 5% fill (C2 tile pattern, all tiles staged).
set -u
O=gpurun_out/s4b; mkdir -p $O
timeout 300 python bench.py --fill 0.05 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('fill 0.05', round(d['roofline']['kernel_ms'],3), d['roofline']['frac'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sparse_spmm_kernel -s 1 -c 1 -o $O/prof_staged5 -f \
  python bench.py --fill 0.05 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu.log 2>&1; tail -1 $O/ncu.log
