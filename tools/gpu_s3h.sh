#!/bin/bash
# Evidence refresh: ncu of the symmetric small-tile CSR on a basis skeleton; C3 on one GPU; C5 LOBPCG; C1.
set -u
O=gpurun_out/s3h; mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:csr_spmm -s 2 -c 1 -o $O/prof_csr_sym -f \
  python tools/bench_basis_spmm.py --n 262144 --bias 0.05 --reps 3 > $O/ncu_csr.log 2>&1
tail -1 $O/ncu_csr.log
timeout 600 python bench.py --tiles-per-gpu 3906250 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c3.json 2>/dev/null
timeout 300 python tools/bench_lobpcg.py > $O/lobpcg.json 2>/dev/null
timeout 300 python bench.py --n 65536 --tiles-per-gpu 6268 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 4 > $O/c1.json 2>/dev/null
for f in c3 c1; do python -c "
import json;d=json.load(open('$O/$f.json'));r=d['roofline'];print('$f', round(r['kernel_ms'],4), round(r['frac'],3), d['clocks']['reasons'])"; done
tail -2 $O/lobpcg.json | cut -c1-300
