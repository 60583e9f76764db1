#!/bin/bash
# Column bands on the split-TF32 kernel at k = 16 / 32, plus the ncu DRAM bytes at k = 16.
set -u
O=gpurun_out/s2i; mkdir -p $O
for k in 16 32; do for B in 1 2 4; do
timeout 120 python bench.py --layout tc --k $k --bands $B --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/tc_k${k}_b$B.json 2> $O/tc_k${k}_b$B.err
python -c "
import json;d=json.load(open('$O/tc_k${k}_b$B.json'));r=d['roofline'];print('tc k=$k bands=$B', round(r['kernel_ms'],3))" 2>/dev/null || tail -3 $O/tc_k${k}_b$B.err
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sym_spmm_tc -c 2 --csv \
  python bench.py --layout tc --k 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_k16.csv 2> $O/ncu_k16.err
grep -E "dram__bytes|gpu__time|hit_rate" $O/ncu_k16.csv | tail -4
