#!/bin/bash
# ncu --set full of the split-TF32 kernel at k = 16 and 64 (source page for the stall hotspots).
set -u
O=gpurun_out/s2d; mkdir -p $O
for k in 16 64; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_spmm_tc -s 3 -c 1 -o $O/prof_tc_k$k -f \
  python bench.py --layout tc --k $k --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_tc_k$k.log 2>&1
tail -1 $O/ncu_tc_k$k.log
ncu -i $O/prof_tc_k$k.ncu-rep --page source --csv --print-source sass > $O/src_tc_k$k.csv 2>/dev/null
done
