#!/bin/bash
# ncu --set full of the two tensor-core kernels at k = 16 (f32 tcgen05, f64 DMMA) and their launch lists.
set -u
O=gpurun_out/s2n; mkdir -p $O
for cfg in "f32 16 tc" "f64 16 dmma"; do set -- $cfg
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_spmm_$3 -s 3 -c 1 -o $O/prof_$3_$1_k$2 -f \
  python bench.py --dtype $1 --layout tc --k $2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_$3.log 2>&1
tail -1 $O/ncu_$3.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches_$3_$1_k$2.csv \
  python bench.py --dtype $1 --layout tc --k $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
