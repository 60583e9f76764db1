#!/bin/bash
# DRAM bytes and time of the tc kernel at k = 8 (vs the three-ring kernel's 9.19 + 0.60 GB).
set -u
O=gpurun_out/s2v; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum --clock-control none -k regex:sym_spmm -c 2 --csv python bench.py --layout tc --k 8 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_tc_k8.csv 2>/dev/null
grep -E "sym_spmm" $O/ncu_tc_k8.csv | tail -6 | awk -F'","' '{print $(NF-2), $NF}'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k8r3 -c 2 --csv python bench.py --k 8 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_frag_k8.csv 2>/dev/null
grep -E "k8r3" $O/ncu_frag_k8.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
