#!/bin/bash
# ncu: launch list and a full capture of csr_spmm_kernel on the n=262144 basis skeleton.
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/basis_launches.csv \
  python tools/bench_basis_spmm.py --n 262144 --bias 0.05 --reps 3 > gpurun_out/basis_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_spmm -s 2 -c 1 -o gpurun_out/csr_spmm -f \
  python tools/bench_basis_spmm.py --n 262144 --bias 0.05 --reps 3 > gpurun_out/csr_ncu.log 2>&1
tail -3 gpurun_out/csr_ncu.log
