#!/bin/bash
# ncu of the symmetric CSR walk at k = 8 and k = 16 (lanes sharing an entry's X row) on basis n = 262,144.
set -u
O=gpurun_out/s4m; mkdir -p $O
for k in 8 16; do
timeout 900 ncu --set full --clock-control none -k regex:csr_sym -s 2 -c 1 -o $O/prof_csr_sym_k$k -f \
  python tools/bench_basis_spmm.py --n 262144 --bias 0.05 --reps 3 --k $k > $O/ncu$k.log 2>&1; tail -1 $O/ncu$k.log
done
