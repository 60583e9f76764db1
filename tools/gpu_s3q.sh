#!/bin/bash
# ncu of the LOBPCG Gram kernel (the masked S^T[S AS] pass) on C2 rows.
set -u
O=gpurun_out/s3q; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_partial -s 12 -c 2 -o $O/prof_gram -f \
  python tools/bench_lobpcg.py --iters 3 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
