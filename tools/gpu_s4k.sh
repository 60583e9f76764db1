#!/bin/bash
# Reference-style basis skeletons at growing n (k = 8 / 16): construction on the device + apply rates.
set -u
O=gpurun_out/s4k; mkdir -p $O
for args in "--n 262144 --bias 0.05" "--n 1048576 --bias 0.03" "--n 2097152 --bias 0.02"; do for k in 8 16; do
  timeout 900 python tools/bench_basis_spmm.py $args --k $k > $O/b.json 2>$O/b.err
  echo "$args k=$k: $(tail -1 $O/b.json | cut -c1-330)"
done; done
