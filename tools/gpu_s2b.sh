#!/bin/bash
# Full -m gpu suite on the restored tree + ncu full captures of the C4 compute-bound widths.
set -u
O=gpurun_out/s2b; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
for cfg in "f64 8" "f64 16" "f32 16"; do set -- $cfg
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_spmm -s 3 -c 1 -o $O/prof_$1_k$2 -f \
  python bench.py --steps 1 --warmup 3 --dtype $1 --k $2 --no-cpu-baseline --e2e-steps 1 > $O/ncu_$1_k$2.log 2>&1
tail -2 $O/ncu_$1_k$2.log
done
