#!/bin/bash
# compute-sanitizer memcheck over the round-2 tests and the kernels they drive
# (three-ring / paired passes, row-CSR, drop-in contraction, scan, sharded groups).
set -u
O=gpurun_out/r2n; mkdir -p $O
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_scale_parity.py tests/test_dropin_contraction.py -q -m gpu -k "not c2_full and not c3_full and not sharded" --timeout 2400 > $O/memcheck_new.txt 2>&1
echo "memcheck new exit $?" >> $O/memcheck_new.txt
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -m gpu -k "k_sweep or multipass or chunked or host_batch or sparse" --timeout 2400 > $O/memcheck_parity.txt 2>&1
echo "memcheck parity exit $?" >> $O/memcheck_parity.txt
tail -4 $O/memcheck_new.txt; tail -4 $O/memcheck_parity.txt; grep -c "Invalid\|ERROR SUMMARY" $O/memcheck_*.txt
