#!/bin/bash
# compute-sanitizer memcheck over the tensor-core kernels' tests (f32 tcgen05, f64 DMMA; bulk reductions).
set -u
O=gpurun_out/s2r; mkdir -p $O
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" --timeout 2400 > $O/memcheck_tc.txt 2>&1
echo "memcheck tc exit $?" >> $O/memcheck_tc.txt
tail -4 $O/memcheck_tc.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python bench.py --dtype f64 --layout tc --k 16 --tiles-per-gpu 150000 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/memcheck_dmma_bench.txt 2>&1
echo "memcheck dmma bench exit $?" >> $O/memcheck_dmma_bench.txt
grep -E "ERROR SUMMARY|exit" $O/memcheck_dmma_bench.txt
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python bench.py --layout tc --k 32 --tiles-per-gpu 150000 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/memcheck_tc_bench.txt 2>&1
echo "memcheck tc bench exit $?" >> $O/memcheck_tc_bench.txt
grep -E "ERROR SUMMARY|exit" $O/memcheck_tc_bench.txt
