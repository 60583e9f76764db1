#!/bin/bash
# memcheck of this session's new kernels: symmetric CSR walk (SUB lanes), fused Ritz update,
# DMMA with the TMA X stage, plus a 150k-tile f64 k=16/32 apply.
set -u
O=gpurun_out/s4d; mkdir -p $O
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -m gpu \
  -k "small_tiles_csr or basis_65k or basis_skeleton or ritz or (tc and float64) or k_sweep_f64" --timeout 2000 > $O/memcheck_s4.txt 2>&1
echo "memcheck exit $?" >> $O/memcheck_s4.txt
tail -4 $O/memcheck_s4.txt
for k in 16 32; do
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 python bench.py --dtype f64 --k $k --layout tc \
  --tiles-per-gpu 150000 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/mc_dmma$k.txt 2>&1; echo "dmma k=$k memcheck exit $?" | tee -a $O/mc_dmma$k.txt
grep "ERROR SUMMARY" $O/mc_dmma$k.txt
done
