#!/bin/bash
# Staged sparse kernel: lane-dependent half order of the 32-byte X gathers vs the previous build.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -m gpu -k "sparse or csr or basis or fill" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for v in swap noswap; do
  if [ $v = swap ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/sp_noswap/libcim_b200.so; fi
  for f in 0.05 0.09 0.17; do
  timeout 300 python bench.py --fill $f --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$v fill $f', round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))"
  done
  timeout 300 python bench.py --fill 0.05 --dtype f64 --k 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$v fill 0.05 f64 k4', round(d['roofline']['kernel_ms'],3))"
done; done
