#!/bin/bash
# DMMA permuted k-slots (PERM=1: k = 32; PERM=2: k = 16 and 32; PERM=0: off), parity and kernel ms.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s4h; mkdir -p $O
for v in perm1 dperm2; do
  if [ $v = perm1 ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -m gpu -k "float64 or f64 or tc64" -x --timeout 300 > $O/pytest_$v.txt 2>&1; echo "$v pytest exit $? $(tail -1 $O/pytest_$v.txt)"
done
for rep in 1 2; do for v in perm1 dperm0 dperm2; do
  if [ $v = perm1 ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
  for k in 16 32; do
  timeout 300 python bench.py --dtype f64 --k $k --layout tc --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$v f64 k=$k', round(d['roofline']['kernel_ms'],3), d['clocks']['reasons'])"
  done
done; done
