#!/bin/bash
# tc kernel at k = 32: three A/B stages (ND = 2 accumulators, scalar Y reductions) vs two (ND = 4, bulk).
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s3u; mkdir -p $O
for rep in 1 2; do for v in base na3; do
  if [ $v = base ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/tc_na3/libcim_b200.so; fi
  for k in 32 24; do
  timeout 300 python bench.py --k $k --layout tc --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$v k=$k', round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])"
  done
done; done
export CIM_B200_LIB=build/variants/tc_na3/libcim_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc and (32 or 24)" -x > $O/pytest.txt 2>&1; echo "pytest(na3) exit $?"; tail -1 $O/pytest.txt
