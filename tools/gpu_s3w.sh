#!/bin/bash
# DMMA kernel: paired column blocks with interleaved vectors (16-byte B loads, conflict-free) vs the previous build.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s3w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -m gpu -k "float64 or f64" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/dmma_old/libcim_b200.so; fi
  for k in 8 16 24 32; do
  timeout 300 python bench.py --dtype f64 --k $k --layout tc --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$v f64 k=$k', round(d['roofline']['kernel_ms'],3), round(d['value']/1e3,2), 'TF', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done
unset CIM_B200_LIB
timeout 600 ncu --set full --clock-control none -k regex:dmma -s 2 -c 1 -o $O/prof_dmma16 -f python bench.py --dtype f64 --k 16 --layout tc --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu.log 2>&1; tail -1 $O/ncu.log
