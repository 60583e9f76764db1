#!/bin/bash
# First run of the split-TF32 tensor-core kernel: tc parity tests, then bench k = 8/16/32/64.
set -u
O=gpurun_out/s2c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" -x --timeout 120 > $O/pytest_tc.txt 2>&1; echo "pytest exit $?" >> $O/pytest_tc.txt
tail -15 $O/pytest_tc.txt
for k in 8 16 32 64; do
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/tc_k$k.json 2> $O/tc_k$k.err
echo "k=$k exit $?"; tail -2 $O/tc_k$k.err | cut -c1-300
python -c "
import json;d=json.load(open('$O/tc_k$k.json'));r=d['roofline'];print('tc k=$k', d['ms_per_step'], r['kernel_ms'], d['value'], d['clocks']['sm_mhz'])" 2>/dev/null
done
