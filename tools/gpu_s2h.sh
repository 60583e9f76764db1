#!/bin/bash
# split-TF32 kernel: tc parity tests, bench k = 8..64, role timers.
set -u
O=gpurun_out/s2h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" -x --timeout 120 > $O/pytest_tc.txt 2>&1; echo "pytest exit $?" >> $O/pytest_tc.txt
tail -3 $O/pytest_tc.txt
for k in 8 16 32 64; do
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/tc_k$k.json 2> $O/tc_k$k.err
python -c "
import json;d=json.load(open('$O/tc_k$k.json'));r=d['roofline'];print('tc k=$k', round(r['kernel_ms'],3), round(d['value']), d['clocks']['sm_mhz'])" 2>/dev/null || tail -3 $O/tc_k$k.err
done
export CIM_B200_LIB=build/variants/tc_prof/libcim_b200.so
for k in 16 64; do timeout 120 python tools/tc_profile.py $k 2>&1 | tail -5; done | tee $O/tc_prof.txt
