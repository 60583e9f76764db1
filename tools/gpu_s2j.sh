#!/bin/bash
# f64 DMMA kernel: tc parity tests (both dtypes), then bench f64 k = 8/16/32 on both layouts.
set -u
O=gpurun_out/s2j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc or f64" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -15 $O/pytest.txt
for k in 8 16 32; do for L in tc frag; do
timeout 120 python bench.py --dtype f64 --layout $L --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/f64_${L}_k$k.json 2> $O/f64_${L}_k$k.err
python -c "
import json;d=json.load(open('$O/f64_${L}_k$k.json'));r=d['roofline'];print('f64 $L k=$k', round(r['kernel_ms'],3), round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || tail -3 $O/f64_${L}_k$k.err
done; done
