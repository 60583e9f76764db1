#!/bin/bash
# DMMA kernel with interleaved B fragments: f64 tests + bench k = 8/16/24/32.
set -u
O=gpurun_out/s2o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "f64" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for k in 8 16 24 32; do
timeout 120 python bench.py --dtype f64 --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/f64_k$k.json 2> $O/f64_k$k.err
python -c "
import json;d=json.load(open('$O/f64_k$k.json'));r=d['roofline'];print('f64 tc k=$k', round(r['kernel_ms'],3), round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "k=$k FAILED"; tail -2 $O/f64_k$k.err)
done
