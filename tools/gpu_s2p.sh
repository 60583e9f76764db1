#!/bin/bash
# tc kernel with bulk Y reductions: tests, then A/B against per-row reds (CIM_TC_SCALAR_RED=1) at k = 8/16/32.
set -u
O=gpurun_out/s2p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for k in 8 16 32; do for v in bulk scalar; do
if [ $v = scalar ]; then export CIM_TC_SCALAR_RED=1; else unset CIM_TC_SCALAR_RED; fi
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/$v.k$k.json 2> $O/$v.k$k.err
python -c "
import json;d=json.load(open('$O/$v.k$k.json'));r=d['roofline'];print('tc $v k=$k', round(r['kernel_ms'],3))" 2>/dev/null || (echo "$v k=$k FAILED"; tail -2 $O/$v.k$k.err)
done; done; done
