#!/bin/bash
# tc kernel with pipelined unit metadata: tc tests, bench k = 8 / 16 / 32.
set -u
O=gpurun_out/s2w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for k in 8 16 32; do
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/k$k.json 2> $O/k$k.err
python -c "
import json;d=json.load(open('$O/k$k.json'));r=d['roofline'];print('tc k=$k', round(r['kernel_ms'],3))" 2>/dev/null || (echo "k=$k FAILED"; tail -2 $O/k$k.err)
done; done
timeout 120 python bench.py --k 8 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/frag8.json 2>/dev/null
python -c "
import json;d=json.load(open('$O/frag8.json'));r=d['roofline'];print('frag k=8', round(r['kernel_ms'],3))"
