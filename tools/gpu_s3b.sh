#!/bin/bash
# tc epilogue staging depth: 4 vs 2 blocks per role (CIM_TC_NEB2=1), alternating, k = 8/16/32; tc tests first.
set -u
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for k in 8 16 32; do for v in neb4 neb2; do
if [ $v = neb2 ]; then export CIM_TC_NEB2=1; else unset CIM_TC_NEB2; fi
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/b.json 2>/dev/null
python -c "
import json;d=json.load(open('/tmp/b.json'));print('k=$k $v', round(d['roofline']['kernel_ms'],3))" 2>/dev/null || echo "k=$k $v failed"
done; done; done
