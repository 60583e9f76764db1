#!/bin/bash
# With both triangles in the CSR: does the row walk now beat the entry-parallel small kernel (1% fill) and the staged ring (5% fill)?
set -u
for f in 0.01 0.05 0.09; do
for v in default csr_all; do
if [ $v = csr_all ]; then export CIM_CSR_MIN_ROW=0 CIM_CSR_SMALL_SHARE=0; else unset CIM_CSR_MIN_ROW CIM_CSR_SMALL_SHARE; fi
timeout 300 python bench.py --fill $f --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/f.json 2>/dev/null
python -c "
import json;d=json.load(open('/tmp/f.json'));print('fill $f $v', round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))" 2>/dev/null || echo "fill $f $v failed"
done; done
