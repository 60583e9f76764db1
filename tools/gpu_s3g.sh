#!/bin/bash
# Symmetric CSR for the staged (mid-fill) tiles too (A/B, CIM_CSR_ALL_TILES=1 CIM_CSR_SMALL_SHARE=0).
set -u
for f in 0.03 0.05 0.09 0.13; do
for v in default csr; do
if [ $v = csr ]; then export CIM_CSR_ALL_TILES=1 CIM_CSR_SMALL_SHARE=0; else unset CIM_CSR_ALL_TILES CIM_CSR_SMALL_SHARE; fi
timeout 300 python bench.py --fill $f --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/f.json 2>/dev/null
python -c "
import json;d=json.load(open('/tmp/f.json'));print('fill $f $v', round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))" 2>/dev/null || echo "fill $f $v failed"
done; done
