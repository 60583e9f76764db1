#!/bin/bash
set -u
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -m gpu -k "csr or basis or skeleton or sparse" --timeout 300 2>&1 | tail -2
for f in 0.01 0.02; do
timeout 300 python bench.py --fill $f --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/f.json 2>/dev/null
python -c "
import json;d=json.load(open('/tmp/f.json'));print('fill $f', round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))"
done
