#!/bin/bash
# Compressed-tile expansion: where the time goes (variants without zeroing / scatter / expansion; timing only).
set -u
for v in base tcz_NO_ZERO tcz_NO_SCATTER tcz_NO_EXPAND; do
if [ $v = base ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
for f in 0.05 0.17; do
timeout 300 python bench.py --fill $f --layout tcz --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/z.json 2>/dev/null
python -c "
import json;d=json.load(open('/tmp/z.json'));print('$v fill $f', round(d['roofline']['kernel_ms'],3))" 2>/dev/null || echo "$v $f failed"
done; done
