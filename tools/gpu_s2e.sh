#!/bin/bash
# Where the split-TF32 kernel's time goes: variants with one role's work removed (wrong results, timing only).
set -u
O=gpurun_out/s2e; mkdir -p $O
for k in 8 16 64; do
for v in base tc_NO_BUILDB tc_NO_COLS tc_NO_ROWS tc_NO_MMA; do
if [ $v = base ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
timeout 120 python bench.py --layout tc --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/$v.k$k.json 2> $O/$v.k$k.err
python -c "
import json;d=json.load(open('$O/$v.k$k.json'));r=d['roofline'];print('$v k=$k', round(r['kernel_ms'],3))" 2>/dev/null || echo "$v k=$k failed"
done; done
