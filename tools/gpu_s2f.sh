#!/bin/bash
# k = 8 bound of the split-TF32 kernel: producer-only / no-reduction variants against frag and the full tc kernel.
set -u
O=gpurun_out/s2f; mkdir -p $O
for rep in 1 2; do
for v in frag base tc_NOWORK tc_NOWORK_NORED tc_NORED; do
L=tc; if [ $v = frag ]; then L=frag; fi
if [ $v = base ] || [ $v = frag ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
timeout 120 python bench.py --layout $L --k 8 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/$v.$rep.json 2> $O/$v.$rep.err
python -c "
import json;d=json.load(open('$O/$v.$rep.json'));r=d['roofline'];print('$v k=8', round(r['kernel_ms'],3))" 2>/dev/null || echo "$v failed"
done; done
