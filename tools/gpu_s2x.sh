#!/bin/bash
# Three-ring kernel with pipelined work-item metadata: parity tests, A/B against the previous producer (alternating).
set -u
O=gpurun_out/s2x; mkdir -p $O
#timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -m gpu -k "frag or k_sweep_f32 or multipass or c2_full_size_256 or skeleton or host_batch" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
#tail
for rep in 1 2 3; do for v in new old; do
if [ $v = old ]; then export CIM_B200_LIB=build/variants/frag_old/libcim_b200.so; else unset CIM_B200_LIB; fi
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/$v.$rep.json 2> $O/$v.$rep.err
python -c "
import json;d=json.load(open('$O/$v.$rep.json'));r=d['roofline'];print('$v', round(r['kernel_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$v FAILED"; tail -2 $O/$v.$rep.err)
done; done
unset CIM_B200_LIB
for k in 16 32; do
timeout 120 python bench.py --k $k --layout frag --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/k$k.json 2>/dev/null
python -c "
import json;d=json.load(open('$O/k$k.json'));r=d['roofline'];print('frag k=$k', round(r['kernel_ms'],4))"
done
