#!/bin/bash
# Three-ring kernel with bulk Y reductions: parity tests, then A/B vs red.v4 (CIM_K8_SCALAR_RED=1), C2 k=8, alternating.
set -u
O=gpurun_out/s2q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -m gpu -k "frag or k_sweep_f32 or c2_full or skeleton or sharded or host_batch" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2 3; do for v in bulk scalar; do
if [ $v = scalar ]; then export CIM_K8_SCALAR_RED=1; else unset CIM_K8_SCALAR_RED; fi
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/$v.$rep.json 2> $O/$v.$rep.err
python -c "
import json;d=json.load(open('$O/$v.$rep.json'));r=d['roofline'];print('$v', round(r['kernel_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$v FAILED"; tail -2 $O/$v.$rep.err)
done; done
unset CIM_K8_SCALAR_RED
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k8r3 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_bulk.csv 2>/dev/null
grep -E "dram__bytes|gpu__time" $O/ncu_bulk.csv | tail -3 | awk -F'","' '{print $(NF-2), $NF}'
