#!/bin/bash
# Even rings for the two-group tensor-core kernels: tests, racecheck, bench f64 / f32 tc widths.
set -u
O=gpurun_out/s2l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tc or f64" -x --timeout 120 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for cfg in "f64 8" "f32 16"; do set -- $cfg
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python bench.py --dtype $1 --layout tc --k $2 --tiles-per-gpu 100000 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/racecheck_$1_$2.txt 2>&1
grep "RACECHECK SUMMARY\|ERROR SUMMARY" $O/racecheck_$1_$2.txt
done
for cfg in "f64 8" "f64 16" "f64 24" "f64 32" "f32 16" "f32 24" "f32 32" "f32 64"; do set -- $cfg
timeout 120 python bench.py --dtype $1 --layout tc --k $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/$1_k$2.json 2> $O/$1_k$2.err
python -c "
import json;d=json.load(open('$O/$1_k$2.json'));r=d['roofline'];print('$1 tc k=$2', round(r['kernel_ms'],3), round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$1 k=$2 FAILED"; tail -2 $O/$1_k$2.err)
done
