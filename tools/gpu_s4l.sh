#!/bin/bash
# Final evidence run: full -m gpu suite, smoke, bench (20 steps, as the driver), reference arm, launch list.
set -u
O=gpurun_out/s4l; mkdir -p $O
timeout 2000 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt; tail -2 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt; tail -1 $O/smoke.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json | cut -c1-160
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
python -c "
import json;d=json.loads(open('$O/bench20.json').read().strip().splitlines()[-1]);r=d['roofline'];print('bench', d['ms_per_step'], r['frac'], r['kernel_ms'], d['e2e']['value'], d['clocks'], d['gpu_launches'], d['cpu_baseline']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_k8_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu exit $?"; grep -c sym_spmm $O/launches_k8_final.csv
