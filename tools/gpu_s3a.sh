#!/bin/bash
# Round-end rehearsal: smoke, full -m gpu suite, default bench (20 and 100 steps), reference arm, C4 sweep, launch list.
set -u
O=gpurun_out/s3a; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 4 > $O/bench100.json 2> $O/bench100.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_k8.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 1500 bash tools/sweep_k.sh > $O/k_sweep.txt 2>&1; cp gpurun_out/k_sweep.jsonl $O/ 2>/dev/null
cat $O/smoke.txt; tail -2 $O/pytest_gpu.txt
for f in bench20 bench100; do python -c "
import json;d=json.load(open('$O/$f.json'));r=d['roofline'];print('$f', d['ms_per_step'], r['kernel_ms'], round(r['frac'],4), d['e2e']['value'], d['clocks'])"; done
python -c "
import json;d=json.load(open('$O/bench_ref.json'));print('ref', d['value'], d['config'].get('same_config'), d.get('cpu_baseline',{}).get('cores'))"
cat $O/k_sweep.txt
