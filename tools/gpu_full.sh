#!/bin/bash
# The driver's round-end checks: smoke, the whole -m gpu suite, the default bench line, the reference arm.
set -u
O=gpurun_out/full; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
cat $O/smoke.txt; tail -3 $O/pytest_gpu.txt; python -c "
import json;d=json.load(open('$O/bench.json'));print('bench', d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"; python -c "
import json;d=json.load(open('$O/bench_ref.json'));print('ref', d['value'], d['config']['same_config'])"
