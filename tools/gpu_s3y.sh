#!/bin/bash
# End-of-round validation: full -m gpu suite, smoke, default bench (20 steps), C4 sweep on both layouts.
set -u
O=gpurun_out/s3y; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt; tail -2 $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; tail -1 $O/bench20.json | cut -c1-300
bash tools/sweep_k.sh 2>&1 | tail -20
cp gpurun_out/k_sweep.jsonl $O/k_sweep.jsonl
