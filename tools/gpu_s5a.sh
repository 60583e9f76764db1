#!/bin/bash
# Final C4 sweep on both layouts, plus the column-pass widths added this session.
set -u
O=gpurun_out/s5a; mkdir -p $O
bash tools/sweep_k.sh > $O/sweep.txt 2>&1; cp gpurun_out/k_sweep.jsonl $O/k_sweep.jsonl
for cfg in "f64 64 tc" "f64 64 frag" "f64 40 frag" "f64 20 frag" "f32 40 frag" "f32 56 frag" "f32 24 tc"; do
  set -- $cfg
  timeout 300 python bench.py --steps 10 --warmup 3 --dtype $1 --k $2 --layout $3 --no-cpu-baseline --e2e-steps 1 > $O/x.json 2>/dev/null && cat $O/x.json >> $O/k_sweep.jsonl
  python -c "import json;d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]);print('$1 k=$2 $3', round(d['roofline']['kernel_ms'],3), round(d['value']), 'GFLOP/s', d['clocks']['reasons'])"
done
cat $O/sweep.txt | tail -20
