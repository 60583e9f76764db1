#!/bin/bash
# Round-2 measurement batch: headline bench (20 / 100 steps), ncu launch list +
# one full capture of the k8 kernel, C1 (L2-flushed), C3 on one GPU, the C4 k
# sweep, C5 LOBPCG, the 17%-fill sparse line.
set -u
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench100.json 2> $O/bench100.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_bench.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_spmm_k8 -s 3 -c 1 -o $O/prof_k8 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full.log 2>&1
timeout 300 python bench.py --n 65536 --tiles-per-gpu 6268 --steps 200 --warmup 10 > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --tiles-per-gpu 3906250 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c3.json 2> $O/c3.err
timeout 300 python bench.py --steps 20 --warmup 3 --fill 0.17 --no-cpu-baseline --e2e-steps 1 > $O/fill17.json 2> $O/fill17.err
timeout 300 python tools/bench_lobpcg.py > $O/lobpcg.json 2> $O/lobpcg.err
timeout 1200 bash tools/sweep_k.sh > $O/k_sweep.txt 2>&1; cp gpurun_out/k_sweep.jsonl $O/ 2>/dev/null
for f in bench20 bench100 c1 c3 fill17; do python -c "
import json;d=json.load(open('$O/$f.json'));print('$f', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'kern', round(d['roofline']['kernel_ms'],4), d['clocks'])" || tail -3 $O/$f.err; done
cat $O/k_sweep.txt; cat $O/lobpcg.json | head -c 600
