#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list + one full capture.
# Usage (from the repo root on the GPU box): bash tools/gpu_check.sh [pytest-args]
# SKIP_NCU=1 skips the ncu passes; WITH_CONFIGS=1 also runs C1, C3 (one GPU),
# the C4 k sweep and the C5 LOBPCG iteration into gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_spmm -s 3 -c 1 -o gpurun_out/prof -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
fi
if [ "${WITH_CONFIGS:-0}" = "1" ]; then  # the other BASELINE configs and C5 (≈ 3 min more)
  timeout 300 python bench.py --n 65536 --tiles-per-gpu 6268 --steps 200 --warmup 10 > gpurun_out/c1_1gpu.json 2>/dev/null
  timeout 600 python bench.py --tiles-per-gpu 3906250 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_1gpu.json 2>/dev/null
  timeout 900 bash tools/sweep_k.sh > gpurun_out/k_sweep.txt 2>&1
  timeout 300 python tools/bench_lobpcg.py > gpurun_out/lobpcg.json 2>/dev/null
fi
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
