#!/bin/bash
# Quick GPU iteration: GPU parity tests + a 50-step bench (no ncu).
# Usage (repo root on the GPU box): bash tools/gpu_quick.sh [extra bench args]
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
