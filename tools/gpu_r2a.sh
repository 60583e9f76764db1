#!/bin/bash
# Round-2 check: new parity tests first, then the whole -m gpu suite, the
# default bench line and the reference arm.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
free -g >> gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests/test_dropin_contraction.py tests/test_gpu_scale_parity.py -q -m gpu --timeout 600 -x ${PYTEST_ARGS:-} > gpurun_out/pytest_new.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_new.txt
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
tail -5 gpurun_out/pytest_new.txt; tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err gpurun_out/bench_ref.err
