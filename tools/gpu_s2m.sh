#!/bin/bash
# Full -m gpu suite (incl. the C2 tensor-core full-size cases), then the C4 sweep on both layouts.
set -u
O=gpurun_out/s2m; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 1500 bash tools/sweep_k.sh > $O/k_sweep.txt 2>&1; cp gpurun_out/k_sweep.jsonl $O/ 2>/dev/null
cat $O/k_sweep.txt
