#!/bin/bash
# Round-2: the small-tile row-CSR path — tests, basis skeleton and 1%-fill timings (CSR on / off).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -m gpu -k "csr or sparse or sharded" --timeout 600 > gpurun_out/pytest_csr.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_csr.txt
for csr in 1 0; do
  CIM_SPARSE_CSR=$csr timeout 600 python tools/bench_basis_spmm.py --n 262144 --bias 0.05 >> gpurun_out/basis_csr.jsonl 2>>gpurun_out/basis_csr.err
  CIM_SPARSE_CSR=$csr timeout 600 python tools/bench_basis_spmm.py --n 65536 --bias 0.1 >> gpurun_out/basis_csr.jsonl 2>>gpurun_out/basis_csr.err
  CIM_SPARSE_CSR=$csr timeout 600 python bench.py --steps 20 --warmup 3 --fill 0.01 --no-cpu-baseline --e2e-steps 1 >> gpurun_out/fill_csr.jsonl 2>>gpurun_out/fill_csr.err
done
tail -3 gpurun_out/pytest_csr.txt; cat gpurun_out/basis_csr.jsonl; python - <<'P'
import json
for l in open("gpurun_out/fill_csr.jsonl"):
    d=json.loads(l); print(d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel_ms"])
P
