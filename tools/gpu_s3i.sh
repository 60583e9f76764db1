#!/bin/bash
# Symmetric CSR row walk: four gathers in flight per lane vs two (A/B on basis skeletons), CSR tests.
set -u
O=gpurun_out/s3i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -m gpu -k "csr or basis or sparse" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for rep in 1 2; do for v in ilp4 ilp2; do for args in "--n 262144 --bias 0.05" "--n 65536 --bias 0.1" "--n 262144 --bias 0.05 --k 16"; do
  if [ $v = ilp2 ]; then export CIM_B200_LIB=build/variants/csr_ilp2/libcim_b200.so; else unset CIM_B200_LIB; fi
  timeout 600 python tools/bench_basis_spmm.py $args > $O/b.json 2>&1
  echo "$v $args: $(tail -1 $O/b.json | cut -c1-300)"
done; done; done
