#!/bin/bash
# Symmetric CSR walk: lanes sharing an entry's X row (SUB) and gathers in flight (ILP) — A/B on basis skeletons.
set -u
O=gpurun_out/s3l; mkdir -p $O
: timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -m gpu -k "csr or basis or sparse" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
: tail -3
for rep in 1 2; do for v in new minb4 minb5 minb6 prev; do for args in "--n 262144 --bias 0.05" "--n 262144 --bias 0.05 --k 16" "--n 262144 --bias 0.05 --k 32" "--n 65536 --bias 0.1"; do
  case $v in new) unset CIM_B200_LIB;;
    minb*) export CIM_B200_LIB=build/variants/csr_$v/libcim_b200.so;; prev) export CIM_B200_LIB=build/variants/csr_ilp2/libcim_b200.so;; esac
  timeout 600 python tools/bench_basis_spmm.py $args > $O/b.json 2>&1
  echo "$v $args: $(tail -1 $O/b.json | grep -o '"ms_per_apply": [0-9.]*')"
done; done; done
