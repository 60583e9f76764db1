#!/bin/bash
# Symmetric (both-triangle) CSR for the small sparse tiles: tests, then basis skeletons half vs symmetric.
set -u
O=gpurun_out/s3d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -m gpu -k "csr" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for sym in 0 1; do for args in "--n 262144 --bias 0.05" "--n 65536 --bias 0.1"; do
CIM_SPARSE_CSR_SYM=$sym timeout 600 python tools/bench_basis_spmm.py $args > $O/basis_sym$sym.json 2>&1
echo "sym=$sym $args: $(tail -1 $O/basis_sym$sym.json | cut -c1-400)"
done; done
