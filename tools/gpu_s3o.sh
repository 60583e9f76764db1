#!/bin/bash
# LOBPCG: Cholesky Rayleigh-Ritz + fused projection/orth + fused Ritz update/residual vs the previous solver (same box).
# scratch_ab/lobpcg_prev.py is the previous solver: git show 6227252:paper_2110_10765_b200/lobpcg.py > scratch_ab/lobpcg_prev.py
set -u
O=gpurun_out/s3o; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or ritz or tsmm or gram" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
rm -rf /tmp/oldrepo; cp -r . /tmp/oldrepo; cp scratch_ab/lobpcg_prev.py /tmp/oldrepo/paper_2110_10765_b200/lobpcg.py
for rep in 1 2 3; do
  timeout 600 python tools/bench_lobpcg.py > $O/new.json 2>&1; echo "new $(tail -1 $O/new.json | cut -c1-200)"
  (cd /tmp/oldrepo && timeout 600 python tools/bench_lobpcg.py) > $O/old.json 2>&1; echo "old $(tail -1 $O/old.json | cut -c1-200)"
done
