#!/bin/bash
# LOBPCG per-kernel breakdown, new vs previous solver; fused-kernel parity.
# scratch_ab/lobpcg_prev.py is the previous solver: git show 6227252:paper_2110_10765_b200/lobpcg.py > scratch_ab/lobpcg_prev.py
set -u
O=gpurun_out/s3p; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or ritz" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
rm -rf /tmp/oldrepo; cp -r . /tmp/oldrepo; cp scratch_ab/lobpcg_prev.py /tmp/oldrepo/paper_2110_10765_b200/lobpcg.py
for rep in 1 2; do
  timeout 600 python tools/prof_lobpcg.py > $O/new.json 2>$O/new.err; echo "new $(tail -1 $O/new.json)"
  (cd /tmp/oldrepo && timeout 600 python tools/prof_lobpcg.py) > $O/old.json 2>$O/old.err; echo "old $(tail -1 $O/old.json)"
  timeout 600 python tools/bench_lobpcg.py > $O/bn.json 2>&1; echo "bench new $(tail -1 $O/bn.json | cut -c1-120)"
  (cd /tmp/oldrepo && timeout 600 python tools/bench_lobpcg.py) > $O/bo.json 2>&1; echo "bench old $(tail -1 $O/bo.json | cut -c1-120)"
done
