#!/bin/bash
# Gram kernel with 8x4 blocks per thread (FAST): parity + LOBPCG per-kernel times.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s3r; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or ritz or gram" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do
  timeout 600 python tools/prof_lobpcg.py > $O/new.json 2>$O/new.err; echo "new $(tail -1 $O/new.json)"
  timeout 600 python tools/bench_lobpcg.py > $O/bn.json 2>&1; echo "bench $(tail -1 $O/bn.json | cut -c1-120)"
done
