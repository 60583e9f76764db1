#!/bin/bash
# Gram on DMMA (exact f64 products) vs the FFMA2 FAST kernel: parity, LOBPCG per-kernel times.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s3z; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or gram or ritz or tsmm" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for rep in 1 2; do for v in dmma ffma; do
  if [ $v = dmma ]; then unset CIM_GRAM_NO_DMMA; else export CIM_GRAM_NO_DMMA=1; fi
  timeout 600 python tools/prof_lobpcg.py > $O/p.json 2>$O/p.err
  python -c "
import json; d=json.load(open('$O/p.json')); print('$v', round(d['wall_ms_per_iter'],3), round(d['device_ms_per_iter'],3), {k: v for k, v in d.items() if 'gram' in k})"
  timeout 600 python tools/bench_lobpcg.py > $O/b.json 2>&1; echo "$v bench $(tail -1 $O/b.json | cut -c80-160)"
done; done
