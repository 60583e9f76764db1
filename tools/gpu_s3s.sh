#!/bin/bash
# Gram FAST row loop: rows per step 1 / 2 (default) / 4 — parity and LOBPCG per-kernel times.
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s3s; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or gram" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for rep in 1 2; do for v in ru2 gram_ru1 gram_ru4; do
  if [ $v = ru2 ]; then unset CIM_B200_LIB; else export CIM_B200_LIB=build/variants/$v/libcim_b200.so; fi
  timeout 600 python tools/prof_lobpcg.py > $O/p.json 2>$O/p.err
  python -c "
import json; d=json.load(open('$O/p.json')); print('$v', round(d['wall_ms_per_iter'],3), round(d['device_ms_per_iter'],3), {k: v for k, v in d.items() if 'gram' in k})"
done; done
