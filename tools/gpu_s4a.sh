#!/bin/bash
# DMMA Gram: steps per iteration 1 / 2 / 4 vs the FFMA2 FAST kernel (LOBPCG per-kernel times).
# (A/B of a variant that was measured and reverted — see profiles/r02; the variant code is no longer in the tree)
set -u
O=gpurun_out/s4a; mkdir -p $O
timeout 900 python -m pytest tests/test_lobpcg.py tests/test_gpu_parity.py -q -m gpu -k "lobpcg or gram" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for v in u2 gd1 gd4 ffma; do
  unset CIM_GRAM_NO_DMMA CIM_B200_LIB
  case $v in gd*) export CIM_B200_LIB=build/variants/$v/libcim_b200.so;; ffma) export CIM_GRAM_NO_DMMA=1;; esac
  timeout 600 python tools/prof_lobpcg.py > $O/p.json 2>$O/p.err
  python -c "
import json; d=json.load(open('$O/p.json')); g={k: v for k, v in d.items() if 'gram' in k}; print('$v', round(d['device_ms_per_iter'],3), round(sum(g.values()),4), g)"
done
