#!/bin/bash
# Compressed tensor-core tiles: tcz tests, then 17%-fill C2 on every storage (sparse COO, dense frag, tcz) and dense tcz.
set -u
O=gpurun_out/s2y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tcz" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -15 $O/pytest.txt
for L in tcz; do for f in 0.05 0.17 0.3; do
timeout 300 python bench.py --fill $f --layout $L --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/fill${f}_$L.json 2> $O/fill${f}_$L.err
python -c "
import json;d=json.load(open('$O/fill${f}_$L.json'));r=d['roofline'];print('fill $f $L', round(r['kernel_ms'],3), 'frac', round(r['frac'],3), round(d['value']))" 2>/dev/null || (echo "fill $f $L FAILED"; tail -3 $O/fill${f}_$L.err)
done; done
for k in 8 16; do
timeout 300 python bench.py --layout tcz --k $k --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/dense_tcz_k$k.json 2> $O/dense_tcz_k$k.err
python -c "
import json;d=json.load(open('$O/dense_tcz_k$k.json'));r=d['roofline'];print('dense tcz k=$k', round(r['kernel_ms'],3))" 2>/dev/null || (echo "dense tcz FAILED"; tail -3 $O/dense_tcz_k$k.err)
done
