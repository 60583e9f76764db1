#!/bin/bash
# Re-entry check + column-band A/B on the three-ring kernel (C2, k = 8 f32).
set -u
O=gpurun_out/s2a; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke exit $?" >> $O/smoke.txt
cat $O/smoke.txt
for rep in 1 2; do
for B in 1 2 3 4; do
timeout 300 python bench.py --steps 20 --warmup 5 --bands $B --no-cpu-baseline --e2e-steps 1 > $O/bands$B.$rep.json 2> $O/bands$B.$rep.err
python -c "
import json;d=json.load(open('$O/bands$B.$rep.json'));r=d['roofline'];print('bands $B', d['ms_per_step'], r['kernel_ms'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
