#!/bin/bash
# Drop-in contraction timing; basis skeleton with every sparse tile on the CSR path (CIM_SPARSE_SMALL=4096) vs default.
set -u
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python tools/bench_dropin_contract.py --n 4096 > $O/dropin_4096.json 2> $O/dropin.err
timeout 600 python tools/bench_dropin_contract.py --n 16384 --bias 0.1 > $O/dropin_16384.json 2>> $O/dropin.err
for sm in 128 256 512 4096; do
  CIM_SPARSE_SMALL=$sm timeout 600 python tools/bench_basis_spmm.py --n 262144 --bias 0.05 > $O/basis_small$sm.json 2>>$O/basis.err
done
cat $O/dropin_*.json; tail -3 $O/dropin.err; for f in $O/basis_small*.json; do echo $f; cat $f; done; tail -3 $O/basis.err
