#!/bin/bash
# Role timers of the split-TF32 kernel (CIM_TC_PROF build) at k = 8, 16, 64.
set -u
O=gpurun_out/s2g; mkdir -p $O
export CIM_B200_LIB=build/variants/tc_prof/libcim_b200.so
for k in 8 16 64; do timeout 120 python tools/tc_profile.py $k 2>&1 | tail -5; done | tee $O/tc_prof.txt
