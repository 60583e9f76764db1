#!/bin/bash
# Role timers of the current tc kernel at k = 8 and 16.
set -u
O=gpurun_out/s2u; mkdir -p $O
export CIM_B200_LIB=build/variants/tc_prof/libcim_b200.so
for k in 8 16; do timeout 120 python tools/tc_profile.py $k 2>&1 | tail -5; done | tee $O/tc_prof.txt
