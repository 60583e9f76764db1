#!/bin/bash
# Role timers of the tc kernel at k = 16, 32, 64 (where the MMA pipe is 65% / ~40% / ? busy).
set -u
O=gpurun_out/s3t; mkdir -p $O
export CIM_B200_LIB=build/variants/tc_prof/libcim_b200.so
for k in 16 32 64; do timeout 180 python tools/tc_profile.py $k 2>&1 | tail -6; done | tee $O/tc_prof.txt
