#!/bin/bash
# A/B timing of library variants on the default bench workload (+ a quick parity
# run on each).  Usage: VARIANTS="main diagbranch rowatomic" bash tools/ab.sh [bench args]
mkdir -p gpurun_out
for v in ${VARIANTS:-main}; do
  if [ "$v" = main ]; then L=paper_2110_10765_b200/libcim_b200.so; else L=build/variants/$v/libcim_b200.so; fi
  if [ "${PARITY:-1}" = 1 ]; then
    CIM_B200_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/ab_pytest_$v.txt 2>&1
    echo "$v parity: $(tail -1 gpurun_out/ab_pytest_$v.txt)"
  fi
  for rep in 1 2; do
    CIM_B200_LIB=$L timeout 300 python bench.py --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['roofline']['kernel_ms'],4), 'ms', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'), d['clocks']['reasons'])" || tail -3 gpurun_out/ab_$v.err
  done
done
