#!/bin/bash
# Symmetric CSR walk: dedicated kernel (4 gathers in flight, k=16 in one pass) vs the previous build; ncu L1 breakdown.
set -u
O=gpurun_out/s3j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -m gpu -k "csr or basis or sparse" -x --timeout 300 > $O/pytest.txt 2>&1; echo "pytest exit $?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for rep in 1 2; do for v in new old; do for args in "--n 262144 --bias 0.05" "--n 262144 --bias 0.05 --k 16" "--n 65536 --bias 0.1 --k 16"; do
  if [ $v = old ]; then export CIM_B200_LIB=build/variants/csr_ilp2/libcim_b200.so; else unset CIM_B200_LIB; fi
  timeout 600 python tools/bench_basis_spmm.py $args > $O/b.json 2>&1
  echo "$v $args: $(tail -1 $O/b.json | grep -o '"ms_per_apply": [0-9.]*')"
done; done; done
unset CIM_B200_LIB
timeout 900 ncu --set full --metrics breakdown:l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum --clock-control none -k regex:csr_sym -s 2 -c 1 -o $O/prof_csr_sym2 -f \
  python tools/bench_basis_spmm.py --n 262144 --bias 0.05 --reps 3 > $O/ncu_csr.log 2>&1
tail -1 $O/ncu_csr.log
