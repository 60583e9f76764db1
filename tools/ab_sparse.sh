# A/B of sparse-kernel variants (build with tools/build_variant.sh): synthetic fills and a basis skeleton
for v in main ${VARIANTS:-}; do
  if [ "$v" = main ]; then L=paper_2110_10765_b200/libcim_b200.so; else L=build/variants/$v/libcim_b200.so; fi
  for f in 0.03 0.05 0.09; do
    CIM_B200_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fill $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v fill $f', round(d['ms_per_step'],3))"
  done
  CIM_B200_LIB=$L timeout 300 python tools/bench_basis_spmm.py --n 65536 --bias 0.1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v basis65k', d['ms_per_apply'], d['dense_tiles'], d['sparse_tiles'])"
done
