# A/B of the multi-pass widths (C4): the shipped library vs a variant built with
# tools/build_variant.sh (e.g. VARIANT=rowpasses after -DCIM_K8_ROW_PASSES).
# A/B of the multi-pass widths: the shipped library vs a variant (VARIANT=name under build/variants)
for v in main ${VARIANT:-}; do
  if [ "$v" = main ]; then L=paper_2110_10765_b200/libcim_b200.so; else L=build/variants/$v/libcim_b200.so; fi
  for a in "--dtype f64 --k 16" "--dtype f64 --k 32" "--k 32" "--k 24" "--k 64"; do
    CIM_B200_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 $a 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$a', round(d['ms_per_step'],3))"
  done
done
