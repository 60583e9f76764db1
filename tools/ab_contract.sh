# A/B of contraction-kernel variants (build with tools/build_variant.sh): C1 pattern, n_vec x m_ops cases
for v in main ${VARIANTS:-}; do
  if [ "$v" = main ]; then L=paper_2110_10765_b200/libcim_b200.so; else L=build/variants/$v/libcim_b200.so; fi
  CIM_B200_LIB=$L timeout 300 python tools/bench_contract.py --cases 8x4,8x16,16x16 2>/dev/null | python -c "
import json,sys
for line in sys.stdin:
    d=json.loads(line); print('$v', d['n_vec'], d['m_ops'], d['fused']['ms'])"
done
