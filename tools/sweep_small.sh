mkdir -p gpurun_out
for t in 0 32 64 128 256; do
  echo "== CIM_SPARSE_SMALL=$t"
  CIM_SPARSE_SMALL=$t timeout 300 python tools/bench_basis_spmm.py --n 262144 --bias 0.05
  CIM_SPARSE_SMALL=$t timeout 300 python tools/bench_basis_spmm.py --n 65536 --bias 0.2
  CIM_SPARSE_SMALL=$t timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fill 0.05 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fill0.05', d['ms_per_step'])"
  CIM_SPARSE_SMALL=$t timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --fill 0.01 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fill0.01', d['ms_per_step'])"
done
