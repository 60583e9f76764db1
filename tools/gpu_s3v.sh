#!/bin/bash
# Harness check of bench.py's N > 1 path on one GPU (gloo, host-staged exchange): not a measurement.
set -u
O=gpurun_out/s3v; mkdir -p $O
for N in 2 3; do
CIM_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
  bench.py --gpus $N --tiles-per-gpu 60000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench_gloo$N.json 2> $O/bench_gloo$N.err
echo "N=$N exit $?"; tail -2 $O/bench_gloo$N.err | cut -c1-300
python -c "
import json;d=json.load(open('$O/bench_gloo$N.json'));print({k:d[k] for k in ('n_gpus','ms_per_step','value','overlap_check_rel_diff','strong_scaling','gpu_launches')}); print(d['config']['parallelism'])"
done
