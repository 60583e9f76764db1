"""BASELINE config 5: LOBPCG-style iteration, lowest 8 eigenpairs.

    python tools/bench_lobpcg.py [--n N] [--tiles T] [--iters I]
    torchrun --nproc-per-node G tools/bench_lobpcg.py ...   (row-sharded)

Times LOBPCG iterations (one sharded SpMM + Gram all-reduce + Rayleigh-Ritz
+ Cholesky-QR each) on the synthetic half-stored H; prints one JSON line with
ms/iteration (max over ranks), the Ritz values and residual norms.
"""
import argparse, json, os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as pkg
from paper_2110_10765_b200.lobpcg import lobpcg
from paper_2110_10765_b200.sharded import ShardedSymSpmm

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--tiles-per-gpu", type=int, default=488_281)
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local); dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
nb = (args.n + 63) // 64
n_off = max(0, world * args.tiles_per_gpu - nb)
p = n_off / (nb * (nb - 1) // 2)
S = ShardedSymSpmm.synthetic(args.n, k=args.m, p=p, seed=0, device=dev)
g = torch.Generator(device="cpu").manual_seed(rank)
X0 = torch.randn((S.rows_per_rank, args.m), generator=g, dtype=torch.float32).to(dev)
lo, hi = S.local_rows(); X0[max(0, hi - lo):] = 0
lobpcg(S.apply, X0, max_iter=3, tol=0.0)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
res = lobpcg(S.apply, X0, max_iter=args.iters, tol=0.0)
torch.cuda.synchronize()
dt = torch.tensor([(time.perf_counter() - t0) / args.iters], device=dev, dtype=torch.float64)
if world > 1:
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
if rank == 0:
    print(json.dumps({"metric": "LOBPCG iteration time (lowest 8, sharded SpMM + 24x24 Gram all-reduce)",
                      "value": float(dt) * 1e3, "unit": "ms/iteration", "n_gpus": world, "n": args.n,
                      "stored_tiles": S.H.meta.get("global_tiles"), "iterations": res.iterations,
                      "ritz_values": [float(x) for x in res.eigenvalues],
                      "residual_norms": [float(x) for x in res.residual_norms], "spmm_calls": res.spmm_calls}))
if world > 1:
    dist.destroy_process_group()
