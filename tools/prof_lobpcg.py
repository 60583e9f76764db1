"""Per-kernel device time of LOBPCG iterations (torch.profiler / CUPTI) on
the C2 matrix: prints one JSON line {kernel: ms per iteration} plus the
wall time per iteration, so the host share is the difference."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_10765_b200.lobpcg import lobpcg
from paper_2110_10765_b200.sharded import ShardedSymSpmm

n, iters = 1 << 22, 10
dev = torch.device("cuda", 0)
nb = (n + 63) // 64
p = max(0, 488_281 - nb) / (nb * (nb - 1) // 2)
S = ShardedSymSpmm.synthetic(n, k=8, p=p, seed=0, device=dev)
X0 = torch.randn((S.rows_per_rank, 8), generator=torch.Generator().manual_seed(0)).to(dev)
lobpcg(S.apply, X0, max_iter=3, tol=0.0)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    res = lobpcg(S.apply, X0, max_iter=iters, tol=0.0)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / res.iterations
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        key = e.name.replace("(anonymous namespace)::", "").split("(")[0][:90] or "<unnamed>"
        tot[key] = tot.get(key, 0.0) + e.device_time_total / 1e3 / res.iterations
out = {"wall_ms_per_iter": wall * 1e3, "device_ms_per_iter": sum(tot.values())}
out.update({k: round(v, 4) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])})
print(json.dumps(out))
