"""Where an LOBPCG iteration (config C5) spends its time: torch.profiler over a
few iterations on the C2 matrix, kernel table sorted by device time.
Usage (GPU box): python tools/profile_lobpcg.py [--iters 5]"""
import argparse, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_10765_b200.lobpcg import lobpcg
from paper_2110_10765_b200.sharded import ShardedSymSpmm

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--tiles", type=int, default=488_281)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--cprofile", action="store_true", help="host-side (Python) profile instead of the kernel table")
a = ap.parse_args()
dev = torch.device("cuda", 0)
nb = (a.n + 63) // 64
p = max(0, a.tiles - nb) / (nb * (nb - 1) // 2)
S = ShardedSymSpmm.synthetic(a.n, k=8, p=p, seed=0, device=dev)
X0 = torch.randn((S.rows_per_rank, 8), generator=torch.Generator().manual_seed(0)).to(dev)
X0[a.n:] = 0
lobpcg(S.apply, X0, max_iter=3, tol=0.0)
torch.cuda.synchronize()
if a.cprofile:
    import cProfile, pstats
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    lobpcg(S.apply, X0, max_iter=a.iters, tol=0.0)
    torch.cuda.synchronize()
    pr.disable()
    print(f"wall per iteration {(time.perf_counter() - t0) / a.iters * 1e3:.2f} ms (under cProfile)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    sys.exit(0)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    lobpcg(S.apply, X0, max_iter=a.iters, tol=0.0)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.iters
print(f"wall per iteration {wall*1e3:.2f} ms")
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/lobpcg_trace.json")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
# the device-side sequence of one iteration (the last): kernel name, duration
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
seq = [(e.name[:60], e.device_time if hasattr(e, "device_time") else e.cuda_time) for e in evs]
spmm = [k for k, (n, _) in enumerate(seq) if "sym_spmm" in n]
if len(spmm) >= 2:
    print("\nlast iteration, device sequence (us):")
    for n, t in seq[spmm[-2] + 1: spmm[-1] + 1]:
        print(f"  {t:9.1f}  {n}")
