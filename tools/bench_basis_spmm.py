"""SpMM on reference-style matrices built from a many-body basis
(HalfTiles.from_basis): per-apply time and rates for the dense / sparse tile
split the construction picks.

    python tools/bench_basis_spmm.py [--n 262144] [--bias 0.05] [--k 8]
"""
import argparse, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as b2

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=262144)
ap.add_argument("--particles", type=int, default=6)
ap.add_argument("--bias", type=float, default=0.05)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--dense-fill", type=float, default=None)
a = ap.parse_args()

rng = np.random.default_rng(0)
n_sp = 128
w = np.exp(-a.bias * np.arange(1, n_sp + 1))
occ = np.zeros((0, a.particles), np.uint16)
for _ in range(50):
    if occ.shape[0] >= a.n:
        break
    m = 2 * (a.n - occ.shape[0]) + 1024
    keys = np.log(rng.random((m, n_sp))) / w
    pick = np.sort(np.argpartition(-keys, a.particles, axis=1)[:, :a.particles] + 1, axis=1).astype(np.uint16)
    occ = np.unique(np.concatenate([occ, pick]), axis=0)
if occ.shape[0] < a.n:
    sys.exit(f"only {occ.shape[0]} distinct states at bias {a.bias}: lower --bias")
occ = occ[rng.permutation(occ.shape[0])[:a.n]]
lo = np.zeros(a.n, np.uint64)
for q in range(a.particles):
    sel = occ[:, q] <= 64
    lo[sel] |= np.left_shift(np.uint64(1), (occ[sel, q] - 1).astype(np.uint64))
order = np.argsort(lo & np.uint64(0xFF), kind="stable")
occ, lo = occ[order], lo[order]
H = b2.HalfTiles.from_basis(occ, lo, dense_fill=a.dense_fill)
X = torch.randn((a.n, a.k), device="cuda")
Y = b2.sym_spmm(H, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    b2.sym_spmm(H, X, out=Y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
stored = H.meta["stored_entries"]
n_diag_entries = None
ab = H.algorithmic_bytes(a.k)
out = {"n": a.n, "bias": a.bias, "k": a.k, "csr": os.environ.get("CIM_SPARSE_CSR", "1") != "0",
       "stored_entries": stored, "dense_tiles": H.n_tiles, "algorithmic_bytes": ab,
       "hbm_frac": round(ab / (ms / 1e3) / 1e9 / 6548.5, 4),
       "sparse_tiles": H.n_sparse_tiles, "ms_per_apply": round(ms, 4),
       "G_stored_entries_per_s": round(stored / ms / 1e6, 2),
       "GFLOP_per_s_approx": round(4 * a.k * stored / ms / 1e6, 1)}
print(json.dumps(out))
