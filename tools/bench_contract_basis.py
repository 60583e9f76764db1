"""The observables contraction on basis-built (reference-shaped) patterns:
HalfTiles.from_basis skeletons are mostly small COO-in-tile tiles.

    python tools/bench_contract_basis.py [--n 262144] [--bias 0.05] [--m 16] [--nvec 8]
"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as b2

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=262144)
ap.add_argument("--particles", type=int, default=6)
ap.add_argument("--bias", type=float, default=0.05)
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--nvec", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
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
lo = b2.construct._pack_lo(occ)
g_occ, g_lo, _, _ = b2.group_basis(occ, lo, 16)
H = b2.HalfTiles.from_basis(g_occ, g_lo)
stored = H.meta["stored_entries"]
diag = int((H.tile_rc_host[:, 0] == H.tile_rc_host[:, 1]).sum()) if H.n_tiles else 0
c = b2.random_coefficients(a.nvec, a.n, seed=1)
inp = b2.ObservablesInput(c=c, m_ops=a.m, seed=3)
b2.contract_pattern(H, inp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    b2.contract_pattern(H, inp)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(json.dumps({"n": a.n, "bias": a.bias, "n_vec": a.nvec, "m_ops": a.m, "stored_entries": stored,
                  "dense_tiles": H.n_tiles, "sparse_tiles": H.n_sparse_tiles, "ms": round(ms, 3),
                  "G_stored_pair_ops_per_s": round(stored * a.m / ms / 1e6, 1)}))
