"""The drop-in contraction (contract_observables / contract_oracle with the
reference's signature, cim_contract_tiles) on a desk-scale basis: n states,
grouped with the reference's default key, every orbital pair passing the
key filter as a Tile — the reference's own workflow (pipeline.py:123-192,
:534-589).  Prints one JSON line: per-call wall time (host tile-range build,
uploads, kernel, readback) and pair rates.

    python tools/bench_dropin_contract.py [--n 4096] [--particles 6] [--bias 0.2] [--m 4] [--nvec 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as b2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--particles", type=int, default=6)
ap.add_argument("--bias", type=float, default=0.2)
ap.add_argument("--m", type=int, default=4)
ap.add_argument("--nvec", type=int, default=8)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

# a random many-body basis (the reference's random_basis is out of scope: a
# Gumbel-top-N draw over 128 single-particle states with weights exp(-bias·k))
rng = np.random.default_rng(0)
n_sp = 128
w = np.exp(-a.bias * np.arange(1, n_sp + 1))
occ = np.zeros((0, a.particles), np.uint16)
while occ.shape[0] < a.n:
    keys = np.log(rng.random((2 * a.n, n_sp))) / w
    pick = np.sort(np.argpartition(-keys, a.particles, axis=1)[:, :a.particles] + 1, axis=1).astype(np.uint16)
    occ = np.unique(np.concatenate([occ, pick]), axis=0)
occ = occ[rng.permutation(occ.shape[0])[:a.n]]
lo = np.zeros(a.n, np.uint64)
for q in range(a.particles):
    sel = occ[:, q] <= 64
    lo[sel] |= np.left_shift(np.uint64(1), (occ[sel, q] - 1).astype(np.uint64))
basis = b2.BasisArrays(occ, lo, n_sp)
t0 = time.perf_counter()
grouped, orbs = b2.group_orbitals(basis, group_bits=8)
rank = b2.InteractionRank()
tiles = b2.enumerate_tiles(orbs, orbs, rank)
t_setup = time.perf_counter() - t0
c = b2.random_coefficients(a.nvec, a.n, seed=1)
H = b2.HalfTiles.from_basis(grouped, rank=rank)  # only to count the stored pairs
pairs = 2 * int(H.meta["stored_entries"])  # full pair set ≈ 2 × block-half (diagonal blocks counted twice)

def call():
    return b2.contract_observables(tiles, orbs, grouped, rank, b2.ObservablesInput(c=c, m_ops=a.m, seed=3))

call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.reps):
    out = call()
dt = (time.perf_counter() - t0) / a.reps
t0 = time.perf_counter()
ref = b2.contract_oracle(tiles, orbs, grouped, rank, b2.ObservablesInput(c=c, m_ops=a.m, seed=3))
dt_oracle = time.perf_counter() - t0
print(json.dumps({"n": a.n, "orbitals": len(orbs), "tiles": len(tiles), "n_vec": a.nvec, "m_ops": a.m,
                  "approx_pairs": pairs, "setup_s": round(t_setup, 3), "ms_per_call": round(dt * 1e3, 3),
                  "mpairs_per_s": round(pairs / dt / 1e6, 1),
                  "mpair_ops_per_s": round(pairs * a.m / dt / 1e6, 1),
                  "oracle_ms": round(dt_oracle * 1e3, 3),
                  "max_abs_diff_vs_oracle": float(np.abs(out.astype(np.float64) - ref).max())}))
