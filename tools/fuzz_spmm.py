"""Robustness sweep (not part of the suite): N seeded random configurations
through the public API — dtype, layout, n, density, dense / sparse mix via
from_coo, k (padded widths too), unit size, CSR forms, deterministic mode,
accumulate, (k, n) input, the host-buffer pipeline and the sharded
operator at world 1 — each against the f64 oracle.  Prints a summary
line; exits 1 on the first failure with its seed.

    python tools/fuzz_spmm.py [N] [first_seed] [max_n]
"""
import os, sys, traceback
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2110_10765_b200 as pkg
from oracle import oracle

N = int(sys.argv[1]) if len(sys.argv) > 1 else 500
S0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
N_MAX = int(sys.argv[3]) if len(sys.argv) > 3 else 5000  # larger n: sparser patterns (the oracle is numpy)


def one(seed):
    rng = np.random.default_rng(seed)
    dtype = torch.float32 if rng.random() < 0.6 else torch.float64
    layout = "tc" if rng.random() < 0.5 else "frag"
    n = int(rng.integers(1, N_MAX))
    nb = (n + 63) // 64
    k = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 20, 24, 32, 40, 48, 56, 64]))
    p = float(rng.choice([0.0, 0.02, 0.1, 0.4, 1.0] if n <= 5000 else [0.0, 0.002, 0.01]))
    rc = pkg.synthetic_pattern(nb, p, seed=seed)
    # per-tile fill → from_coo decides dense / sparse per tile
    ii, jj = [], []
    for R, C in rc:
        f = float(rng.choice([0.005, 0.03, 0.15, 0.6, 1.0]))
        m = rng.random((64, 64)) < f
        if R == C:
            m = m | m.T
        a, b = np.nonzero(m)
        ii.append(R * 64 + a)
        jj.append(C * 64 + b)
    if not ii:
        ii, jj = [np.array([0])], [np.array([0])]
    i, j = np.concatenate(ii), np.concatenate(jj)
    ok = (i < n) & (j < n)
    key = np.unique(np.minimum(i[ok], j[ok]) * n + np.maximum(i[ok], j[ok]))
    lo, hi = key // n, key % n
    if lo.size == 0:
        lo, hi = np.array([0]), np.array([0])
    I = np.concatenate([lo, hi[lo != hi]])
    J = np.concatenate([hi, lo[lo != hi]])
    V = oracle.h_values(I, J, seed).astype(np.float64)
    H = pkg.HalfTiles.from_coo(n, I, J, V, dtype=dtype, layout=layout, dense_fill=float(rng.choice([0.1, 0.5, 2.0, 0.0])))
    if H.sparse is not None and rng.random() < 0.5:
        H.use_symmetric_csr(bool(rng.random() < 0.5))
    rcd, tiles = H.export_dense()
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(seed), dtype=dtype)
    det = bool(rng.random() < 0.15)
    kn = bool(rng.random() < 0.3)
    Xin = np.ascontiguousarray(X.numpy().T) if kn else X.cuda()
    Y = pkg.sym_spmm(H, Xin, deterministic=det, layout="kn" if kn else "nk")
    Y = Y.T if kn else Y.cpu().numpy()
    Y_ref = oracle.sym_spmm(n, rcd, tiles.astype(np.float64), X.numpy().astype(np.float64))
    err = oracle.normwise_error(Y, Y_ref, max(oracle.frobenius_full(rcd, tiles.astype(np.float64)), 1e-300), X.numpy())
    gate = 1e-5 if dtype == torch.float32 else 1e-12
    if not err <= gate:
        raise AssertionError(f"seed {seed}: err {err:.3e} dtype={dtype} layout={layout} n={n} k={k} p={p} det={det} kn={kn}")
    if not det and rng.random() < 0.25 and pkg.padded_k(dtype, k, layout) == k:  # host-buffer pipeline
        Yb = pkg.sym_spmm_host_batch(H, [X.pin_memory(), X])
        for yb in Yb:
            e = oracle.normwise_error(yb.numpy(), Y_ref, max(oracle.frobenius_full(rcd, tiles.astype(np.float64)),
                                                             1e-300), X.numpy())
            if not e <= gate:
                raise AssertionError(f"seed {seed}: host batch err {e:.3e}")
    if not det and rng.random() < 0.25:  # the sharded operator at world 1 (rows padded to n_pad)
        S = pkg.ShardedSymSpmm(n, k, dtype, torch.device("cuda"), H_local=H)
        Xs = torch.zeros((S.rows_per_rank, k), dtype=dtype)
        Xs[:n] = X
        Ys = S.apply(Xs.cuda()).cpu().numpy()
        e = oracle.normwise_error(Ys[:n], Y_ref, max(oracle.frobenius_full(rcd, tiles.astype(np.float64)), 1e-300),
                                  X.numpy())
        if not e <= gate or np.any(Ys[n:] != 0):
            raise AssertionError(f"seed {seed}: sharded world-1 err {e:.3e}")
    if rng.random() < 0.2:  # accumulate on top
        out = torch.from_numpy(np.ascontiguousarray(Y)).to(dtype).cuda()
        pkg.sym_spmm(H, X.cuda(), out=out, accumulate=True, layout="nk")
        err2 = np.abs(out.cpu().numpy() - 2 * Y_ref).max() / max(np.abs(Y_ref).max(), 1e-300)
        if not err2 <= 10 * gate * max(1, np.sqrt(k)):
            raise AssertionError(f"seed {seed}: accumulate err {err2:.3e}")


fails = 0
for s in range(S0, S0 + N):
    try:
        one(s)
    except Exception:
        traceback.print_exc()
        print(f"FAIL seed {s}")
        fails += 1
        if fails >= 3:
            break
print(f"fuzz: {N} configurations from seed {S0}, {fails} failures")
sys.exit(1 if fails else 0)
