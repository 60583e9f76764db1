"""The observables contraction (contract_observables, pipeline.py:534-570) on
the GPU: the fused tile walk (cim_contract_observables, O_ij(k) hashed on the
fly) against the materialised composition (fill O_k + sym_spmm + dot).

    python tools/bench_contract.py [--n 65536] [--p 0.01] [--reps 10]

The pattern is BASELINE C1's (n = 65,536, all diagonal tiles + Bernoulli-0.01
upper tiles, fully dense: 47.2 M pairs of the full symmetric pattern).  Rates
are pairs/s of the full pattern, and pair·operator/s.  The reference's CPU
rate on its own pair stream is quoted from SURVEY.md §8(a) (8 threads,
n_vec = 8, m_ops = 1: array_clause 58.3, generated_scalars 213.1 Mpair/s).
"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as b2
from paper_2110_10765_b200.observables import contract_materialized

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--p", type=float, default=0.01)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--cases", default="8x1,8x16,16x16")
a = ap.parse_args()

nb = (a.n + 63) // 64
rc = b2.synthetic_pattern(nb, a.p, seed=0)
H = b2.HalfTiles.synthetic(a.n, tile_rc=rc)  # nonzero everywhere: the full tiles are the pattern
n_diag = int((rc[:, 0] == rc[:, 1]).sum())
pairs = (2 * (len(rc) - n_diag) + n_diag) * 4096
out = []
for case in a.cases.split(","):
    nv, m = (int(x) for x in case.split("x"))
    c = b2.random_coefficients(nv, a.n, seed=1)
    inp = b2.ObservablesInput(c=c, m_ops=m, seed=3)
    row = {"n_vec": nv, "m_ops": m, "pairs": pairs}
    for name, fn in (("fused", lambda: b2.contract_pattern(H, inp)),
                     ("materialized", lambda: contract_materialized(H, inp))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        row[name] = {"ms": round(ms, 3), "Mpair_per_s": round(pairs / ms / 1e3, 1),
                     "Gpair_op_per_s": round(pairs * m / ms / 1e6, 1)}
    d = np.abs(b2.contract_pattern(H, inp).astype(np.float64) - contract_materialized(H, inp)).max()
    row["max_abs_diff"] = float(d)
    out.append(row)
    print(json.dumps(row), flush=True)
