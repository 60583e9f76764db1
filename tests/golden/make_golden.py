"""Generate the golden fixtures that pin the oracle to the REAL reference.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package ``cimotifs`` from
/root/reference/pkg/src and records, with the reference's own functions:

* hash_kat.json       — _h_values_np / _h_value / _op_values_np known answers
                        (pipeline.py:216-263), incl. the SURVEY.md §8(a) KATs;
* skel_small.npz      — test_pipeline.small_problem (n=192, seed=13, gb=8,
                        test_pipeline.py:39-44): full reference COO of the
                        built skeleton, its pair-set digest, a coefficient
                        block, contract_observables(array_clause) and
                        contract_oracle results, and Y_ref = A·X (float64,
                        scipy, computed here from the reference COO);
* skel_n1024.npz      — n=1024, 6 particles, bias 0.2, gb 8, seed 0: a
                        medium reference skeleton with the same records;
* skel_identity.npz   — test_acceptance.py:307-321: n=1024, 8 particles,
                        CALIBRATION_BIAS, identity operator with ±n^-½ sign
                        vectors (contraction exactly 1 ± 2⁻²⁰).

Each skeleton fixture also carries its grouped basis (occupation lists and
packed words) so the GPU construction (HalfTiles.from_basis) can be checked
against the reference's own build_skeleton output, and basis_<name>.txt is
the same basis in sampled order written by the reference's save_basis
(mbstate.py:242-246; `--basis-files` regenerates only these).

* contraction_cases.npz — the bases of the reference's TestContraction
                        problems (test_pipeline.py:244-305: small_problem
                        n=64 / n=128 and the n=256 identity basis) as
                        random_basis produced them (ungrouped occupation
                        lists and words), the reference's grouping and tile
                        list for each, and the reference's own outputs of
                        contract_observables (every strategy, forward and
                        transposed) and contract_oracle on the tests' inputs,
                        so the test bodies rerun against the GPU package with
                        only the import swapped (`--contraction` regenerates
                        only this file).

The GPU box never reads /root/reference: tests load only these files.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, str(REF))

from cimotifs._util import digest  # noqa: E402
from cimotifs.mbstate import CALIBRATION_BIAS, random_basis, save_basis  # noqa: E402
from cimotifs.pipeline import (  # noqa: E402
    ObservablesInput,
    _h_value,
    _h_values_np,
    _op_value,
    _op_values_np,
    _collect_pairs,
    build_skeleton,
    contract_observables,
    contract_oracle,
    enumerate_tiles,
    group_orbitals,
    random_coefficients,
)
from cimotifs.sparsity import InteractionRank, count_pairs  # noqa: E402


def f32bits(x) -> int:
    return int(np.float32(x).view(np.uint32))


def hash_kat():
    rng = np.random.default_rng(123)
    cases = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (12345, 678, 0), (65535, 0, 0),
             (4194303, 4194240, 0), (2 ** 40, 3, 7), (0, 0, 9), (17, 1000, 7)]
    ii = rng.integers(0, 2 ** 40, size=64)
    jj = rng.integers(0, 2 ** 40, size=64)
    ss = rng.integers(0, 2 ** 31, size=64)
    cases += [(int(a), int(b), int(s)) for a, b, s in zip(ii, jj, ss)]
    h = []
    for i, j, s in cases:
        v_np = _h_values_np(np.array([i], np.int64), np.array([j], np.int64), s)[0]
        v_jit = _h_value(i, j, s)
        assert f32bits(v_np) == f32bits(v_jit)
        h.append({"i": i, "j": j, "seed": s, "bits": f32bits(v_np)})
    ops = []
    for (i, j, s), k in zip(cases, range(len(cases))):
        kk = k % 5
        for code in (0, 1):
            v_np = _op_values_np(np.array([i], np.int64), np.array([j], np.int64), kk, code, s)[0]
            v_jit = _op_value(i, j, kk, code, s)
            assert f32bits(v_np) == f32bits(v_jit)
            ops.append({"i": i, "j": j, "k": kk, "op_code": code, "seed": s, "bits": f32bits(v_np)})
    ops.append({"i": 3, "j": 5, "k": 0, "op_code": 1, "seed": 4,
                "bits": f32bits(_op_values_np(np.array([3]), np.array([5]), 0, 1, 4)[0])})
    ops.append({"i": 7, "j": 7, "k": 2, "op_code": 1, "seed": 5,
                "bits": f32bits(_op_values_np(np.array([7]), np.array([7]), 2, 1, 5)[0])})
    (OUT / "hash_kat.json").write_text(json.dumps({"h": h, "op": ops}, indent=0))
    print(f"hash_kat.json: {len(h)} h, {len(ops)} op")


def skeleton_fixture(name, n, particles, bias, group_bits, seed, n_vec, m_ops, op_kind, coeff_kind,
                     coeff_seed, op_seed, value_seed=0):
    basis = random_basis(n, particles, bias=bias, seed=seed)
    grouped, orbs = group_orbitals(basis, group_bits=group_bits)
    rank = InteractionRank()
    tiles = enumerate_tiles(orbs, orbs, rank)
    sk = build_skeleton(tiles, orbs, grouped, rank, seed=value_seed)
    whole = count_pairs(grouped, grouped, rank, "combined").total
    assert sk.nnz == whole
    # reference COO through the reference's own pair walk (pipeline.py:428-458)
    pi, pj = _collect_pairs(tiles, orbs, grouped, rank)
    # values in skeleton order: rows recovered from segments
    start = {o.id: o.start for o in orbs}
    size = {o.id: o.size for o in orbs}
    seg_row = np.concatenate([start[t.row_orbital] + np.arange(size[t.row_orbital]) for t in sk.tiles])
    si = np.repeat(seg_row, sk.segments.counts)
    assert np.array_equal(si, pi) and np.array_equal(sk.colind, pj)
    A = sp.coo_matrix((sk.values.astype(np.float64), (si, sk.colind)), shape=(n, n)).tocsr()
    assert abs(A - A.T).max() == 0.0, "reference matrix must be exactly symmetric"
    c = random_coefficients(n_vec, n, seed=coeff_seed, kind=coeff_kind)
    X = c.T.copy()  # (n, n_vec)
    Y_ref = A @ X.astype(np.float64)
    inputs = ObservablesInput(c=c, m_ops=m_ops, op_kind=op_kind, seed=op_seed)
    acc = contract_observables(tiles, orbs, grouped, rank, inputs, "array_clause").copy()
    acc_t = contract_observables(tiles, orbs, grouped, rank,
                                 ObservablesInput(c=c, m_ops=m_ops, op_kind=op_kind, seed=op_seed),
                                 "array_clause", transpose=True).copy()
    acc_oracle = contract_oracle(tiles, orbs, grouped, rank, inputs)
    order = np.lexsort((pj, pi))
    pair_digest = digest(pi[order], pj[order])
    np.savez_compressed(
        OUT / name,
        n=n, i=si.astype(np.int32), j=sk.colind.astype(np.int32), v=sk.values,
        seg_counts=sk.segments.counts, seg_offsets=sk.segments.offsets,
        tiles_rc=np.array([(t.row_orbital, t.col_orbital, t.cnt, t.offset) for t in sk.tiles], np.int64),
        orb=np.array([(o.id, o.start, o.stop) for o in orbs], np.int64),
        pair_digest=np.array(pair_digest), nnz=sk.nnz, whole_pairs=whole,
        X=X, Y_ref=Y_ref, accum=acc, accum_transpose=acc_t, accum_oracle=acc_oracle,
        m_ops=m_ops, op_kind=np.array(op_kind), op_seed=op_seed,
        diag_value_bits=f32bits(_h_value(0, 0, value_seed)), value_seed=value_seed,
        # the grouped basis itself (mbstate.py Basis arrays), for the GPU
        # construction path: occupation lists (n, N) uint16, packed words
        basis_occ=grouped.occ_mat.astype(np.uint16), basis_bits_lo=grouped.bits_lo.astype(np.uint64),
        basis_n_sp=grouped.n_sp, rank_threshold=rank.threshold,
    )
    print(f"{name}: n={n} nnz={sk.nnz} tiles={len(tiles)} orbitals={len(orbs)} digest={pair_digest}")


def basis_files():
    """The fixtures' bases as reference basis files (save_basis, mbstate.py:242-246),
    in sampled (ungrouped) order, plus the grouping they were built with."""
    meta = {}
    for name, n, particles, bias, group_bits, seed in (
            ("skel_small", 192, 6, 0.2, 8, 13), ("skel_n1024", 1024, 6, 0.2, 8, 0),
            ("skel_identity", 1024, 8, CALIBRATION_BIAS, 8, 0)):
        basis = random_basis(n, particles, bias=bias, seed=seed)
        save_basis(basis, OUT / f"basis_{name}.txt")
        meta[name] = {"group_bits": group_bits, "n": n}
    (OUT / "basis_files.json").write_text(json.dumps(meta, indent=1))
    print("basis files:", sorted(meta))


def contraction_cases():
    """The reference TestContraction problems and outputs (test_pipeline.py:39-44, :244-305)."""
    out = {}

    def put(name, basis, group_bits):
        grouped, orbs = group_orbitals(basis, group_bits=group_bits)
        rank = InteractionRank()
        tiles = enumerate_tiles(orbs, orbs, rank)
        out[f"{name}_occ"] = basis.occ_mat.astype(np.uint16)
        out[f"{name}_bits_lo"] = basis.bits_lo.astype(np.uint64)
        out[f"{name}_n_sp"] = basis.n_sp
        out[f"{name}_group_bits"] = group_bits
        out[f"{name}_grouped_occ"] = grouped.occ_mat.astype(np.uint16)
        out[f"{name}_orb"] = np.array([(o.id, o.start, o.stop, o.key) for o in orbs], np.int64)
        out[f"{name}_tiles"] = np.array([(t.row_orbital, t.col_orbital) for t in tiles], np.int64)
        out[f"{name}_n_pairs"] = count_pairs(grouped, grouped, rank).total
        return grouped, orbs, tiles, rank

    put("p64", random_basis(64, 6, bias=0.2, seed=13), 8)
    g, o, t, r = put("p128", random_basis(128, 6, bias=0.2, seed=13), 8)
    put("p256", random_basis(256, 8, bias=0.1, seed=17), 8)
    # test_strategies_match_oracle inputs and the reference's outputs
    c = random_coefficients(4, 128, seed=2)
    for strat in ("array_clause", "atomic_per_element", "generated_scalars"):
        out[f"strat_{strat}"] = contract_observables(t, o, g, r, ObservablesInput(c=c, m_ops=3, seed=4), strat).copy()
    out["strat_oracle"] = contract_oracle(t, o, g, r, ObservablesInput(c=c, m_ops=3, seed=4))
    # test_hermitian_symmetry
    c3 = random_coefficients(4, 128, seed=3)
    out["herm_fwd"] = contract_observables(t, o, g, r, ObservablesInput(c=c3, m_ops=2, seed=6)).copy()
    out["herm_rev"] = contract_observables(t, o, g, r, ObservablesInput(c=c3, m_ops=2, seed=6), transpose=True).copy()
    np.savez_compressed(OUT / "contraction_cases.npz", **out)
    print("contraction_cases.npz:", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    if sys.argv[1:] == ["--contraction"]:
        contraction_cases()
        sys.exit(0)
    if sys.argv[1:] == ["--basis-files"]:
        basis_files()
        sys.exit(0)
    hash_kat()
    basis_files()
    contraction_cases()
    skeleton_fixture("skel_small.npz", n=192, particles=6, bias=0.2, group_bits=8, seed=13,
                     n_vec=4, m_ops=3, op_kind="symmetric_hash", coeff_kind="gauss",
                     coeff_seed=2, op_seed=4)
    skeleton_fixture("skel_n1024.npz", n=1024, particles=6, bias=0.2, group_bits=8, seed=0,
                     n_vec=8, m_ops=2, op_kind="symmetric_hash", coeff_kind="gauss",
                     coeff_seed=0, op_seed=6)
    skeleton_fixture("skel_identity.npz", n=1024, particles=8, bias=CALIBRATION_BIAS, group_bits=8,
                     seed=0, n_vec=8, m_ops=4, op_kind="identity", coeff_kind="signs",
                     coeff_seed=1, op_seed=5)
