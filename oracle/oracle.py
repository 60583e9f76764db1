"""CPU oracle for the half-stored symmetric SpMM  Y = U·X + U_offᵀ·X.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2110_10765_b200/`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs use it, as the checker.

It is a plain-numpy restatement of the reference package ``cimotifs``
(``/root/reference/pkg/src/cimotifs``) for everything the hot path touches:

* the value hashes ``_mix64_np``/``_to_unit_np``/``_h_values_np``/
  ``_op_values_np`` (pipeline.py:235-263) — pinned bit-exact against the
  reference's own outputs in ``tests/golden/hash_kat.json``;
* the storage walk that recovers (i, j, value) from a ``SparseSkeleton``
  (tiles + per-(tile,row) segments, pipeline.py:96-116 and :319-330) —
  pinned against reference-built skeletons in ``tests/golden/*.npz``;
* the block-half convention (tiles R ≤ C, diagonal tiles in
  full, ``Y = U·X + U_offᵀ·X``);
* the contraction oracle ``contract_oracle`` (pipeline.py:573-589), used as
  the VMV bridge ``diag(Xᵀ O X)`` to the reference's ``contract_observables``;
* the reference's tolerance envelope ``2⁻²⁰·terms·max|x|·max|y|``
  (reduce.py:65, :213-219; test_pipeline.py:33-36).

The SpMM itself has no reference implementation (SPEC.md:388 lists SpMV as a
non-goal); its f64 arithmetic here is the definition  Y[R] += T·X[C],
Y[C] += Tᵀ·X[R] (R < C)  evaluated tile by tile in float64.
"""

from __future__ import annotations

import hashlib

import numpy as np

BLOCK = 64
TOLERANCE_EPS = 2.0 ** -20  # reduce.py:65

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)  # pipeline.py:199
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)  # pipeline.py:200
_MIX2 = np.uint64(0x94D049BB133111EB)  # pipeline.py:201


# ----------------------------------------------------------------------------
# value hashes (pipeline.py:235-263)
# ----------------------------------------------------------------------------

def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer after +golden (pipeline.py:235-240)."""
    with np.errstate(over="ignore"):
        z = np.asarray(z).astype(np.uint64) + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def to_unit(u: np.ndarray) -> np.ndarray:
    """Top 53 bits → [0,1) → [-1,1) in float64 (pipeline.py:243-244)."""
    return (u >> np.uint64(11)) * (2.0 ** -53) * 2.0 - 1.0


def h_values(i, j, seed: int) -> np.ndarray:
    """H_ij = f32(h(i XOR j; seed)) (pipeline.py:247-249)."""
    u = mix64(np.asarray(i).astype(np.uint64) ^ np.asarray(j).astype(np.uint64))
    return to_unit(mix64(u ^ np.uint64(seed))).astype(np.float32)


def op_values(i, j, k: int, op_code: int, seed: int) -> np.ndarray:
    """O_ij(k): identity (op_code 0) or symmetric hash (pipeline.py:252-263)."""
    i = np.asarray(i)
    j = np.asarray(j)
    if op_code == 0:
        return (i == j).astype(np.float32)
    lo = np.minimum(i, j).astype(np.uint64)
    hi = np.maximum(i, j).astype(np.uint64)
    with np.errstate(over="ignore"):
        u = mix64(lo + _GOLDEN * hi)
        u = mix64(u ^ (np.uint64(k) + np.uint64(1)) * _MIX1)
    return to_unit(mix64(u ^ np.uint64(seed))).astype(np.float32)


# ----------------------------------------------------------------------------
# storage: reference skeleton → COO → block-half tiles
# ----------------------------------------------------------------------------

def skeleton_coo(tiles, orbitals, segments_counts, segments_offsets, colind, values):
    """(i, j, v) of every stored entry of a reference SparseSkeleton.

    Walks tiles in order; each tile contributes one segment per row of its row
    orbital, whose row is ``orbital.start + local_row`` (pipeline.py:319-330,
    the same walk as test_pipeline.py:160-172).
    """
    start = {o.id: o.start for o in orbitals}
    size = {o.id: o.stop - o.start for o in orbitals}
    rows = []
    for t in tiles:
        rows.append(start[t.row_orbital] + np.arange(size[t.row_orbital], dtype=np.int64))
    seg_row = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    counts = np.asarray(segments_counts, dtype=np.int64)
    i = np.repeat(seg_row, counts)
    return i, np.asarray(colind, dtype=np.int64), np.asarray(values, dtype=np.float32)


def coo_to_half_tiles(n: int, i, j, v, dtype=np.float32):
    """Block-half 64-tiles from a full symmetric COO.

    Keeps entries with ⌊i/64⌋ ≤ ⌊j/64⌋ (diagonal tiles keep both triangles),
    returns (tile_rc int32 (T,2) sorted by (R,C), dense row-major tiles (T,64,64)).
    Duplicate (i,j) entries are summed, like a COO→dense conversion.
    """
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    v = np.asarray(v)
    R = i // BLOCK
    C = j // BLOCK
    keep = R <= C
    i, j, v, R, C = i[keep], j[keep], v[keep], R[keep], C[keep]
    nb = (n + BLOCK - 1) // BLOCK
    key = R * nb + C
    uniq, inv = np.unique(key, return_inverse=True)
    tiles = np.zeros((uniq.size, BLOCK, BLOCK), dtype=np.float64)
    np.add.at(tiles, (inv, i % BLOCK, j % BLOCK), v.astype(np.float64))
    rc = np.stack([uniq // nb, uniq % nb], axis=1).astype(np.int32)
    return rc, tiles.astype(dtype)


def half_tiles_to_coo(n: int, tile_rc, tiles):
    """Full symmetric COO (i, j, v) of the matrix A described by half tiles."""
    rc = np.asarray(tile_rc, dtype=np.int64)
    t, a, b = np.nonzero(tiles)
    i = rc[t, 0] * BLOCK + a
    j = rc[t, 1] * BLOCK + b
    v = tiles[t, a, b]
    off = rc[t, 0] < rc[t, 1]
    ii = np.concatenate([i, j[off]])
    jj = np.concatenate([j, i[off]])
    vv = np.concatenate([v, v[off]])
    return ii, jj, vv


def synthetic_dense_tiles(n: int, tile_rc, seed: int = 0, kind: int = 0, op_k: int = 0, dtype=np.float32):
    """Host twin of cim_fill_synthetic_values: tile values h(i XOR j; seed)
    (kind 0), O_ij(op_k; seed) (kind 1) or δ_ij (kind 2); 0 outside [0,n)."""
    rc = np.asarray(tile_rc, dtype=np.int64)
    a = np.arange(BLOCK, dtype=np.int64)
    i = rc[:, 0, None, None] * BLOCK + a[None, :, None]
    j = rc[:, 1, None, None] * BLOCK + a[None, None, :]
    i, j = np.broadcast_arrays(i, j)
    if kind == 0:
        val = h_values(i, j, seed)
    elif kind == 1:
        val = op_values(i, j, op_k, 1, seed)
    else:
        val = op_values(i, j, 0, 0, seed)
    val = np.where((i < n) & (j < n), val, np.float32(0))
    return val.astype(dtype)


def synthetic_sparse_tiles(n: int, tile_rc, fill: float, fill_seed: int, value_seed: int = 0,
                           dtype=np.float32) -> np.ndarray:
    """Host twin of HalfTiles.synthetic_sparse (cim_sparse_count_rows /
    cim_sparse_fill_entries): dense row-major (T,64,64) tiles holding h(i XOR j;
    value_seed) where mix64(mix64(min ⊕ 0x5bd1e995·max) ⊕ fill_seed) < fill·2⁶⁴
    and i, j < n, else 0.  (Test infrastructure; the keep rule is the
    generator's own, the values the reference hash, pipeline.py:216-222.)"""
    rc = np.asarray(tile_rc, dtype=np.int64)
    a = np.arange(BLOCK, dtype=np.int64)
    i = rc[:, 0, None, None] * BLOCK + a[None, :, None]
    j = rc[:, 1, None, None] * BLOCK + a[None, None, :]
    i, j = np.broadcast_arrays(i, j)
    lo = np.minimum(i, j).astype(np.uint64)
    hi = np.maximum(i, j).astype(np.uint64)
    with np.errstate(over="ignore"):
        key = mix64(mix64(lo ^ (hi * np.uint64(0x5BD1E995))) ^ np.uint64(fill_seed))
    thresh = np.uint64(min(int(fill * 18446744073709551616.0), (1 << 64) - 1)) if fill < 1.0 else None
    keep = (i < n) & (j < n) & ((key < thresh) if thresh is not None else True)
    val = np.where(keep, h_values(i, j, value_seed), np.float32(0))
    return val.astype(dtype)


# ----------------------------------------------------------------------------
# the SpMM definition in float64
# ----------------------------------------------------------------------------

def sym_spmm(n: int, tile_rc, tiles, X, chunk: int = 4096) -> np.ndarray:
    """Y = U·X + U_offᵀ·X in float64 (SURVEY.md §8 convention).

    X: (n, k) (any float dtype, promoted to f64).  tiles: (T, 64, 64) row-major.
    """
    rc = np.asarray(tile_rc, dtype=np.int64)
    X = np.asarray(X, dtype=np.float64)
    k = X.shape[1]
    nb = (n + BLOCK - 1) // BLOCK
    Xp = np.zeros((nb * BLOCK, k))
    Xp[:n] = X
    Xb = Xp.reshape(nb, BLOCK, k)
    Yb = np.zeros_like(Xb)
    for s in range(0, rc.shape[0], chunk):
        r = rc[s:s + chunk, 0]
        c = rc[s:s + chunk, 1]
        T = np.asarray(tiles[s:s + chunk], dtype=np.float64)
        np.add.at(Yb, r, np.einsum("tab,tbv->tav", T, Xb[c]))
        off = r < c
        if off.any():
            np.add.at(Yb, c[off], np.einsum("tab,tav->tbv", T[off], Xb[r[off]]))
    return Yb.reshape(-1, k)[:n]


def frobenius_full(tile_rc, tiles) -> float:
    """‖A‖_F of the full matrix: ‖A‖² = 2‖U_off‖² + ‖U_diag‖²."""
    rc = np.asarray(tile_rc)
    sq = (np.asarray(tiles, dtype=np.float64) ** 2).sum(axis=(1, 2))
    w = np.where(rc[:, 0] < rc[:, 1], 2.0, 1.0)
    return float(np.sqrt((w * sq).sum()))


def abs_product(n: int, tile_rc, tiles, X) -> np.ndarray:
    """(|A|·|X|) for the componentwise error bound."""
    return sym_spmm(n, tile_rc, np.abs(np.asarray(tiles, dtype=np.float64)), np.abs(np.asarray(X, np.float64)))


def normwise_error(Y, Y_ref, A_fro: float, X) -> float:
    """‖ΔY‖_F / (‖A‖_F·‖X‖_F) — the north-star gate (≤1e-5 f32, ≤1e-12 f64)."""
    d = np.asarray(Y, np.float64) - np.asarray(Y_ref, np.float64)
    return float(np.linalg.norm(d) / (A_fro * np.linalg.norm(np.asarray(X, np.float64)) + 1e-300))


def componentwise_ok(Y, Y_ref, absAX, max_row_nnz: int, unit_roundoff: float) -> bool:
    """|ΔY_iv| ≤ c·u·(|A||X|)_iv with c = max row nnz (+2 for the final adds)."""
    d = np.abs(np.asarray(Y, np.float64) - np.asarray(Y_ref, np.float64))
    return bool(np.all(d <= (max_row_nnz + 2) * unit_roundoff * absAX + 1e-300))


# ----------------------------------------------------------------------------
# contraction bridge (pipeline.py:573-589) and tolerance (reduce.py:213-219)
# ----------------------------------------------------------------------------

def contract_vmv(c, pairs_i, pairs_j, m_ops: int, op_code: int, seed: int) -> np.ndarray:
    """a[v,k] = Σ_(i,j) c[v,i]·O_ij(k)·c[v,j] in float64 (pipeline.py:573-589)."""
    c = np.asarray(c, dtype=np.float64)
    out = np.zeros((c.shape[0], m_ops))
    for k in range(m_ops):
        o = op_values(pairs_i, pairs_j, k, op_code, seed).astype(np.float64)
        for v in range(c.shape[0]):
            out[v, k] = np.sum(c[v, pairs_i] * o * c[v, pairs_j])
    return out


def occ_diff(a, b) -> int:
    """Lockstep walk of two sorted occupation lists: 2·max(#only-in-a,
    #only-in-b) (_occ_diff, sparsity.py:132-151)."""
    i1 = i2 = d1 = d2 = 0
    while i1 < len(a) and i2 < len(b):
        if a[i1] == b[i2]:
            i1 += 1
            i2 += 1
        elif a[i1] < b[i2]:
            d1 += 1
            i1 += 1
        else:
            d2 += 1
            i2 += 1
    return 2 * max(d1, d2)


def scan_serial(x) -> np.ndarray:
    """Exclusive prefix sum, sequential (scan_serial, scan.py:131-139): y[i] =
    Σ_(j<i) x[j] in int64 (wrapping like the reference's njit int64 adds)."""
    x = np.ascontiguousarray(x, dtype=np.int64)
    y = np.empty_like(x)
    s = np.int64(0)
    if x.size <= 4096:
        for i in range(x.size):
            y[i] = s
            s = np.int64(s + x[i])
        return y
    with np.errstate(over="ignore"):
        c = np.cumsum(x, dtype=np.int64)  # same wrapping integer sums, vectorised
    y[0] = 0
    y[1:] = c[:-1]
    return y


def counts_to_offsets(counts):
    """(offsets, total) of a CountsAndOffsets (scan.py:45-65) built from counts."""
    off = scan_serial(counts)
    total = int(off[-1] + np.int64(counts[-1])) if off.size else 0
    return off, total


def contraction_tolerance(c, n_pairs: int) -> float:
    """2⁻²⁰·n_pairs·max|c|² (test_pipeline.py:33-36)."""
    return TOLERANCE_EPS * max(n_pairs, 1) * float(np.abs(c).max()) ** 2


def digest(*parts) -> str:
    """16-hex sha256 with '|' separators (_util.py:65-76)."""
    h = hashlib.sha256()
    for p in parts:
        if isinstance(p, np.ndarray):
            h.update(np.ascontiguousarray(p).tobytes())
        elif isinstance(p, bytes):
            h.update(p)
        else:
            h.update(str(p).encode())
        h.update(b"|")
    return h.hexdigest()[:16]


def pair_set_digest(i, j) -> str:
    """Digest of the sorted (i, j) pair set (structure parity, bit-exact)."""
    i = np.asarray(i, np.int64)
    j = np.asarray(j, np.int64)
    order = np.lexsort((j, i))
    return digest(i[order], j[order])
