"""The reference's observables API, on the GPU.

``contract_observables`` computes, like pipeline.py:534-570,

    accum[v, k] = Σ_(i,j) c[v,i] · O_ij(k) · c[v,j]      (= c_vᵀ O_k c_v)

over the interacting pairs (i, j) of a stored pattern.  Where the reference
re-walks every tile's pairs on the CPU, here the pattern is a ``HalfTiles``
(its nonzero entries mark the pairs, e.g. ``HalfTiles.from_skeleton`` of a
reference skeleton with unit values) and ``cim_contract_observables`` walks
its tiles once, computing O_ij(k) on the fly (bit-exact to
``_op_values_np``) and reducing c[v,i]·O_ij(k)·c[v,j] per (v, k) in
registers — no operator is materialised (csrc/contract.cu).
``contract_materialized`` keeps the composition through ``sym_spmm`` (O_k
filled on the pattern by ``cim_fill_masked_values``) as an independent
cross-check.

``ObservablesInput``, ``random_coefficients``, ``STRATEGIES`` and
``OP_KINDS`` keep the reference's names and validation (pipeline.py:64,
:384-425; reduce.py:62) so reference callers switch by changing an import.
The strategy names are accepted for compatibility; on the GPU the merge
discipline is the kernel's (register/shared-memory reduction + red.global).

Two entry points:

* ``contract_observables(tiles, orbitals, basis, rank, inputs, strategy,
  workers, transpose)`` and ``contract_oracle(tiles, orbitals, basis, rank,
  inputs)`` — the reference's exact signatures (pipeline.py:534-589): the
  pair set is the reference's own (each orbital Tile re-walked with the
  count predicate, _collect_pairs :428-458), evaluated on the device by
  ``cim_contract_tiles`` — a reference caller switches by changing the
  import.  ``Orbital``, ``Tile``, ``InteractionRank``, ``group_orbitals`` and
  ``enumerate_tiles`` mirror the reference types and host helpers that build
  those arguments (pipeline.py:68-192, sparsity.py:49-60).
* ``contract_pattern(pattern, inputs, ...)`` — the same contraction over a
  stored ``HalfTiles`` pattern (``cim_contract_observables``), the fast path
  when the pattern is already on the device.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import CIM_ACCUMULATE, CIM_CONTRACT_EXACT_F64, check, lib
from .halftiles import LAYOUTS, HalfTiles, _dtype_code
from .spmm import sym_spmm

STRATEGIES = ("array_clause", "atomic_per_element", "generated_scalars")  # reduce.py:62
OP_KINDS = ("symmetric_hash", "identity")  # pipeline.py:64
_OP_CODES = {"identity": 2, "symmetric_hash": 1}  # C-ABI value kinds


@dataclass
class ObservablesInput:
    """Eigenvector stubs, operator kind, and the flat accumulator a(1..n_vec*m)
    (pipeline.py:384-406)."""

    c: np.ndarray  # (n_vec, n) float32
    m_ops: int
    op_kind: str = "symmetric_hash"
    seed: int = 0
    accum: np.ndarray = field(init=False)

    def __post_init__(self):
        self.c = np.ascontiguousarray(self.c, dtype=np.float32)
        if self.c.ndim != 2:
            raise ValueError("coefficients must be (n_vec, n)")
        if self.m_ops < 1:
            raise ValueError("m_ops must be >= 1")
        if self.op_kind not in OP_KINDS:
            raise ValueError(f"unknown op_kind {self.op_kind!r}, expected one of {OP_KINDS}")
        self.accum = np.zeros(self.c.shape[0] * self.m_ops, dtype=np.float32)

    @property
    def n_vec(self) -> int:
        return int(self.c.shape[0])


def random_coefficients(n_vec: int, n: int, seed: int = 0, kind: str = "gauss") -> np.ndarray:
    """Unit-normalised pseudorandom eigenvector stubs (pipeline.py:409-425):
    ``gauss`` rows of N(0,1) normalised to 1; ``signs`` ±n^-½ entries."""
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        c = rng.standard_normal((n_vec, n))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
    elif kind == "signs":
        c = (rng.integers(0, 2, size=(n_vec, n)) * 2 - 1) / np.sqrt(n)
    else:
        raise ValueError(f"unknown coefficient kind {kind!r}")
    return c.astype(np.float32)


def operator_tiles(pattern: HalfTiles, op_kind: str, k: int, seed: int) -> HalfTiles:
    """O_k restricted to the stored pattern, as a HalfTiles on the device."""
    vals = torch.empty_like(pattern.vals)
    stream = torch.cuda.current_stream(pattern.device).cuda_stream
    with torch.cuda.device(pattern.device):
        check(lib().cim_fill_masked_values(
            pattern.tile_rc.data_ptr() if pattern.n_tiles else None, pattern.n_tiles, pattern.n,
            _dtype_code(pattern.dtype), LAYOUTS[pattern.layout], _OP_CODES[op_kind], seed, k,
            pattern.vals.data_ptr() if pattern.n_tiles else None, vals.data_ptr() if pattern.n_tiles else None,
            stream), "cim_fill_masked_values")
    sparse = None
    if pattern.sparse is not None:
        sp = pattern.sparse
        svals = torch.zeros_like(sp.vals)  # tile padding stays zero
        with torch.cuda.device(pattern.device):
            check(lib().cim_fill_sparse_values(sp.descriptor(), pattern.n, _dtype_code(pattern.dtype),
                                               _OP_CODES[op_kind], seed, k, sp.vals.data_ptr() if sp.n_entries else None,
                                               svals.data_ptr() if sp.n_entries else None, stream),
                  "cim_fill_sparse_values")
        sparse = sp.with_values(svals)
    return HalfTiles(n=pattern.n, tile_rc=pattern.tile_rc, units=pattern.units, vals=vals,
                     tile_rc_host=pattern.tile_rc_host, units_host=pattern.units_host, layout=pattern.layout,
                     meta=dict(pattern.meta, op_kind=op_kind, op_k=k, op_seed=seed), sparse=sparse)


def contract_pattern(pattern: HalfTiles, inputs: ObservablesInput, strategy: str = "array_clause",
                     workers: int | None = None, transpose: bool = False) -> np.ndarray:
    """accum[v,k] = Σ over stored pairs (i,j) of c[v,i]·O[i,j,k]·c[v,j].

    Fills ``inputs.accum`` in place and returns its (n_vec, m_ops) view, as
    pipeline.py:569-570.  ``transpose`` walks Aᵀ, which equals A for the
    symmetric pattern (the reference's test_hermitian_symmetry pin,
    test_pipeline.py:278-286); ``workers`` is accepted and ignored (GPU).
    """
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}, expected one of {STRATEGIES}")
    if not isinstance(pattern, HalfTiles):
        raise ValueError("pattern must be a HalfTiles (e.g. HalfTiles.from_skeleton(...)); reference-style "
                         "(tiles, orbitals, basis, rank, inputs) arguments go to contract_observables")
    if inputs.c.shape[1] != pattern.n:
        raise ValueError(f"coefficients cover {inputs.c.shape[1]} states, basis has {pattern.n}")
    dev = pattern.device
    c = torch.from_numpy(inputs.c).to(dev).t().contiguous()  # (n, n_vec) f32
    out = torch.empty((inputs.n_vec, inputs.m_ops), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        check(lib().cim_contract_observables(pattern.descriptor(), c.data_ptr(), inputs.n_vec, inputs.m_ops,
                                             _OP_CODES[inputs.op_kind], inputs.seed, out.data_ptr(), 0, stream),
              "cim_contract_observables")
    inputs.accum[:] = out.cpu().numpy().astype(np.float32).reshape(-1)
    return inputs.accum.reshape(inputs.n_vec, inputs.m_ops)


def contract_materialized(pattern: HalfTiles, inputs: ObservablesInput) -> np.ndarray:
    """The same contraction through materialised operators — O_k filled on the
    pattern, one sym_spmm per operator, then c_vᵀ(O_k c_v) — an independent
    GPU composition the tests cross-check the fused kernel with.  Returns the
    (n_vec, m_ops) f64 result without touching ``inputs.accum``."""
    dev = pattern.device
    X = torch.from_numpy(inputs.c).to(dev, dtype=pattern.dtype).t().contiguous()  # (n, n_vec)
    out = torch.empty((inputs.n_vec, inputs.m_ops), dtype=torch.float64, device=dev)
    for k in range(inputs.m_ops):
        O = operator_tiles(pattern, inputs.op_kind, k, inputs.seed)
        Y = sym_spmm(O, X)
        out[:, k] = (X.to(torch.float64) * Y.to(torch.float64)).sum(dim=0)
    return out.cpu().numpy()


# ----------------------------------------------------------------------------
# The reference's own signature: orbital tiles + basis + rank (pipeline.py)
# ----------------------------------------------------------------------------

MAX_WORKERS_ENV = "CIMOTIFS_MAX_WORKERS"  # _util.py:22


@dataclass(frozen=True)
class Orbital:
    """A contiguous run [start, stop) of basis states sharing a grouping key
    (pipeline.py:68-83)."""

    id: int
    key: object
    start: int
    stop: int

    def __post_init__(self):
        if self.stop <= self.start:
            raise ValueError(f"orbital {self.id} is empty: [{self.start}, {self.stop})")

    @property
    def size(self) -> int:
        return self.stop - self.start


@dataclass
class Tile:
    """A row-orbital/col-orbital pair that may hold interacting state pairs
    (pipeline.py:86-93)."""

    row_orbital: int
    col_orbital: int
    cnt: int = 0
    offset: int = 0


@dataclass(frozen=True)
class InteractionRank:
    """Particle rank d of the operator; pairs connect iff they differ in ≤ 2d
    (sparsity.py:49-60)."""

    d: int = 2

    def __post_init__(self):
        if self.d < 1:
            raise ValueError(f"rank must be >= 1, got d={self.d}")

    @property
    def threshold(self) -> int:
        return 2 * self.d


@dataclass(frozen=True)
class BasisArrays:
    """The kernel-side views of a reference ``Basis`` (mbstate.py:140-190):
    ``occ_mat`` (n, N) uint16 and ``bits_lo`` (n,) uint64 — what the device
    predicate reads.  Anything with those two attributes and ``len()`` (the
    reference ``Basis`` itself) is accepted where a basis is expected."""

    occ_mat: np.ndarray
    bits_lo: np.ndarray
    n_sp: int = 0

    def __len__(self) -> int:
        return int(self.occ_mat.shape[0])


def group_orbitals(basis, group_bits: int = 16):
    """The reference's default grouping (group_orbitals with
    bitrep_prefix_key, pipeline.py:123-159) on the basis arrays: states
    reordered so equal keys ``bits_lo & (2^group_bits − 1)`` are contiguous
    (ascending keys, input order inside a group).  Returns
    (BasisArrays in grouped order, [Orbital])."""
    from .construct import group_basis

    occ = np.ascontiguousarray(basis.occ_mat, dtype=np.uint16)
    lo = np.ascontiguousarray(basis.bits_lo, dtype=np.uint64)
    g_occ, g_lo, _, starts = group_basis(occ, lo, group_bits)
    mask = (1 << group_bits) - 1
    stops = np.append(starts[1:], g_occ.shape[0])
    orbs = [Orbital(id=q, key=int(g_lo[a]) & mask, start=int(a), stop=int(b))
            for q, (a, b) in enumerate(zip(starts, stops))]
    return BasisArrays(g_occ, g_lo, int(getattr(basis, "n_sp", 0))), orbs


def enumerate_tiles(row_orbs, col_orbs, rank: InteractionRank = InteractionRank()) -> list:
    """Orbital pairs passing the coarse ≤ 2d key test, row-major
    (enumerate_tiles / _orbital_pair_passes, pipeline.py:162-192): integer
    keys pass iff popcount(key_r ^ key_c) ≤ threshold; other keys always pass."""
    thr = rank.threshold
    out = []
    int_c = [isinstance(c.key, int) for c in col_orbs]
    for r in row_orbs:
        for c, ci in zip(col_orbs, int_c):
            if not (ci and isinstance(r.key, int)) or (r.key ^ c.key).bit_count() <= thr:
                out.append(Tile(row_orbital=r.id, col_orbital=c.id))
    return out


def _check_workers(workers) -> None:
    """The reference's worker validation (resolve_workers / env_worker_cap,
    _util.py:27-48).  On the GPU the grid is sized by the SM count; the value
    is validated and otherwise unused."""
    raw = os.environ.get(MAX_WORKERS_ENV)
    if raw is not None and raw.strip() and int(raw) < 1:
        raise ValueError(f"{MAX_WORKERS_ENV} must be >= 1, got {raw!r}")
    if workers is not None and workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")


def _tile_ranges(tiles, orbitals, transpose: bool) -> np.ndarray:
    """(T, 4) int32 (r0, r1, c0, c1) of each tile's orbitals, swapped for the
    transposed walk (pipeline.py:437-447)."""
    no, nt = len(orbitals), len(tiles)
    ids = np.fromiter((o.id for o in orbitals), np.int64, no)
    start = np.fromiter((o.start for o in orbitals), np.int64, no)
    stop = np.fromiter((o.stop for o in orbitals), np.int64, no)
    r = np.fromiter((t.row_orbital for t in tiles), np.int64, nt)
    c = np.fromiter((t.col_orbital for t in tiles), np.int64, nt)
    order = np.argsort(ids, kind="stable")
    sid = ids[order]
    pos_r = np.minimum(np.searchsorted(sid, r), max(no - 1, 0))
    pos_c = np.minimum(np.searchsorted(sid, c), max(no - 1, 0))
    if nt and (no == 0 or np.any(sid[pos_r] != r) or np.any(sid[pos_c] != c)):
        bad = [int(x) for x in np.concatenate([r, c]) if no == 0 or x not in set(ids.tolist())][:1]
        raise KeyError(bad[0] if bad else -1)  # the reference's orb_by_id lookup (pipeline.py:436-443)
    ri, ci = order[pos_r], order[pos_c]
    if transpose:
        ri, ci = ci, ri
    return np.stack([start[ri], stop[ri], start[ci], stop[ci]], axis=1)


def _contract_tiles(tiles, orbitals, basis, rank, inputs: ObservablesInput, transpose: bool, exact: bool,
                    device=None) -> np.ndarray:
    n = len(basis)
    occ = np.ascontiguousarray(basis.occ_mat, dtype=np.uint16)
    lo = np.ascontiguousarray(basis.bits_lo, dtype=np.uint64)
    if occ.ndim != 2 or occ.shape[0] != n or lo.shape != (n,):
        raise ValueError(f"basis arrays must be occ_mat (n, N) and bits_lo (n,), got {occ.shape} and {lo.shape}")
    rng = _tile_ranges(tiles, orbitals, transpose)
    if rng.size and (rng[:, [0, 2]].min() < 0 or rng[:, [1, 3]].max() > n
                     or np.any(rng[:, 1] <= rng[:, 0]) or np.any(rng[:, 3] <= rng[:, 2])):
        raise ValueError(f"orbital ranges must lie in [0, {n}) and be non-empty")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    T = rng.shape[0]
    d_rng = torch.from_numpy(rng.astype(np.int32)).to(dev)
    d_lo = torch.from_numpy(lo.view(np.int64)).to(dev)
    d_occ = torch.from_numpy(occ.view(np.int16)).to(dev)
    c = torch.from_numpy(inputs.c).to(dev).t().contiguous()  # (n, n_vec) f32
    out = torch.empty((inputs.n_vec, inputs.m_ops), dtype=torch.float64, device=dev)
    code = _OP_CODES[inputs.op_kind]
    flags = CIM_CONTRACT_EXACT_F64 if exact else 0
    with torch.cuda.device(dev):
        check(lib().cim_contract_tiles(d_lo.data_ptr(), d_occ.data_ptr(), n, occ.shape[1], int(rank.threshold),
                                       d_rng.data_ptr() if T else None, T, c.data_ptr(), inputs.n_vec,
                                       inputs.n_vec, inputs.m_ops, code, inputs.seed, out.data_ptr(), flags,
                                       torch.cuda.current_stream(dev).cuda_stream), "cim_contract_tiles")
    return out.cpu().numpy()


def contract_observables(tiles, orbitals, basis, rank, inputs: ObservablesInput, strategy: str = "array_clause",
                         workers: int | None = None, transpose: bool = False) -> np.ndarray:
    """accum[v,k] = Σ over interacting pairs (i,j) of c[v,i]·O[i,j,k]·c[v,j]
    — the reference operator with its exact signature and checks
    (pipeline.py:534-570).

    Walks ``tiles`` (orbital pairs; ``transpose`` walks each as (col, row))
    with the count predicate of ``rank`` over ``basis`` (grouped order) on the
    device (``cim_contract_tiles``): the reference's f32 products, summed in
    f32 per lane and f64 across lanes.  Raises ``ValueError`` for an unknown
    strategy, a coefficient/basis size mismatch and a bad worker count, in the
    reference's order.  ``strategy`` names the reference's CPU merge
    discipline (validated; the device reduction is the kernel's).  Fills
    ``inputs.accum`` in place and returns its (n_vec, m_ops) view.
    """
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}, expected one of {STRATEGIES}")
    if inputs.c.shape[1] != len(basis):
        raise ValueError(f"coefficients cover {inputs.c.shape[1]} states, basis has {len(basis)}")
    _check_workers(workers)
    a = _contract_tiles(tiles, orbitals, basis, rank, inputs, transpose, exact=False)
    inputs.accum[:] = a.astype(np.float32).reshape(-1)
    return inputs.accum.reshape(inputs.n_vec, inputs.m_ops)


def contract_oracle(tiles, orbitals, basis, rank, inputs: ObservablesInput) -> np.ndarray:
    """Double-precision contraction over the same pair set
    (pipeline.py:573-589): f64 products and sums on the device
    (``CIM_CONTRACT_EXACT_F64``).  Returns a fresh (n_vec, m_ops) f64 array."""
    if inputs.c.shape[1] != len(basis):
        raise ValueError(f"coefficients cover {inputs.c.shape[1]} states, basis has {len(basis)}")
    return _contract_tiles(tiles, orbitals, basis, rank, inputs, False, exact=True)
