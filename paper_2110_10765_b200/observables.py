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
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import check, lib
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


def contract_observables(pattern: HalfTiles, inputs: ObservablesInput, strategy: str = "array_clause",
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
        raise ValueError("pattern must be a HalfTiles (e.g. HalfTiles.from_skeleton(...))")
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
