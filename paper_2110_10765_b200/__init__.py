"""B200-native half-stored symmetric SpMM  Y = H·X + Hᵀ·X  (arXiv 2110.10765).

Public API (host side; compute runs only in the sm_100a kernels behind the
C-ABI in ``libcim_b200.so``, include/cim_b200.h):

* ``HalfTiles``         — block-half tile storage (replaces SparseSkeleton,
                          pipeline.py:96-116)
* ``sym_spmm``          — the operator (drop-in boundary of
                          contract_observables, pipeline.py:534-570)
* ``ShardedSymSpmm``    — row-block sharding over GPUs (NCCL all-gather X /
                          reduce-scatter Y)
* ``contract_observables``, ``ObservablesInput``, ``random_coefficients``,
  ``STRATEGIES``, ``OP_KINDS`` — the reference's observables API on the GPU
"""

from ._lib import BLOCK, CimError, lib
from .halftiles import HalfTiles, partition_units, plan_units, synthetic_pattern
from .observables import (
    OP_KINDS,
    STRATEGIES,
    ObservablesInput,
    contract_observables,
    random_coefficients,
)
from .sharded import ShardedSymSpmm, row_chunks
from .spmm import padded_k, supported_k, sym_spmm

__version__ = "1.0.0"

__all__ = [
    "BLOCK",
    "CimError",
    "HalfTiles",
    "ObservablesInput",
    "OP_KINDS",
    "STRATEGIES",
    "ShardedSymSpmm",
    "contract_observables",
    "lib",
    "padded_k",
    "partition_units",
    "plan_units",
    "random_coefficients",
    "row_chunks",
    "supported_k",
    "sym_spmm",
    "synthetic_pattern",
]
