"""B200-native half-stored symmetric SpMM  Y = H·X + Hᵀ·X  (arXiv 2110.10765).

Public API (host side; compute runs only in the sm_100a kernels behind the
C-ABI in ``libcim_b200.so``, include/cim_b200.h):

* ``HalfTiles``         — block-half tile storage (replaces SparseSkeleton,
                          pipeline.py:96-116)
* ``sym_spmm``          — the operator (drop-in boundary of
                          contract_observables, pipeline.py:534-570)
* ``sym_spmm_host_batch`` — the operator over a stream of host-resident vector
                          blocks, copies and kernels pipelined (PCIe-bound)
* ``ShardedSymSpmm``    — row-block sharding over GPUs (NCCL all-gather X /
                          reduce-scatter Y)
* ``contract_observables`` / ``contract_oracle`` (the reference's exact
  signatures over orbital tiles, pipeline.py:534-589), ``contract_pattern``
  (over a stored HalfTiles pattern), ``ObservablesInput``,
  ``random_coefficients``, ``STRATEGIES``, ``OP_KINDS``, and the argument
  types ``Orbital`` / ``Tile`` / ``InteractionRank`` with ``group_orbitals`` /
  ``enumerate_tiles`` — the reference's observables API on the GPU
* ``lobpcg`` / ``lobpcg_sym`` — block LOBPCG eigensolver over the SpMM
  (single GPU or row-sharded with the 3m×3m Gram all-reduce)
* ``load_basis`` / ``save_basis`` / ``group_basis`` and
  ``HalfTiles.from_basis_file`` — reference basis files (mbstate.py:242-267)
  to the device matrix without the Python skeleton build
"""

from ._lib import BLOCK, CimError, lib
from .construct import group_basis, load_basis, save_basis
from .halftiles import HalfTiles, default_layout, partition_units, plan_units, synthetic_pattern
from .lobpcg import LobpcgResult, lobpcg, lobpcg_sym
from .observables import (
    OP_KINDS,
    STRATEGIES,
    BasisArrays,
    InteractionRank,
    ObservablesInput,
    Orbital,
    Tile,
    contract_observables,
    contract_oracle,
    contract_pattern,
    enumerate_tiles,
    group_orbitals,
    random_coefficients,
)
from .sharded import ShardedSymSpmm, row_chunks
from .spmm import padded_k, supported_k, sym_spmm, sym_spmm_host_batch

__version__ = "1.0.0"

__all__ = [
    "default_layout",
    "BLOCK",
    "CimError",
    "HalfTiles",
    "LobpcgResult",
    "ObservablesInput",
    "OP_KINDS",
    "STRATEGIES",
    "ShardedSymSpmm",
    "BasisArrays",
    "InteractionRank",
    "Orbital",
    "Tile",
    "contract_observables",
    "contract_oracle",
    "contract_pattern",
    "enumerate_tiles",
    "group_orbitals",
    "group_basis",
    "lib",
    "load_basis",
    "lobpcg",
    "lobpcg_sym",
    "padded_k",
    "partition_units",
    "plan_units",
    "random_coefficients",
    "row_chunks",
    "save_basis",
    "supported_k",
    "sym_spmm",
    "sym_spmm_host_batch",
    "synthetic_pattern",
]
