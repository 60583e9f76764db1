"""ctypes binding of the C-ABI library ``libcim_b200.so`` (include/cim_b200.h).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2110_10765_b200/csrc``).  There is no fallback: if the shared object is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libcim_b200.so"

CIM_OK, CIM_EINVAL, CIM_ECUDA, CIM_EUNSUPPORTED = 0, 1, 2, 3
CIM_F32, CIM_F64 = 0, 1
CIM_ACCUMULATE = 1
CIM_DETERMINISTIC = 2
CIM_GRAM_FAST = 1
CIM_CONTRACT_EXACT_F64 = 4
CIM_VALUES_H_XOR, CIM_VALUES_OP_HASH, CIM_VALUES_IDENTITY = 0, 1, 2
CIM_LAYOUT_FRAG, CIM_LAYOUT_TC = 0, 1
BLOCK = 64

EXPORTS = (
    "cim_version",
    "cim_last_error",
    "cim_sym_spmm",
    "cim_sym_spmm_supported",
    "cim_layout_supports",
    "cim_plan_units",
    "cim_plan_units_banded",
    "cim_partition_units",
    "cim_fill_synthetic_values",
    "cim_fill_masked_values",
    "cim_pack_tiles",
    "cim_unpack_tiles",
    "cim_hash_values",
    "cim_sym_spmm_host_batch",
    "cim_sym_spmm_chunked",
    "cim_host_batch_workspace_bytes",
    "cim_fill_sparse_values",
    "cim_sparse_count_rows",
    "cim_sparse_fill_entries",
    "cim_sparse_build_columns",
    "cim_basis_count_tiles",
    "cim_basis_fill_dense",
    "cim_basis_fill_sparse",
    "cim_gram",
    "cim_gram_workspace_bytes",
    "cim_tsmm",
    "cim_gram_blocked",
    "cim_tsmm_blocked",
    "cim_contract_observables",
    "cim_gram_blocked_ex",
    "cim_sparse_small_max",
    "cim_tsmm_blocked_hc",
    "cim_block_residual",
    "cim_contract_tiles",
    "cim_exclusive_scan_i64",
    "cim_sparse_tile_offsets",
    "cim_sparse_csr_count",
    "cim_sparse_csr_fill",
    "cim_ritz_update_b8",
)


class CimSparseTiles(ctypes.Structure):
    """Mirror of ``struct cim_sparse_tiles``."""

    _fields_ = [
        ("n_tiles", ctypes.c_int64),
        ("n_entries", ctypes.c_int64),
        ("tile_rc", ctypes.c_void_p),
        ("entry_off", ctypes.c_void_p),
        ("rowptr", ctypes.c_void_p),
        ("colptr", ctypes.c_void_p),
        ("col", ctypes.c_void_p),
        ("row", ctypes.c_void_p),
        ("cperm", ctypes.c_void_p),
        ("vals", ctypes.c_void_p),
        ("staged_tiles", ctypes.c_void_p),
        ("n_staged", ctypes.c_int64),
        ("small_tiles", ctypes.c_void_p),
        ("n_small", ctypes.c_int64),
        ("staged_max_entries", ctypes.c_int64),
        ("csr_ptr", ctypes.c_void_p),
        ("csr_col", ctypes.c_void_p),
        ("csr_val", ctypes.c_void_p),
        ("csr_rows", ctypes.c_int64),
        ("csr_nnz", ctypes.c_int64),
        ("csr_all", ctypes.c_int64),
        ("csr_symmetric", ctypes.c_int64),
    ]


class CimHalfTiles(ctypes.Structure):
    """Mirror of ``struct cim_half_tiles``."""

    _fields_ = [
        ("n", ctypes.c_int64),
        ("block", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("n_tiles", ctypes.c_int64),
        ("n_units", ctypes.c_int64),
        ("tile_rc", ctypes.c_void_p),
        ("units", ctypes.c_void_p),
        ("vals", ctypes.c_void_p),
        ("layout", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("sparse", ctypes.POINTER(CimSparseTiles)),
        ("det_row_ptr", ctypes.c_void_p),
        ("det_row_tiles", ctypes.c_void_p),
        ("det_col_ptr", ctypes.c_void_p),
        ("det_col_tiles", ctypes.c_void_p),
    ]


class CimError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("CIM_B200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"libcim_b200.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    L = ctypes.CDLL(str(path))
    c = ctypes
    L.cim_version.restype = c.c_char_p
    L.cim_last_error.restype = c.c_char_p
    L.cim_sym_spmm.argtypes = [c.POINTER(CimHalfTiles), c.c_void_p, c.c_void_p, c.c_int32, c.c_int64,
                               c.c_int64, c.c_uint32, c.c_void_p]
    L.cim_sym_spmm_supported.argtypes = [c.c_int32, c.c_int32]
    L.cim_layout_supports.argtypes = [c.c_int32, c.c_int32, c.c_int32]
    L.cim_plan_units.argtypes = [c.c_void_p, c.c_int64, c.c_int64, c.c_int32, c.c_void_p, c.POINTER(c.c_int64)]
    L.cim_plan_units_banded.argtypes = [c.c_void_p, c.c_int64, c.c_int64, c.c_int32, c.c_int64, c.c_void_p,
                                        c.POINTER(c.c_int64)]
    L.cim_partition_units.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_void_p]
    L.cim_fill_synthetic_values.argtypes = [c.c_void_p, c.c_int64, c.c_int64, c.c_int32, c.c_int32, c.c_int32,
                                            c.c_uint64, c.c_int32, c.c_void_p, c.c_void_p]
    L.cim_fill_masked_values.argtypes = [c.c_void_p, c.c_int64, c.c_int64, c.c_int32, c.c_int32, c.c_int32,
                                         c.c_uint64, c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p]
    L.cim_sparse_small_max.argtypes = []
    L.cim_sparse_small_max.restype = c.c_int32
    L.cim_contract_observables.argtypes = [c.POINTER(CimHalfTiles), c.c_void_p, c.c_int32, c.c_int32, c.c_int32,
                                           c.c_uint64, c.c_void_p, c.c_uint32, c.c_void_p]
    L.cim_pack_tiles.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_void_p, c.c_void_p]
    L.cim_unpack_tiles.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_void_p, c.c_void_p]
    L.cim_hash_values.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_uint64, c.c_int32,
                                  c.c_void_p, c.c_void_p]
    L.cim_sym_spmm_host_batch.argtypes = [c.POINTER(CimHalfTiles), c.POINTER(c.c_void_p), c.POINTER(c.c_void_p),
                                          c.c_int32, c.c_int32, c.c_void_p, c.c_uint64]
    L.cim_sym_spmm_chunked.argtypes = [c.POINTER(CimHalfTiles), c.POINTER(c.c_void_p), c.POINTER(c.c_void_p),
                                       c.c_int32, c.c_int64, c.c_int32, c.c_int64, c.c_void_p]
    L.cim_host_batch_workspace_bytes.argtypes = [c.POINTER(CimHalfTiles), c.c_int32]
    L.cim_fill_sparse_values.argtypes = [c.POINTER(CimSparseTiles), c.c_int64, c.c_int32, c.c_int32, c.c_uint64,
                                         c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p]
    L.cim_sparse_count_rows.argtypes = [c.c_void_p, c.c_int64, c.c_int64, c.c_double, c.c_uint64, c.c_void_p,
                                        c.c_void_p]
    L.cim_sparse_fill_entries.argtypes = [c.POINTER(CimSparseTiles), c.c_int64, c.c_int32, c.c_double, c.c_uint64,
                                          c.c_int32, c.c_uint64, c.c_int32, c.c_void_p]
    L.cim_sparse_build_columns.argtypes = [c.POINTER(CimSparseTiles), c.c_void_p]
    L.cim_basis_count_tiles.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_void_p, c.c_int64,
                                        c.c_void_p, c.c_void_p]
    L.cim_basis_fill_dense.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_void_p, c.c_int64,
                                       c.c_int32, c.c_int32, c.c_uint64, c.c_void_p, c.c_void_p]
    L.cim_basis_fill_sparse.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_int32,
                                        c.POINTER(CimSparseTiles), c.c_int32, c.c_uint64, c.c_void_p]
    L.cim_gram.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int32,
                           c.c_void_p, c.c_void_p, c.c_uint64, c.c_void_p]
    L.cim_gram_workspace_bytes.argtypes = [c.c_int64, c.c_int32, c.c_int32]
    L.cim_tsmm.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_void_p, c.c_int32, c.c_float, c.c_float, c.c_void_p,
                           c.c_int64, c.c_int64, c.c_void_p]
    L.cim_gram_blocked.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_int64,
                                   c.c_int32, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_void_p,
                                   c.c_uint64, c.c_uint64, c.c_void_p]
    L.cim_gram_blocked_ex.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_int64,
                                   c.c_int32, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_void_p,
                                   c.c_uint64, c.c_uint64, c.c_uint32, c.c_void_p]
    L.cim_tsmm_blocked.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_int32,
                                   c.c_float, c.c_float, c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int64,
                                   c.c_void_p]
    L.cim_tsmm_blocked_hc.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int32, c.c_void_p, c.c_int32,
                                      c.c_float, c.c_float, c.c_void_p, c.c_int64, c.c_int32, c.c_int64, c.c_int64,
                                      c.c_void_p]
    L.cim_contract_tiles.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_void_p, c.c_int64,
                                     c.c_void_p, c.c_int64, c.c_int32, c.c_int32, c.c_int32, c.c_uint64, c.c_void_p,
                                     c.c_uint32, c.c_void_p]
    L.cim_exclusive_scan_i64.argtypes = [c.c_void_p, c.c_int64, c.c_void_p, c.c_void_p]
    L.cim_sparse_tile_offsets.argtypes = [c.c_void_p, c.c_int64, c.c_int32, c.c_void_p, c.c_void_p, c.c_void_p,
                                          c.c_void_p]
    L.cim_sparse_csr_count.argtypes = [c.POINTER(CimSparseTiles), c.c_int64, c.c_void_p, c.c_void_p]
    L.cim_sparse_csr_fill.argtypes = [c.POINTER(CimSparseTiles), c.c_int32, c.c_void_p, c.c_void_p, c.c_int64,
                                      c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p]
    for name in EXPORTS:
        if name not in ("cim_version", "cim_last_error"):
            getattr(L, name).restype = c.c_int
    L.cim_block_residual.argtypes = [c.c_void_p, c.c_void_p, c.c_void_p, c.c_int32, c.c_void_p, c.c_int64, c.c_int32,
                                     c.c_void_p]
    L.cim_ritz_update_b8.argtypes = [c.c_void_p, c.c_void_p, c.c_int64, c.c_int32, c.c_void_p, c.c_void_p, c.c_int32,
                                     c.c_void_p, c.c_int64, c.c_int64, c.c_void_p]
    L.cim_host_batch_workspace_bytes.restype = c.c_uint64
    L.cim_gram_workspace_bytes.restype = c.c_uint64
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception conventions:
    CIM_EINVAL → ValueError (pipeline.py:550-555 style), others → RuntimeError."""
    if rc == CIM_OK:
        return
    msg = lib().cim_last_error().decode(errors="replace")
    if rc == CIM_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == CIM_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise CimError(f"{what}: {msg} (code {rc})")
