"""TEST INFRASTRUCTURE: ctypes wrapper of oracle/build/liboracle.so.

Used only by tests/, __graft_entry__.smoke() and bench.py (CPU baseline and
``--impl reference``).  See sym_spmm_ref.c for what it restates.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"
BLOCK = 64

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        p = ctypes.c_void_p
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_fill_h.argtypes = [p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, p, ctypes.c_int]
        L.oracle_sym_spmm_f32.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int, p, ctypes.c_int64, p,
                                          ctypes.c_int64, p, ctypes.c_int]
        L.oracle_sym_spmm_f32.restype = ctypes.c_int
        L.oracle_sym_spmm_f64.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int, p, ctypes.c_int64]
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def fill_h(tile_rc: np.ndarray, n: int, seed: int = 0, threads: int | None = None) -> np.ndarray:
    rc = np.ascontiguousarray(tile_rc, dtype=np.int32)
    out = np.empty((rc.shape[0], BLOCK, BLOCK), dtype=np.float32)
    lib().oracle_fill_h(rc.ctypes.data, rc.shape[0], n, seed, out.ctypes.data, threads or max_threads())
    return out


class F32Problem:
    """A (possibly sampled) tile set prepared for the f32 CPU SpMM."""

    def __init__(self, tile_rc: np.ndarray, tiles: np.ndarray, X: np.ndarray):
        self.rc = np.ascontiguousarray(tile_rc, dtype=np.int32)
        self.tiles = np.ascontiguousarray(tiles, dtype=np.float32)
        self.X = np.ascontiguousarray(X, dtype=np.float32)
        self.k = self.X.shape[1]
        off = self.rc[:, 0] != self.rc[:, 1]
        cols = np.unique(self.rc[off, 1]).astype(np.int32)
        nb = self.X.shape[0] // BLOCK
        self.col_map = np.zeros(nb, dtype=np.int32)
        self.col_map[cols] = np.arange(cols.size, dtype=np.int32)
        self.slot_block = cols
        self.Y = np.zeros_like(self.X)

    def flops(self) -> int:
        off = int(np.count_nonzero(self.rc[:, 0] != self.rc[:, 1]))
        return 2 * self.k * (2 * off + (self.rc.shape[0] - off)) * BLOCK * BLOCK

    def run(self, threads: int | None = None) -> np.ndarray:
        th = threads or max_threads()
        rc = lib().oracle_sym_spmm_f32(self.rc.shape[0], self.rc.ctypes.data, self.tiles.ctypes.data,
                                       self.X.ctypes.data, self.k, self.Y.ctypes.data, self.X.shape[0],
                                       self.col_map.ctypes.data, self.slot_block.size,
                                       self.slot_block.ctypes.data if self.slot_block.size else None, th)
        if rc != 0:
            raise MemoryError("oracle_sym_spmm_f32: allocation failed")
        return self.Y


def sym_spmm_f64(n_pad: int, tile_rc: np.ndarray, tiles: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Single-thread f64 oracle, X (n_pad, k)."""
    rc = np.ascontiguousarray(tile_rc, dtype=np.int32)
    T = np.ascontiguousarray(tiles, dtype=np.float64)
    Xd = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.empty_like(Xd)
    lib().oracle_sym_spmm_f64(rc.shape[0], rc.ctypes.data, T.ctypes.data, Xd.ctypes.data, Xd.shape[1],
                              Y.ctypes.data, n_pad)
    return Y
