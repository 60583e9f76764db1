"""Block-half tile storage of a symmetric matrix, laid out for B200 streaming.

``HalfTiles`` is the B200 replacement of the reference's ``SparseSkeleton``
(pkg/src/cimotifs/pipeline.py:96-116).  The reference stores BOTH triangles
entry by entry (int64 column + f32 value per entry, segmented per
(tile,row)).  Here only the upper block triangle is stored, as dense 64×64
tiles in the fragment order the sm_100a kernel consumes (include/cim_b200.h):

* ``tile_rc``  int32 (T, 2): (R, C) with R ≤ C, sorted — diagonal tiles first
  in each block row and stored in full;
* ``units``    int32 (U, 4): the kernel's work units (≤ ``max_unit`` tiles of
  one block row), from the native planner ``cim_plan_units``;
* ``vals``     (T, 4096) f32/f64 in HBM, 16 KB (f32) per tile, one
  ``cp.async.bulk`` each.

Constructors mirror how the reference gets a matrix:
``from_skeleton`` (a reference ``SparseSkeleton`` + orbitals),
``from_coo`` (any exactly-symmetric COO), and ``synthetic`` (the BASELINE
configs: seeded Bernoulli tile pattern, values ``h(i XOR j; seed)`` generated
bit-exactly on the device, pipeline.py:216-222).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import BLOCK, CIM_F32, CIM_F64, CIM_LAYOUT_FRAG, CIM_LAYOUT_TC, CimHalfTiles, CimSparseTiles, check, lib

DEFAULT_MAX_UNIT = 32
LAYOUTS = {"frag": CIM_LAYOUT_FRAG, "tc": CIM_LAYOUT_TC}


def default_layout(dtype, k: int | None = None) -> str:
    """Tile layout for vector blocks of width k (the storage is fixed at
    construction, so callers that know their k pass it).  Measured on one
    B200, C2 (profiles/r02/SUMMARY.md): the fragment layout's CUDA-core
    kernels win at f32 k ≤ 8 (FFMA2, at the DRAM bound) and f64 k ≤ 4; the
    tensor-core layout wins above — f32 k ≥ 16 through the split-TF32 tcgen05
    kernel, f64 k ≥ 8 through the DMMA kernel.  Without k: "frag"."""
    dt = _as_torch_dtype(dtype)
    if k is None:
        return "frag"
    k = int(k)
    if dt == torch.float32:
        return "tc" if k > 8 else "frag"
    return "tc" if k > 4 else "frag"


VALUE_KINDS = {"h_xor": _lib.CIM_VALUES_H_XOR, "op_hash": _lib.CIM_VALUES_OP_HASH, "identity": _lib.CIM_VALUES_IDENTITY}


def _dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return CIM_F32
    if dtype == torch.float64:
        return CIM_F64
    raise ValueError(f"dtype must be torch.float32 or torch.float64, got {dtype}")


def _as_torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    d = np.dtype(dtype)
    if d == np.float32:
        return torch.float32
    if d == np.float64:
        return torch.float64
    raise ValueError(f"dtype must be float32 or float64, got {dtype}")


SMALL_MATRIX_TILES = 32768  # below this many tiles the planner cuts finer units
SMALL_MATRIX_MAX_UNIT = 4


def auto_max_unit(n_tiles: int) -> int:
    """Work-unit size for a matrix of n_tiles stored tiles: 32 tiles (one
    direct-accumulator flush per unit) once there is enough work to fill
    every ring; 4 for small matrices, which are latency-bound with a few
    tiles per ring — C1 (6,268 tiles, L2 flushed): 41.0 → 34.9 µs
    (`tools/c1_units.py`)."""
    return DEFAULT_MAX_UNIT if n_tiles >= SMALL_MATRIX_TILES else SMALL_MATRIX_MAX_UNIT


def plan_units(tile_rc: np.ndarray, nb: int, max_unit: int | None = DEFAULT_MAX_UNIT,
               band_cols: int | None = None) -> np.ndarray:
    """Work units (R, t0, t1, 0) via the native planner (validates tile order:
    (R, C) sorted, or (C // band_cols, R, C) when ``band_cols`` is given)."""
    rc = np.ascontiguousarray(tile_rc, dtype=np.int32)
    T = rc.shape[0]
    if max_unit is None:
        max_unit = auto_max_unit(T)
    out = np.zeros((max(T, 1), 4), dtype=np.int32)
    nu = ctypes.c_int64(0)
    check(lib().cim_plan_units_banded(rc.ctypes.data if T else None, T, nb, max_unit,
                                      int(band_cols) if band_cols else int(nb), out.ctypes.data, ctypes.byref(nu)),
          "cim_plan_units_banded")
    return out[: nu.value].copy()


def band_order(tile_rc: np.ndarray, band_cols: int) -> np.ndarray:
    """Permutation putting (R, C)-sorted tiles into column-band order
    (C // band_cols, R, C) — stable, so a single band keeps the input order."""
    rc = np.asarray(tile_rc).reshape(-1, 2)
    return np.lexsort((rc[:, 1], rc[:, 0], rc[:, 1] // max(1, int(band_cols))))


def default_bands(n: int) -> int:
    """Column bands for an order-n matrix: enough that one band's slice of X
    and Y at k = 8 f32 (2·(n/bands)·32 B) stays within ~half of the 126 MB L2
    (the random side of the transposed product); 1 below that."""
    need = 2 * n * 8 * 4
    return max(1, -(-need // (64 << 20)))


def partition_units(units: np.ndarray, parts: int) -> np.ndarray:
    """Balanced contiguous unit ranges for `parts` GPUs (bounds, len parts+1)."""
    u = np.ascontiguousarray(units, dtype=np.int32)
    b = np.zeros(parts + 1, dtype=np.int64)
    check(lib().cim_partition_units(u.ctypes.data if u.size else None, u.shape[0], parts, b.ctypes.data),
          "cim_partition_units")
    return b


def sparse_tile_offsets(rowcnt: torch.Tensor, n_tiles: int):
    """Device scan step of the sparse-tile build (the reference's
    counts_to_offsets / scan motif, scan.py:45-65, :131-139, on the GPU):
    rowcnt int32 (≥T, 64) per-row entry counts → (rowptr int16 (T, 72),
    counts int64 (T,), entry_off int64 (T+1,)) via ``cim_sparse_tile_offsets``
    (warp row scans + ``cim_exclusive_scan_i64`` over the padded tile sizes)."""
    dev = rowcnt.device
    T = int(n_tiles)
    rc = rowcnt.to(torch.int32).contiguous()
    rowptr = torch.empty((max(T, 1), SPARSE_PTR_STRIDE), dtype=torch.int16, device=dev)
    counts = torch.empty(max(T, 1), dtype=torch.int64, device=dev)
    off = torch.empty(T + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().cim_sparse_tile_offsets(rc.data_ptr() if T else None, T, SPARSE_ALIGN,
                                            rowptr.data_ptr() if T else None, counts.data_ptr() if T else None,
                                            off.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
              "cim_sparse_tile_offsets")
    return rowptr[:T], counts[:T], off


def _mirror_csr(ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, n_pad: int):
    """Both triangles of a block-upper row-CSR (device): every entry (i, j)
    whose j lies outside i's 64-block is also stored as (j, i) in row j;
    entries of diagonal blocks are already stored both ways.  Rows stay
    column-sorted.  Returns (ptr, col, val, nnz)."""
    nnz = int(ptr[-1].item())
    if nnz == 0:
        return ptr, col, val, 0
    dev = ptr.device
    counts = ptr[1:] - ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(n_pad, device=dev), counts)
    c = col[:nnz].long()
    v = val[:nnz]
    mask = (c >> 6) != (rows >> 6)
    r2 = torch.cat([rows, c[mask]])
    c2 = torch.cat([c, rows[mask]])
    v2 = torch.cat([v, v[mask]])
    order = torch.argsort(r2 * n_pad + c2)
    r2, c2, v2 = r2[order], c2[order], v2[order]
    cnt = torch.bincount(r2, minlength=n_pad)
    ptr2 = exclusive_scan(cnt[:n_pad].to(torch.int64))
    return ptr2, c2.to(torch.int32).contiguous(), v2.contiguous(), int(r2.numel())


def exclusive_scan(x: torch.Tensor) -> torch.Tensor:
    """Offsets + total of int64 device counts (scan_serial, scan.py:131-139,
    followed by the total, as CountsAndOffsets holds them): y[i] = Σ_(j<i) x[j],
    y[n] = Σ x — ``cim_exclusive_scan_i64``."""
    x = x.to(torch.int64).contiguous()
    n = x.numel()
    y = torch.empty(n + 1, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        check(lib().cim_exclusive_scan_i64(x.data_ptr() if n else None, n, y.data_ptr(),
                                           torch.cuda.current_stream(x.device).cuda_stream), "cim_exclusive_scan_i64")
    return y


def synthetic_pattern(nb: int, p: float, seed: int = 0) -> np.ndarray:
    """Tile pattern of the BASELINE configs: every diagonal tile, plus each
    upper pair (R<C) kept with probability p.

    Small grids (≤ 2²⁶ upper pairs) draw one Bernoulli per pair from
    ``np.random.default_rng(seed)`` in ``triu_indices`` order (SURVEY.md §8(d)
    C1: 5,244 off-diagonal tiles at nb=1024, p=0.01, seed 0).  Large grids
    draw geometric gaps over the same linear order (C2/C3).
    """
    rng = np.random.default_rng(seed)
    n_pairs = nb * (nb - 1) // 2
    if n_pairs == 0 or p <= 0:
        lin = np.zeros(0, dtype=np.int64)
    elif n_pairs <= (1 << 26):
        lin = np.flatnonzero(rng.random(n_pairs) < p).astype(np.int64)
    else:
        parts = []
        pos = -1
        expect = int(n_pairs * p * 1.05) + 1024
        while True:
            gaps = rng.geometric(p, size=expect)
            cs = pos + np.cumsum(gaps, dtype=np.int64)
            parts.append(cs[cs < n_pairs])
            if cs[-1] >= n_pairs:
                break
            pos = int(cs[-1])
        lin = np.concatenate(parts)
    # linear upper-triangle index → (R, C): row R starts at R·(nb-1) − R(R-1)/2
    R_all = np.arange(nb, dtype=np.int64)
    starts = R_all * (nb - 1) - R_all * (R_all - 1) // 2
    R = np.searchsorted(starts, lin, side="right") - 1
    C = lin - starts[R] + R + 1
    diag = np.stack([R_all, R_all], axis=1)
    off = np.stack([R, C], axis=1)
    rc = np.concatenate([diag, off]).astype(np.int32)
    order = np.lexsort((rc[:, 1], rc[:, 0]))
    return np.ascontiguousarray(rc[order])


def tc_index_map() -> np.ndarray:
    """For the TC layout: flat storage index e → row-major index r·64+c
    (include/cim_b200.h CIM_LAYOUT_TC: rows of 256 B, 16-byte chunks
    XOR-swizzled by row % 8)."""
    e = np.arange(4096)
    row = e >> 6
    col = (((e >> 2) & 15) ^ (row & 7)) * 4 + (e & 3)
    return row * BLOCK + col


def fragment_pack_host(tiles: np.ndarray, layout: str = "frag") -> np.ndarray:
    """Row-major (T,64,64) → storage order (T,4096) on the host (numpy).
    Same map as the device ``cim_pack_tiles``; used to cross-check it."""
    T = tiles.shape[0]
    if layout == "tc":
        return np.ascontiguousarray(tiles.reshape(T, 4096)[:, tc_index_map()])
    is64 = tiles.dtype == np.float64
    idx = np.arange(4096)
    if not is64:
        j = idx & 3
        mb = (idx >> 2) & 127
        i = idx >> 9
    else:
        jj = idx & 1
        mb = (idx >> 1) & 127
        h = (idx >> 8) & 1
        i = idx >> 9
        j = 2 * h + jj
    rg = (mb & 31) >> 2
    cg = ((mb >> 5) << 2) | (mb & 3)
    row = rg + 8 * i
    col = cg + 16 * j
    return np.ascontiguousarray(tiles.reshape(T, 4096)[:, row * BLOCK + col])


# mean (one-triangle) entries per non-empty row below which small tiles stay
# entry-parallel: 12 for the half-stored CSR; with both triangles in the rows
# (no per-entry reductions) the row walk already wins at 4.8 (1%-fill C2
# family: 0.511 → 0.490 ms), so 4
CSR_MIN_ROW_ENTRIES = int(os.environ.get("CIM_CSR_MIN_ROW", "12"))
CSR_MIN_ROW_ENTRIES_SYM = int(os.environ.get("CIM_CSR_MIN_ROW_SYM", "4"))
SPARSE_ALIGN = 16  # entries: every sparse tile's entry range starts 16-entry aligned (vector staging)
SPARSE_PTR_STRIDE = 72  # uint16 row / column pointers per sparse tile (65 used): 144-byte, 16-B-aligned rows


def dense_break_even(dtype) -> float:
    """Memory break-even fill of a 64-tile: dense costs 4096·s bytes, a sparse
    tile (4 + s) bytes per entry (column, row, column permutation, value;
    +268 B per tile) — ½ for f32, ⅔ for f64.  Pass it
    as ``dense_fill`` to minimise HBM footprint."""
    return 0.5 if _as_torch_dtype(dtype) == torch.float32 else 2.0 / 3.0


# Time break-even on B200 (C2 pattern, k = 8 f32, profiles/r01/sparse_small.md):
# all-sparse storage runs 1.24 / 1.11 / 1.45 / 2.01 / 2.43 ms at
# 3 / 5 / 9 / 13 / 17% entry fill against 1.61 ms for the same tiles stored
# dense, so tiles below ~10% fill are faster sparse.  The default split
# optimises time (with a margin).
DEFAULT_DENSE_FILL = 0.10


@dataclass
class SparseTiles:
    """COO-in-tile storage of the sparse stored tiles (include/cim_b200.h,
    cim_sparse_tiles): per tile its entries sorted by local row, then column."""

    tile_rc: torch.Tensor  # int32 (Ts,2) device
    entry_off: torch.Tensor  # int64 (Ts+1) device
    rowptr: torch.Tensor  # int16 (Ts,72) device (first 65 used; values ≤ 4096)
    colptr: torch.Tensor  # int16 (Ts,72) device
    col: torch.Tensor  # uint8 (E,) device
    row: torch.Tensor  # uint8 (E,) device
    cperm: torch.Tensor  # int16 (E,) device: tile-relative entry index, column-major order
    vals: torch.Tensor  # (E,) device, matrix dtype
    tile_rc_host: np.ndarray
    entry_off_host: np.ndarray  # tile starts, multiples of SPARSE_ALIGN
    counts_host: np.ndarray  # real entries per tile (the rest of a tile's range is zero padding)
    _desc: CimSparseTiles | None = field(default=None, repr=False)
    _split: tuple | None = field(default=None, repr=False)
    # row-CSR copy of the small tiles (csr_ptr, csr_col, csr_val, nnz), built
    # lazily for the row-walk apply; use_csr=False keeps the entry-parallel path
    use_csr: bool = field(default_factory=lambda: os.environ.get("CIM_SPARSE_CSR", "1") != "0")
    _csr: tuple | None = field(default=None, repr=False)
    # csr_symmetric: the CSR rows also hold the mirrored off-diagonal-block
    # entries (a gather per row, no transposed L2 reductions; 2x the CSR
    # bytes).  The default: the half-stored CSR is bound by the L2's
    # reduction rate (basis skeleton n = 262,144: 0.713 → 0.506 ms per apply);
    # CIM_SPARSE_CSR_SYM=0 keeps one triangle.  The tiles themselves stay
    # half-stored — the CSR is the apply's derived copy either way.
    csr_symmetric: bool = field(default_factory=lambda: os.environ.get("CIM_SPARSE_CSR_SYM", "1") != "0")

    @property
    def n_tiles(self) -> int:
        return int(self.tile_rc_host.shape[0])

    @property
    def n_entries(self) -> int:
        """Length of the entry arrays (real entries + per-tile padding)."""
        return int(self.entry_off_host[-1]) if self.entry_off_host.size else 0

    @property
    def n_real_entries(self) -> int:
        return int(self.counts_host.sum())

    def entries_per_tile(self) -> np.ndarray:
        return self.counts_host

    def work_split(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(staged, small): device int32 tile-index lists of the sparse
        kernel's two paths — tiles above ``cim_sparse_small_max()`` padded
        entries go through the shared-memory ring, the non-empty rest are
        walked entry-parallel (cim_sparse_tiles.staged_tiles / small_tiles)."""
        if self._split is None:
            from ._lib import lib

            thr = int(lib().cim_sparse_small_max())
            ne = np.diff(self.entry_off_host)
            staged = np.flatnonzero(ne > thr).astype(np.int32)
            small = np.flatnonzero((ne > 0) & (ne <= thr)).astype(np.int32)
            dev = self.tile_rc.device
            mk = lambda a: torch.from_numpy(a if a.size else np.zeros(1, np.int32)).to(dev)  # noqa: E731
            self._split = (mk(staged), staged.size, mk(small), small.size,
                           int(ne[staged].max()) if staged.size else 0)
        return self._split[0][: self._split[1]], self._split[2][: self._split[3]]

    def _small_dominated(self) -> bool:
        """Do small tiles hold at least half the (padded) sparse entries?  The
        row-CSR then takes every sparse tile (basis skeletons); matrices of
        mostly staged tiles keep the shared-memory ring."""
        ne = np.diff(self.entry_off_host)
        _, n_st, sm, n_sm, _ = self._split
        small_entries = int(ne[sm[:n_sm].cpu().numpy()].sum()) if n_sm else 0
        return 2 * small_entries >= float(os.environ.get("CIM_CSR_SMALL_SHARE", "0.5")) * 2 * int(ne.sum())

    def build_csr(self, n_pad: int):
        """The row-CSR of the small tiles on the device (cim_sparse_csr_count →
        cim_exclusive_scan_i64 → cim_sparse_csr_fill): (csr_ptr int64
        (n_pad+1), csr_col int32 (nnz), csr_val (nnz), nnz).  Entry order per
        row: the block row's small tiles in list order, then column order."""
        from ._lib import lib

        self.work_split()
        st, n_st, sm, n_sm, st_max = self._split
        dev = self.tile_rc.device
        L = lib()
        stream = torch.cuda.current_stream(dev).cuda_stream
        base = self._base_descriptor()
        # the CSR takes every non-empty tile (staged ones too): on basis
        # skeletons one row walk is faster than the row walk + the staged ring
        # (n = 262,144: 0.739 → 0.716 ms)
        allt = np.sort(np.concatenate([st[:n_st].cpu().numpy(), sm[:n_sm].cpu().numpy()])).astype(np.int32)
        all_dev = torch.from_numpy(allt if allt.size else np.zeros(1, np.int32)).to(dev)
        base.small_tiles, base.n_small = all_dev.data_ptr(), int(allt.size)
        cnt = torch.empty(max(n_pad, 1), dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            check(L.cim_sparse_csr_count(ctypes.byref(base), n_pad, cnt.data_ptr(), stream), "cim_sparse_csr_count")
        ptr = exclusive_scan(cnt[:n_pad])
        nnz = int(ptr[-1].item())
        busy = int((cnt[:n_pad] > 0).sum().item())
        if nnz < (CSR_MIN_ROW_ENTRIES_SYM if self.csr_symmetric else CSR_MIN_ROW_ENTRIES) * max(busy, 1):
            # rows this short leave most lanes of a row group idle: the
            # entry-parallel small-tile kernel is faster (1%-fill C2 family:
            # 4.8 entries per row, 0.52 vs 0.57 ms) — keep it
            self.use_csr = False
            self._desc = None
            return None
        col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(nnz, 1), dtype=self.vals.dtype, device=dev)
        small = allt
        R = self.tile_rc_host[small, 0] if small.size else np.zeros(0, np.int32)
        if R.size and np.any(np.diff(R) < 0):
            raise ValueError("small-tile list must be grouped by block row")
        starts = np.flatnonzero(np.concatenate([[True], R[1:] != R[:-1]])) if R.size else np.zeros(0, np.int64)
        panel_R = torch.from_numpy(np.ascontiguousarray(R[starts], dtype=np.int32)).to(dev)
        panel_ptr = torch.from_numpy(np.append(starts, R.size).astype(np.int64)).to(dev)
        from ._lib import CIM_F32, CIM_F64

        with torch.cuda.device(dev):
            check(L.cim_sparse_csr_fill(ctypes.byref(base), CIM_F32 if self.vals.dtype == torch.float32 else CIM_F64,
                                        panel_R.data_ptr(), panel_ptr.data_ptr(), int(starts.size), ptr.data_ptr(),
                                        col.data_ptr(), val.data_ptr(), stream), "cim_sparse_csr_fill")
        if self.csr_symmetric:
            ptr, col, val, nnz = _mirror_csr(ptr, col, val, int(n_pad))
        self._csr = (ptr, col, val, nnz, int(n_pad))
        self._csr_list = all_dev  # keeps the merged list alive for the fill
        self._desc = None
        return self._csr

    def _base_descriptor(self) -> CimSparseTiles:
        e = self.n_entries > 0
        self.work_split()
        st, n_st, sm, n_sm, st_max = self._split
        return CimSparseTiles(n_tiles=self.n_tiles, n_entries=self.n_entries,
                              tile_rc=self.tile_rc.data_ptr(), entry_off=self.entry_off.data_ptr(),
                              rowptr=self.rowptr.data_ptr(), colptr=self.colptr.data_ptr(),
                              col=self.col.data_ptr() if e else None, row=self.row.data_ptr() if e else None,
                              cperm=self.cperm.data_ptr() if e else None,
                              vals=self.vals.data_ptr() if e else None,
                              staged_tiles=st.data_ptr(), n_staged=n_st,
                              small_tiles=sm.data_ptr(), n_small=n_sm, staged_max_entries=st_max)

    def descriptor(self, n_pad: int | None = None) -> CimSparseTiles:
        """C-ABI view; with ``n_pad`` (the matrix's padded order) and
        ``use_csr`` the small tiles' row-CSR is built once and attached."""
        if self._desc is None or (n_pad is not None and self.use_csr and self._csr is None
                                  and self._split is not None and self._split[3] > 0):
            self.work_split()
            if n_pad is not None and self.use_csr and self._csr is None and self._split[3] > 0:
                if self._small_dominated():
                    self.build_csr(n_pad)
                else:  # mostly staged tiles: the shared-memory ring is the faster walk for them
                    self.use_csr = False
            d = self._base_descriptor()
            if self.use_csr and self._csr is not None:
                ptr, col, val, nnz, rows = self._csr
                d.csr_ptr, d.csr_col, d.csr_val = ptr.data_ptr(), col.data_ptr(), val.data_ptr()
                d.csr_rows, d.csr_nnz, d.csr_all = rows, nnz, 1
                d.csr_symmetric = 1 if self.csr_symmetric else 0
            self._desc = d
        return self._desc

    def select_rows(self, r_lo: int, r_hi: int) -> "SparseTiles":
        """Sparse tiles with R in [r_lo, r_hi): a zero-copy slice (entry
        offsets rebased) when the tiles are (R, C)-ordered, else a gather."""
        rc = self.tile_rc_host
        sel = np.flatnonzero((rc[:, 0] >= r_lo) & (rc[:, 0] < r_hi))
        contiguous = sel.size == 0 or (sel[-1] - sel[0] + 1 == sel.size)
        if contiguous:
            s0 = int(sel[0]) if sel.size else 0
            s1 = s0 + sel.size
            e0, e1 = int(self.entry_off_host[s0]), int(self.entry_off_host[s1])
            off_host = self.entry_off_host[s0:s1 + 1] - e0
            ev = lambda t: t[e0:max(e1, e0 + 1)]  # noqa: E731  (entry arrays keep ≥ 1 slot)
            return SparseTiles(tile_rc=self.tile_rc[s0:s1], entry_off=self.entry_off[s0:s1 + 1] - e0,
                               rowptr=self.rowptr[s0:s1], colptr=self.colptr[s0:s1], col=ev(self.col),
                               row=ev(self.row), cperm=ev(self.cperm), vals=ev(self.vals),
                               tile_rc_host=rc[s0:s1], entry_off_host=off_host, counts_host=self.counts_host[s0:s1])
        tid, r, c, v, _ = self.to_entries()
        m = np.isin(tid, sel)
        remap = np.full(self.n_tiles, -1, np.int64)
        remap[sel] = np.arange(sel.size)
        return SparseTiles.from_entries(rc[sel], remap[tid[m]], r[m], c[m], v[m], self.vals.dtype,
                                        self.tile_rc.device)

    def with_lists(self, staged: np.ndarray, small: np.ndarray) -> "SparseTiles":
        """The same tiles with the kernel work lists restricted to ``staged`` /
        ``small`` (subsets of ``work_split()``'s lists) — a schedule group."""
        self.work_split()
        st_max = self._split[4]
        dev = self.tile_rc.device
        mk = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32) if a.size else np.zeros(1, np.int32)).to(dev)  # noqa: E731
        return SparseTiles(self.tile_rc, self.entry_off, self.rowptr, self.colptr, self.col, self.row, self.cperm,
                           self.vals, self.tile_rc_host, self.entry_off_host, self.counts_host,
                           _split=(mk(staged), int(staged.size), mk(small), int(small.size), st_max))

    def with_values(self, vals: torch.Tensor) -> "SparseTiles":
        return SparseTiles(self.tile_rc, self.entry_off, self.rowptr, self.colptr, self.col, self.row, self.cperm,
                           vals, self.tile_rc_host, self.entry_off_host, self.counts_host, _split=self._split)

    def arrays(self) -> dict:
        """Host copies of every array (npz interchange)."""
        return dict(sp_tile_rc=self.tile_rc_host, sp_entry_off=self.entry_off_host, sp_counts=self.counts_host,
                    sp_rowptr=self.rowptr.cpu().numpy(), sp_colptr=self.colptr.cpu().numpy(),
                    sp_col=self.col.cpu().numpy(), sp_row=self.row.cpu().numpy(), sp_cperm=self.cperm.cpu().numpy(),
                    sp_vals=self.vals.cpu().numpy())

    @classmethod
    def from_arrays(cls, z, dtype, device) -> "SparseTiles":
        dev = torch.device(device)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        return cls(tile_rc=t(z["sp_tile_rc"]), entry_off=t(z["sp_entry_off"]), rowptr=t(z["sp_rowptr"]),
                   colptr=t(z["sp_colptr"]), col=t(z["sp_col"]), row=t(z["sp_row"]), cperm=t(z["sp_cperm"]),
                   vals=t(z["sp_vals"]).to(dtype), tile_rc_host=np.asarray(z["sp_tile_rc"]),
                   entry_off_host=np.asarray(z["sp_entry_off"]), counts_host=np.asarray(z["sp_counts"]))

    @classmethod
    def from_entries(cls, tile_rc: np.ndarray, tile_id: np.ndarray, r: np.ndarray, c: np.ndarray, v: np.ndarray,
                     dtype, device) -> "SparseTiles":
        """Entries (tile_id, local row r, local col c, value v), any order, no
        duplicates; tile_rc[t] = (R, C) of tile t."""
        order = np.lexsort((c, r, tile_id))
        tile_id, r, c, v = tile_id[order], r[order], c[order], v[order]
        T = tile_rc.shape[0]
        counts = np.bincount(tile_id, minlength=T).astype(np.int64)
        off = np.zeros(T + 1, dtype=np.int64)
        np.cumsum((counts + SPARSE_ALIGN - 1) // SPARSE_ALIGN * SPARSE_ALIGN, out=off[1:])
        start = np.zeros(T + 1, dtype=np.int64)
        np.cumsum(counts, out=start[1:])
        local = np.arange(tile_id.size, dtype=np.int64) - start[tile_id]
        pos = off[tile_id] + local  # slot of each (sorted) entry in the padded arrays
        rowcnt = np.zeros((T, 64), dtype=np.int64)
        np.add.at(rowcnt, (tile_id, r), 1)
        rowptr = np.zeros((T, SPARSE_PTR_STRIDE), dtype=np.int64)
        rowptr[:, 1:65] = np.cumsum(rowcnt, axis=1)
        colcnt = np.zeros((T, 64), dtype=np.int64)
        np.add.at(colcnt, (tile_id, c), 1)
        colptr = np.zeros((T, SPARSE_PTR_STRIDE), dtype=np.int64)
        colptr[:, 1:65] = np.cumsum(colcnt, axis=1)
        corder = np.lexsort((r, c, tile_id))  # column-major within each tile, rows ascending
        E = int(off[-1])
        col_a = np.zeros(max(E, 1), np.uint8)
        row_a = np.zeros(max(E, 1), np.uint8)
        cperm_a = np.zeros(max(E, 1), np.int16)
        val_a = np.zeros(max(E, 1), np.float64)
        col_a[pos], row_a[pos], val_a[pos] = c, r, v
        cperm_a[off[tile_id] + local] = local[corder]  # k-th slot of tile t holds its k-th column-major entry
        dev = torch.device(device)
        return cls(tile_rc=torch.from_numpy(np.ascontiguousarray(tile_rc, dtype=np.int32)).to(dev),
                   entry_off=torch.from_numpy(off).to(dev),
                   rowptr=torch.from_numpy(rowptr.astype(np.int16)).to(dev),
                   colptr=torch.from_numpy(colptr.astype(np.int16)).to(dev),
                   col=torch.from_numpy(col_a).to(dev), row=torch.from_numpy(row_a).to(dev),
                   cperm=torch.from_numpy(cperm_a).to(dev),
                   vals=torch.from_numpy(val_a).to(dev, _as_torch_dtype(dtype)),
                   tile_rc_host=np.ascontiguousarray(tile_rc, dtype=np.int32), entry_off_host=off,
                   counts_host=counts)

    def to_entries(self):
        """Host (tile_id, r, c, v, tile-relative index) of every real entry (stored order)."""
        off, cnt = self.entry_off_host, self.counts_host
        tile_id = np.repeat(np.arange(self.n_tiles), cnt)
        start = np.zeros(self.n_tiles + 1, dtype=np.int64)
        np.cumsum(cnt, out=start[1:])
        local = np.arange(int(cnt.sum())) - start[tile_id]
        pos = off[tile_id] + local
        return (tile_id, self.row.cpu().numpy().astype(np.int64)[pos], self.col.cpu().numpy().astype(np.int64)[pos],
                self.vals.cpu().numpy()[pos], local)


@dataclass
class HalfTiles:
    """Half-stored symmetric block-sparse matrix resident in HBM: dense 64-tiles
    (``vals``, fragment order) plus, optionally, sparse tiles (``sparse``)."""

    n: int
    tile_rc: torch.Tensor  # int32 (T,2) on device
    units: torch.Tensor  # int32 (U,4) on device
    vals: torch.Tensor  # (T,4096) on device, fragment order
    tile_rc_host: np.ndarray
    units_host: np.ndarray
    layout: str = "frag"
    meta: dict = field(default_factory=dict)
    _desc: CimHalfTiles | None = field(default=None, repr=False)
    _ws: torch.Tensor | None = field(default=None, repr=False)
    sparse: SparseTiles | None = None
    _det: tuple | None = field(default=None, repr=False)

    # ------------------------------------------------------------------ props
    @property
    def dtype(self) -> torch.dtype:
        return self.vals.dtype

    @property
    def device(self) -> torch.device:
        return self.vals.device

    @property
    def nb(self) -> int:
        return (self.n + BLOCK - 1) // BLOCK

    @property
    def n_pad(self) -> int:
        return self.nb * BLOCK

    @property
    def n_tiles(self) -> int:
        return int(self.tile_rc_host.shape[0])

    @property
    def n_diag_tiles(self) -> int:
        rc = self.tile_rc_host
        return int(np.count_nonzero(rc[:, 0] == rc[:, 1]))

    @property
    def n_off_tiles(self) -> int:
        return self.n_tiles - self.n_diag_tiles

    @property
    def n_sparse_tiles(self) -> int:
        return self.sparse.n_tiles if self.sparse is not None else 0

    def _sparse_split(self) -> tuple[int, int]:
        """(off-diagonal, diagonal) entries of the sparse tiles."""
        if self.sparse is None:
            return 0, 0
        rc = self.sparse.tile_rc_host
        cnt = self.sparse.entries_per_tile()
        diag = int(cnt[rc[:, 0] == rc[:, 1]].sum())
        return int(cnt.sum()) - diag, diag

    @property
    def nnz_stored(self) -> int:
        """Stored entries: 4096 per dense tile plus the sparse tiles' entries."""
        return self.n_tiles * BLOCK * BLOCK + (self.sparse.n_real_entries if self.sparse is not None else 0)

    def flops(self, k: int) -> int:
        """Algorithmic FLOPs of one apply: 2·k·(2·nnz_off + nnz_diag)."""
        s_off, s_diag = self._sparse_split()
        return 2 * k * ((2 * self.n_off_tiles + self.n_diag_tiles) * BLOCK * BLOCK + 2 * s_off + s_diag)

    def algorithmic_bytes(self, k: int) -> int:
        """SURVEY.md §8(d) literally: s·nnz_stored + 2·nnz_COO + 8·n_tiles +
        2·n·k·s — a COO-in-tile entry is credited its value and a 2-byte
        (row, column) index, every stored tile (dense or sparse) its 8-byte
        (R, C) header, X read once and Y written once.  The storage's other
        index bytes (column permutation, per-tile pointer arrays, the
        small-tile CSR) and any extra X gathers or Y updates are overhead,
        not credit."""
        s = self.vals.element_size()
        n_coo, n_sp_tiles = 0, 0
        if self.sparse is not None:
            n_coo, n_sp_tiles = self.sparse.n_real_entries, self.sparse.n_tiles
        return s * self.nnz_stored + 2 * n_coo + 8 * (self.n_tiles + n_sp_tiles) + 2 * self.n * k * s

    def descriptor(self) -> CimHalfTiles:
        if self._desc is None:
            self._desc = CimHalfTiles(
                n=self.n,
                block=BLOCK,
                dtype=_dtype_code(self.dtype),
                n_tiles=self.n_tiles,
                n_units=int(self.units_host.shape[0]),
                tile_rc=self.tile_rc.data_ptr() if self.n_tiles else None,
                units=self.units.data_ptr() if self.units.numel() else None,
                vals=self.vals.data_ptr() if self.n_tiles else None,
                layout=LAYOUTS[self.layout],
                reserved=0,
                sparse=ctypes.pointer(self.sparse.descriptor(self.n_pad)) if self.n_sparse_tiles else None,
            )
            if self._det is not None:
                d = self._desc
                d.det_row_ptr, d.det_row_tiles, d.det_col_ptr, d.det_col_tiles = (t.data_ptr() for t in self._det[:4])
        return self._desc

    def enable_deterministic(self) -> None:
        """Build the per-block-row tile lists CIM_DETERMINISTIC reads (device):
        tiles with R == b and tiles with C == b, R < b, each in (R, C) order;
        sparse tile s appears as ``n_tiles + s``."""
        n_sp = self.sparse.n_tiles if self.sparse is not None else 0
        if self._det is not None and self._det[4] == n_sp:
            return
        rc = self.tile_rc_host.astype(np.int64).reshape(-1, 2)
        if self.sparse is not None and self.sparse.n_tiles:
            # one id space: dense tile t, sparse tile n_tiles + s
            rc = np.concatenate([rc, self.sparse.tile_rc_host.astype(np.int64).reshape(-1, 2)])
        nb = self.nb
        by_row = np.lexsort((rc[:, 1], rc[:, 0]))
        row_ptr = np.searchsorted(rc[by_row, 0], np.arange(nb + 1), side="left").astype(np.int64)
        off = np.flatnonzero(rc[:, 0] < rc[:, 1])
        by_col = off[np.lexsort((rc[off, 1], rc[off, 0], rc[off, 1]))]
        col_ptr = np.searchsorted(rc[by_col, 1], np.arange(nb + 1), side="left").astype(np.int64)
        dev = self.device
        mk = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt) if a.size else np.zeros(1, dt)).to(dev)  # noqa: E731
        self._det = (mk(row_ptr, np.int64), mk(by_row, np.int32), mk(col_ptr, np.int64), mk(by_col, np.int32), n_sp)
        self._desc = None

    def _workspace(self, nbytes: int) -> torch.Tensor:
        """Cached device scratch (host-batch pipeline buffers), grown on demand."""
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=self.device)
        return self._ws

    # ----------------------------------------------------------- constructors
    @classmethod
    def _from_pattern(cls, n: int, tile_rc: np.ndarray, dtype, device, max_unit: int | None,
                      layout: str | None = None, bands: int | None = 1):
        """Empty tile storage for the pattern.  Returns (H, perm): tiles are
        stored in column-band order, ``perm[s]`` = input index of stored tile s."""
        dtype = _as_torch_dtype(dtype)
        _dtype_code(dtype)
        layout = layout or default_layout(dtype)
        if layout not in LAYOUTS:
            raise ValueError(f"unknown layout {layout!r}, expected one of {tuple(LAYOUTS)}")
        device = torch.device(device)
        if device.type != "cuda":
            raise ValueError("HalfTiles live in GPU memory: device must be a CUDA device")
        nb = (n + BLOCK - 1) // BLOCK
        rc = np.ascontiguousarray(tile_rc, dtype=np.int32).reshape(-1, 2)
        plan_units(rc, nb, max_unit)  # validates the (R, C) order / range of the input
        bands = default_bands(n) if bands is None else max(1, int(bands))
        band_cols = -(-nb // bands)
        perm = band_order(rc, band_cols) if bands > 1 else np.arange(rc.shape[0])
        rc = np.ascontiguousarray(rc[perm])
        units = plan_units(rc, nb, max_unit, band_cols)
        t_rc = torch.from_numpy(rc).to(device)
        t_units = torch.from_numpy(units).to(device)
        vals = torch.empty((rc.shape[0], BLOCK * BLOCK), dtype=dtype, device=device)
        H = cls(n=int(n), tile_rc=t_rc, units=t_units, vals=vals, tile_rc_host=rc, units_host=units, layout=layout)
        H.meta.update(bands=bands, band_cols=band_cols)
        return H, perm

    @classmethod
    def synthetic(cls, n: int, p: float | None = None, *, n_off: int | None = None, seed: int = 0,
                  value_seed: int = 0, values: str = "h_xor", op_k: int = 0, dtype=torch.float32,
                  device="cuda", max_unit: int | None = None, tile_rc: np.ndarray | None = None,
                  layout: str | None = None, bands: int | None = 1) -> "HalfTiles":
        """Synthetic half-stored matrix (BASELINE.json configs).

        Pattern: all diagonal tiles plus upper tiles kept with probability p
        (or p = n_off / #upper-pairs).  Values: ``h_xor`` = h(i XOR j;
        value_seed) (reference matrix values), ``op_hash`` = O_ij(op_k;
        value_seed) (no XOR structure — proves the kernel treats values as
        opaque), ``identity`` = δ_ij.  Generated on the device.
        """
        if values not in VALUE_KINDS:
            raise ValueError(f"unknown values {values!r}, expected one of {tuple(VALUE_KINDS)}")
        nb = (n + BLOCK - 1) // BLOCK
        if tile_rc is None:
            n_pairs = nb * (nb - 1) // 2
            if p is None:
                p = 0.0 if n_pairs == 0 else float(n_off or 0) / n_pairs
            if not 0.0 <= p <= 1.0:
                raise ValueError(f"p must be in [0, 1], got {p}")
            tile_rc = synthetic_pattern(nb, p, seed)
        H, _ = cls._from_pattern(n, tile_rc, dtype, device, max_unit, layout, bands)
        stream = torch.cuda.current_stream(H.device).cuda_stream
        with torch.cuda.device(H.device):
            check(lib().cim_fill_synthetic_values(H.tile_rc.data_ptr() if H.n_tiles else None, H.n_tiles, n,
                                                  _dtype_code(H.dtype), LAYOUTS[H.layout], VALUE_KINDS[values],
                                                  value_seed, op_k,
                                                  H.vals.data_ptr() if H.n_tiles else None, stream),
                  "cim_fill_synthetic_values")
        H.meta.update(kind="synthetic", p=p, seed=seed, value_seed=value_seed, values=values, op_k=op_k)
        return H

    @classmethod
    def synthetic_sparse(cls, n: int, p: float | None = None, *, fill: float, n_off: int | None = None, seed: int = 0,
                         fill_seed: int = 1, value_seed: int = 0, values: str = "h_xor", op_k: int = 0,
                         dtype=torch.float32, device="cuda", tile_rc: np.ndarray | None = None) -> "HalfTiles":
        """Synthetic matrix whose stored 64-tiles are all sparse: the tile
        pattern of ``synthetic`` (seed, p / n_off), and inside each tile the
        entries (i, j) kept with probability ``fill`` by a symmetric hash of
        (min, max; fill_seed) — ragged rows like the reference's orbital
        blocks.  Built on the device by count → scan → fill (the reference's
        build_skeleton motif, pipeline.py:290-377): ``cim_sparse_count_rows``,
        torch scans, ``cim_sparse_fill_entries``."""
        if values not in VALUE_KINDS:
            raise ValueError(f"unknown values {values!r}, expected one of {tuple(VALUE_KINDS)}")
        if not 0.0 <= fill <= 1.0:
            raise ValueError(f"fill must be in [0, 1], got {fill}")
        nb = (n + BLOCK - 1) // BLOCK
        if tile_rc is None:
            n_pairs = nb * (nb - 1) // 2
            if p is None:
                p = 0.0 if n_pairs == 0 else float(n_off or 0) / n_pairs
            tile_rc = synthetic_pattern(nb, p, seed)
        dtype = _as_torch_dtype(dtype)
        H, _ = cls._from_pattern(n, np.zeros((0, 2), np.int32), dtype, device, DEFAULT_MAX_UNIT, None, 1)
        rc = np.ascontiguousarray(tile_rc, dtype=np.int32)
        plan_units(rc, nb)  # validates the pattern
        T = rc.shape[0]
        dev = H.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        t_rc = torch.from_numpy(rc).to(dev)
        rowcnt = torch.empty((max(T, 1), 64), dtype=torch.int32, device=dev)
        L = lib()
        with torch.cuda.device(dev):
            check(L.cim_sparse_count_rows(t_rc.data_ptr() if T else None, T, n, float(fill), fill_seed,
                                          rowcnt.data_ptr(), stream), "cim_sparse_count_rows")
        rowptr, counts, off = sparse_tile_offsets(rowcnt, T)
        off_host = off.cpu().numpy()
        E = int(off_host[-1])
        sp = SparseTiles(tile_rc=t_rc, entry_off=off, rowptr=rowptr,
                         colptr=torch.zeros((T, SPARSE_PTR_STRIDE), dtype=torch.int16, device=dev),
                         col=torch.zeros(max(E, 1), dtype=torch.uint8, device=dev),
                         row=torch.zeros(max(E, 1), dtype=torch.uint8, device=dev),
                         cperm=torch.zeros(max(E, 1), dtype=torch.int16, device=dev),
                         vals=torch.zeros(max(E, 1), dtype=dtype, device=dev), tile_rc_host=rc, entry_off_host=off_host,
                         counts_host=counts.cpu().numpy())
        with torch.cuda.device(dev):
            check(L.cim_sparse_fill_entries(sp.descriptor(), n, _dtype_code(dtype), float(fill), fill_seed,
                                            VALUE_KINDS[values], value_seed, op_k, stream), "cim_sparse_fill_entries")
            check(L.cim_sparse_build_columns(sp.descriptor(), stream), "cim_sparse_build_columns")
        H.sparse = sp
        H._desc = None
        H.meta.update(kind="synthetic_sparse", p=p, seed=seed, fill=fill, fill_seed=fill_seed, value_seed=value_seed,
                      values=values, op_k=op_k)
        return H

    @classmethod
    def from_dense_tiles(cls, n: int, tile_rc: np.ndarray, tiles, *, dtype=None, device="cuda",
                         max_unit: int | None = None, layout: str | None = None,
                         bands: int | None = 1) -> "HalfTiles":
        """From row-major dense tiles (T,64,64) given in ``tile_rc`` order;
        repacked on the device (stored in column-band order)."""
        tiles_t = torch.as_tensor(tiles)
        dtype = _as_torch_dtype(dtype if dtype is not None else tiles_t.dtype)
        H, perm = cls._from_pattern(n, tile_rc, dtype, device, max_unit, layout, bands)
        if H.n_tiles:
            src = tiles_t.to(device=H.device, dtype=dtype).reshape(H.n_tiles, BLOCK * BLOCK)
            if H.meta["bands"] > 1:
                src = src[torch.from_numpy(perm).to(H.device)]
            src = src.contiguous()
            stream = torch.cuda.current_stream(H.device).cuda_stream
            with torch.cuda.device(H.device):
                check(lib().cim_pack_tiles(src.data_ptr(), H.n_tiles, _dtype_code(dtype), LAYOUTS[H.layout],
                                           H.vals.data_ptr(), stream), "cim_pack_tiles")
            torch.cuda.current_stream(H.device).synchronize()
        return H

    @classmethod
    def from_coo(cls, n: int, i, j, v, *, dtype=torch.float32, device="cuda", check_symmetric: bool = True,
                 max_unit: int | None = None, layout: str | None = None, bands: int | None = 1,
                 dense_fill: float | None = None) -> "HalfTiles":
        """From a full (both-triangle) symmetric COO, e.g. a reference skeleton.

        Keeps entries with ⌊i/64⌋ ≤ ⌊j/64⌋ — lossless for an exactly symmetric
        matrix.  Tiles filled at least ``dense_fill`` (default
        below) are stored dense, the rest
        as COO-in-tile sparse tiles (``dense_fill=0`` forces all-dense).
        The default is the measured time break-even (``DEFAULT_DENSE_FILL``);
        ``dense_break_even(dtype)`` minimises memory instead.
        Duplicate (i, j) entries are summed.  Raises ValueError if (i,j,v) is
        not exactly symmetric (when check_symmetric) or indices fall outside
        [0, n).
        """
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        v = np.asarray(v)
        if not (i.shape == j.shape == v.shape) or i.ndim != 1:
            raise ValueError("i, j, v must be equal-length 1-D arrays")
        if i.size and (i.min() < 0 or j.min() < 0 or i.max() >= n or j.max() >= n):
            raise ValueError(f"COO indices must lie in [0, {n})")
        if check_symmetric and i.size:
            a = np.lexsort((j, i))
            b = np.lexsort((i, j))
            if not (np.array_equal(i[a], j[b]) and np.array_equal(j[a], i[b]) and np.array_equal(v[a], v[b])):
                raise ValueError("COO is not exactly symmetric; the half-stored format needs A == Aᵀ")
        nb = (n + BLOCK - 1) // BLOCK
        R = i // BLOCK
        C = j // BLOCK
        keep = R <= C
        i, j, v, R, C = i[keep], j[keep], v[keep], R[keep], C[keep]
        # merge duplicate entries, then group by tile
        ekey, einv = np.unique(i * n + j, return_inverse=True)
        vsum = np.zeros(ekey.size, dtype=np.float64)
        np.add.at(vsum, einv, v.astype(np.float64))
        i, j = ekey // n, ekey % n
        R, C = i // BLOCK, j // BLOCK
        key = R * nb + C
        uniq, inv, counts = np.unique(key, return_inverse=True, return_counts=True)
        thr = DEFAULT_DENSE_FILL if dense_fill is None else float(dense_fill)
        is_dense = counts >= thr * BLOCK * BLOCK
        np_dtype = np.float64 if _as_torch_dtype(dtype) == torch.float64 else np.float32
        rc_all = np.stack([uniq // nb, uniq % nb], axis=1).astype(np.int32)
        d_ids = np.flatnonzero(is_dense)
        d_map = np.full(uniq.size, -1, dtype=np.int64)
        d_map[d_ids] = np.arange(d_ids.size)
        de = is_dense[inv]
        tiles = np.zeros((d_ids.size, BLOCK, BLOCK), dtype=np.float64)
        np.add.at(tiles, (d_map[inv[de]], i[de] % BLOCK, j[de] % BLOCK), vsum[de])
        H = cls.from_dense_tiles(n, rc_all[d_ids], tiles.astype(np_dtype), dtype=dtype, device=device,
                                 max_unit=max_unit, layout=layout, bands=bands)
        s_ids = np.flatnonzero(~is_dense)
        if s_ids.size:
            s_map = np.full(uniq.size, -1, dtype=np.int64)
            s_map[s_ids] = np.arange(s_ids.size)
            se = ~de
            H.sparse = SparseTiles.from_entries(rc_all[s_ids], s_map[inv[se]], i[se] % BLOCK, j[se] % BLOCK,
                                                vsum[se], H.dtype, H.device)
            H._desc = None
        H.meta.update(kind="coo", nnz_full=int(keep.size), nnz_half=int(i.size), dense_fill=thr,
                      dense_tiles=int(d_ids.size), sparse_tiles=int(s_ids.size))
        return H

    @classmethod
    def from_basis(cls, basis_or_occ, bits_lo=None, **kw) -> "HalfTiles":
        """Build on the device from a many-body basis (grouped order) — the
        reference's count → scan → fill skeleton build into 64-tiles; see
        ``paper_2110_10765_b200.construct.from_basis``."""
        from .construct import from_basis

        return from_basis(basis_or_occ, bits_lo, **kw)

    @classmethod
    def from_basis_file(cls, path, **kw) -> "HalfTiles":
        """A reference basis file (mbstate.py save_basis format) → grouped
        (group_orbitals order) → built on the device; see
        ``paper_2110_10765_b200.construct.from_basis_file``."""
        from .construct import from_basis_file

        return from_basis_file(path, **kw)

    @classmethod
    def from_skeleton(cls, skeleton, orbitals, n: int | None = None, **kw) -> "HalfTiles":
        """From a reference ``SparseSkeleton`` (pipeline.py:96-116) and its
        orbitals: rows are recovered from the per-(tile,row) segments
        (pipeline.py:319-330), then ``from_coo``."""
        start = {o.id: o.start for o in orbitals}
        size = {o.id: o.stop - o.start for o in orbitals}
        tiles = list(skeleton.tiles)
        seg_row = np.concatenate(
            [start[t.row_orbital] + np.arange(size[t.row_orbital], dtype=np.int64) for t in tiles]
            or [np.zeros(0, np.int64)])
        counts = np.asarray(skeleton.segments.counts, dtype=np.int64)
        colind = np.asarray(skeleton.colind, dtype=np.int64)
        values = np.asarray(skeleton.values)
        # the skeleton invariants (pipeline.py:106-112, scan.py:57-65): one
        # segment per (tile, row), Σ counts = len(colind) = len(values)
        if counts.shape != seg_row.shape:
            raise ValueError(f"skeleton has {counts.size} segments, its tiles span {seg_row.size} rows")
        if not (int(counts.sum()) == colind.size == values.size):
            raise ValueError(f"segment counts ({int(counts.sum())}) and array lengths "
                             f"({colind.size}, {values.size}) disagree")
        i = np.repeat(seg_row, counts)
        if n is None:
            n = max(o.stop for o in orbitals)
        return cls.from_coo(n, i, colind, values, **kw)

    # ----------------------------------------------------------------- export
    def dense_tiles(self) -> torch.Tensor:
        """Row-major (T,64,64) copy of the stored tiles (device)."""
        out = torch.empty((self.n_tiles, BLOCK, BLOCK), dtype=self.dtype, device=self.device)
        if self.n_tiles:
            stream = torch.cuda.current_stream(self.device).cuda_stream
            with torch.cuda.device(self.device):
                check(lib().cim_unpack_tiles(self.vals.data_ptr(), self.n_tiles, _dtype_code(self.dtype),
                                             LAYOUTS[self.layout], out.data_ptr(), stream), "cim_unpack_tiles")
        return out

    def use_symmetric_csr(self, flag: bool = True) -> "HalfTiles":
        """Apply the sparse tiles' row-CSR with both triangles stored (each
        off-diagonal-block entry mirrored into its column's row): every row a
        gather, no per-entry transposed reduction into Y — the L2 reduction
        rate (~95 G rows/s) bounds the half-stored CSR on basis skeletons.
        Costs 2x the CSR entry bytes of the small tiles; the dense tiles stay
        half-stored.  Returns self."""
        if self.sparse is not None:
            self.sparse.csr_symmetric = bool(flag)
            self.sparse._csr = None
            self.sparse._desc = None
            if flag:
                self.sparse.use_csr = True
        self._desc = None
        return self

    def export_dense(self) -> tuple[np.ndarray, np.ndarray]:
        """Host (tile_rc, row-major tiles) of every stored tile — dense and
        sparse (expanded) — sorted by (R, C).  Export / checking only."""
        rc = self.tile_rc_host
        tiles = self.dense_tiles().cpu().numpy()
        if self.sparse is not None and self.sparse.n_tiles:
            tid, r, c, v, _ = self.sparse.to_entries()
            st = np.zeros((self.sparse.n_tiles, BLOCK, BLOCK), dtype=tiles.dtype)
            st[tid, r, c] = v
            rc = np.concatenate([rc, self.sparse.tile_rc_host])
            tiles = np.concatenate([tiles, st])
        order = np.lexsort((rc[:, 1], rc[:, 0]))
        return np.ascontiguousarray(rc[order]), tiles[order]

    def save(self, path) -> None:
        """npz interchange (host): n, dense tile_rc + row-major tiles, and the
        sparse tiles (tile_rc, entry offsets, row pointers, columns, values)."""
        extra = self.sparse.arrays() if self.sparse is not None else {}
        order = np.lexsort((self.tile_rc_host[:, 1], self.tile_rc_host[:, 0]))  # (R, C) order on disk
        np.savez_compressed(path, n=self.n, tile_rc=self.tile_rc_host[order],
                            tiles=self.dense_tiles().cpu().numpy()[order],
                            format="cim_half_tiles_v2", layout=self.layout, **extra)

    @classmethod
    def load(cls, path, device="cuda", **kw) -> "HalfTiles":
        z = np.load(path)
        fmt = str(z["format"])
        if fmt not in ("cim_half_tiles_v1", "cim_half_tiles_v2"):
            raise ValueError(f"{path}: not a cim_half_tiles file")
        kw.setdefault("layout", str(z["layout"]) if "layout" in z.files else None)
        H = cls.from_dense_tiles(int(z["n"]), z["tile_rc"], z["tiles"], device=device, **kw)
        if "sp_tile_rc" in z.files:
            H.sparse = SparseTiles.from_arrays(z, H.dtype, H.device)
            H._desc = None
        return H

    def row_costs(self) -> np.ndarray:
        """Streamed bytes per block row (dense tiles at their full size, sparse
        tiles at value + index bytes per entry) — the balance weight of the
        row-block partition."""
        s = self.vals.element_size()
        cost = np.bincount(self.tile_rc_host[:, 0], minlength=self.nb).astype(np.float64) * (BLOCK * BLOCK * s)
        if self.sparse is not None and self.sparse.n_tiles:
            cost += np.bincount(self.sparse.tile_rc_host[:, 0], weights=self.sparse.counts_host * (s + 4.0),
                                minlength=self.nb)
        return cost

    def partition_rows(self, parts: int) -> np.ndarray:
        """Block-row boundaries (len parts+1) of `parts` contiguous panels with
        balanced streamed bytes (dense and sparse tiles); rows never straddle."""
        if parts < 1:
            raise ValueError("parts must be >= 1")
        pre = np.concatenate([[0.0], np.cumsum(self.row_costs())])
        total = pre[-1]
        b = np.zeros(parts + 1, dtype=np.int64)
        for q in range(1, parts):
            b[q] = max(int(np.searchsorted(pre, total * q / parts, side="left")), b[q - 1])
        b[parts] = self.nb
        return np.minimum(b, self.nb)

    def shard_rows(self, r_lo: int, r_hi: int) -> "HalfTiles":
        """The tiles of block rows [r_lo, r_hi) (dense and sparse; same n) —
        a GPU's panel.  Dense tiles and their arrays are views; sparse tiles
        are a contiguous slice when stored in (R, C) order (every constructor
        here), else gathered."""
        if self.meta.get("bands", 1) > 1:
            raise ValueError("row sharding needs (R, C)-ordered tiles (bands=1)")
        rc = self.tile_rc_host
        t0 = int(np.searchsorted(rc[:, 0], r_lo, side="left"))
        t1 = int(np.searchsorted(rc[:, 0], r_hi, side="left"))
        u = self.units_host
        keep = (u[:, 0] >= r_lo) & (u[:, 0] < r_hi)
        units = u[keep].copy()
        units[:, 1:3] -= t0
        sub = HalfTiles(n=self.n, tile_rc=self.tile_rc[t0:t1], units=torch.from_numpy(units).to(self.device),
                        vals=self.vals[t0:t1], tile_rc_host=rc[t0:t1], units_host=units, layout=self.layout,
                        meta=dict(self.meta, shard_rows=(int(r_lo), int(r_hi))))
        if self.sparse is not None and self.sparse.n_tiles:
            sub.sparse = self.sparse.select_rows(r_lo, r_hi)
        return sub

    def shard(self, unit_lo: int, unit_hi: int) -> "HalfTiles":
        """View of the tiles of units [unit_lo, unit_hi) (same n; GPU panel)."""
        if self.sparse is not None:
            raise NotImplementedError("sharding a matrix with sparse tiles is not supported yet")
        u = self.units_host[unit_lo:unit_hi]
        if u.shape[0] == 0:
            t0 = t1 = 0
        else:
            t0, t1 = int(u[0, 1]), int(u[-1, 2])
        units = u.copy()
        units[:, 1:3] -= t0
        sub = HalfTiles(n=self.n, tile_rc=self.tile_rc[t0:t1], units=torch.from_numpy(units).to(self.device),
                        vals=self.vals[t0:t1], tile_rc_host=self.tile_rc_host[t0:t1], units_host=units,
                        layout=self.layout, meta=dict(self.meta, shard=(unit_lo, unit_hi)))
        return sub
