"""Row-block sharding of the half-stored SpMM over the GPUs of one box.

SURVEY.md §8(e): GPU g owns a contiguous run of block rows chosen so the
streamed tile bytes are balanced (upper-triangular storage puts ~p·(nb−R)
tiles in block row R, so equal row counts would be badly unbalanced; sparse
tiles weigh their entries).  The vectors are distributed separately, in
equal 64-aligned row chunks, so the two exchange steps are plain fixed-size
NCCL collectives over NVLink:

    X_full  = all_gather(X_local)                  (every rank needs any X_C)
    Y_part  = U_g·X_full + U_g,offᵀ·X_full          (local sm_100a kernels)
    Y_local = reduce_scatter(Y_part, SUM)           (Hᵀ·X lands on other ranks)

``overlap=True`` hides both exchanges behind the kernels (§8(e)4):

* the panel's tiles whose R and C blocks both lie in this rank's own X chunk
  run first, straight from ``X_local``, while the all-gather is in flight;
* the rest run in column groups, C's chunk descending (G−1, …, 0).  Y chunk q
  receives direct products only from tiles with R in q (their C ≥ R, so
  chunk(C) ≥ q) and transposed products only from tiles with C in q, so it
  is final once group q has run: its reduction to rank q (``dist.reduce``,
  async on NCCL's stream) overlaps the groups after it, and only chunk 0's
  reduction is exposed.

One process per GPU, ``torch.distributed`` with the NCCL backend (under gloo
— CPU test harnesses — CUDA buffers are staged through host memory).  The
reference has no distribution at all; its only parallelism is
numba's thread pool (_util.py:37-62).
"""

from __future__ import annotations

import ctypes
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from ._lib import BLOCK, CIM_ACCUMULATE, check, lib
from .halftiles import DEFAULT_MAX_UNIT, HalfTiles, partition_units, plan_units, synthetic_pattern
from .spmm import _launch, padded_k


def row_chunks(n: int, world: int) -> tuple[int, int]:
    """(rows per rank, total padded rows) for the equal X/Y row distribution."""
    nb = (n + BLOCK - 1) // BLOCK
    per = ((nb + world - 1) // world) * BLOCK
    return per, per * world


def shard_tile_range(units: np.ndarray, world: int, rank: int) -> tuple[int, int, int, int]:
    """(unit_lo, unit_hi, tile_lo, tile_hi) of `rank` under balanced partition."""
    b = partition_units(units, world)
    lo, hi = int(b[rank]), int(b[rank + 1])
    if hi > lo:
        return lo, hi, int(units[lo, 1]), int(units[hi - 1, 2])
    return lo, hi, 0, 0


def sym_spmm_chunked(H: HalfTiles, X_chunks, Y_chunks, chunk_rows: int, k: int | None = None, stream=None) -> None:
    """Y += A·X with X and Y given as row chunks (``cim_sym_spmm_chunked``):
    chunk c holds rows [c·chunk_rows, (c+1)·chunk_rows).  The chunks may be
    tensors on this GPU or raw device pointers into peer GPUs' memory (the
    fused multi-GPU apply); no chunk is zeroed."""
    ptr = lambda t: t if isinstance(t, int) else t.data_ptr()  # noqa: E731
    n = len(X_chunks)
    if n != len(Y_chunks) or not 1 <= n <= 8:
        raise ValueError("need 1..8 X and Y chunks, equally many")
    if k is None:
        k = X_chunks[0].shape[1]
    xp = (ctypes.c_void_p * n)(*[ptr(t) for t in X_chunks])
    yp = (ctypes.c_void_p * n)(*[ptr(t) for t in Y_chunks])
    s = stream if stream is not None else torch.cuda.current_stream(H.device)
    handle = s.cuda_stream if isinstance(s, torch.cuda.Stream) else int(s)
    with torch.cuda.device(H.device):
        check(lib().cim_sym_spmm_chunked(H.descriptor(), xp, yp, n, chunk_rows, k, k, handle), "cim_sym_spmm_chunked")


def column_groups(H: HalfTiles, rows_per_rank: int, world: int, rank: int, max_unit: int = DEFAULT_MAX_UNIT):
    """Split a panel's tiles into the overlap schedule's groups.

    Returns ``(local, groups)``: ``local`` holds the tiles whose R and C
    blocks both lie in this rank's X chunk; ``groups[q]`` the remaining tiles
    whose C block lies in chunk q.  Each is a ``HalfTiles`` view sharing the
    panel's arrays — dense tiles through their own work units (a row's tiles
    are C-sorted, so every group is a contiguous run of each row's tiles),
    sparse tiles through restricted kernel work lists."""
    bpr = rows_per_rank // BLOCK  # blocks per chunk
    rc = H.tile_rc_host
    chunk_r, chunk_c = rc[:, 0] // bpr, rc[:, 1] // bpr
    gid = np.where((chunk_r == rank) & (chunk_c == rank), -1, chunk_c)
    units = []
    for u in H.units_host:
        R, t0, t1 = int(u[0]), int(u[1]), int(u[2])
        g = gid[t0:t1]
        cuts = np.flatnonzero(np.diff(g)) + 1
        for a, b in zip(np.concatenate([[0], cuts]), np.concatenate([cuts, [t1 - t0]])):
            units.append((int(g[a]), R, t0 + int(a), t0 + int(b)))
    U = np.array(units, dtype=np.int64).reshape(-1, 4)
    sp = H.sparse if (H.sparse is not None and H.sparse.n_tiles) else None
    if sp is not None:
        src = sp.tile_rc_host
        s_gid = np.where((src[:, 0] // bpr == rank) & (src[:, 1] // bpr == rank), -1, src[:, 1] // bpr)
        st, sm = (t.cpu().numpy() for t in sp.work_split())

    def view(g: int) -> HalfTiles | None:
        u = U[U[:, 0] == g][:, 1:]
        units = np.zeros((u.shape[0], 4), dtype=np.int32)
        units[:, :3] = u
        sub = HalfTiles(n=H.n, tile_rc=H.tile_rc, units=torch.from_numpy(units if units.size else np.zeros((1, 4), np.int32)).to(H.device),
                        vals=H.vals, tile_rc_host=H.tile_rc_host, units_host=units, layout=H.layout,
                        meta=dict(H.meta, group=g))
        empty = units.shape[0] == 0
        if sp is not None:
            sst, ssm = st[s_gid[st] == g], sm[s_gid[sm] == g]
            if sst.size or ssm.size:
                sub.sparse = sp.with_lists(sst, ssm)
                empty = False
        return None if empty else sub

    return view(-1), [view(q) for q in range(world)]


class ShardedSymSpmm:
    """Distributed ``Y = A·X`` with A's tiles row-block sharded over ranks.

    ``local_apply(X_full, Y_part)`` computes this rank's panel product into
    the zero-initialised-by-callee ``Y_part``; the default is the sm_100a
    kernel on ``H_local``.  (Tests on CPU/gloo inject the oracle here; the
    product path never does.)
    """

    def __init__(self, n: int, k: int, dtype: torch.dtype, device, H_local: HalfTiles | None = None,
                 group=None, local_apply: Callable | None = None, fused: bool = False, overlap: bool = False):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n = int(n)
        self.dtype = dtype
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:  # "cuda" → the current device, explicitly
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.H = H_local
        if local_apply is None:
            if H_local is None:
                raise ValueError("need H_local (CUDA kernel) or local_apply")
            self.k = padded_k(dtype, k, H_local.layout)
            local_apply = self._cuda_apply
        else:
            self.k = int(k)
        self.k_user = int(k)
        self.local_apply = local_apply
        self.rows_per_rank, self.rows_total = row_chunks(self.n, self.world)
        self.X_full = torch.zeros((self.rows_total, self.k), dtype=dtype, device=self.device)
        self.Y_part = torch.zeros((self.rows_total, self.k), dtype=dtype, device=self.device)
        self.Y_local = torch.zeros((self.rows_per_rank, self.k), dtype=dtype, device=self.device)
        self.n_pad = ((self.n + BLOCK - 1) // BLOCK) * BLOCK
        self.fused = bool(fused) and self.world > 1 and local_apply == self._cuda_apply
        if self.fused:
            if H_local.n_sparse_tiles:
                raise ValueError("the fused peer-memory apply streams dense tiles only; use the NCCL exchange "
                                 "(fused=False) for matrices with sparse tiles")
            self._setup_fused()
        # the own-chunk group reads X through a virtual base (only this rank's
        # rows are backed); sparse tiles too wide for the staged ring (f64
        # k = 64) run as column passes over a pass-major copy of every X row,
        # so that case keeps the serial exchange
        wide_sparse = (H_local is not None and H_local.n_sparse_tiles > 0 and dtype == torch.float64
                       and self.k > 32)
        self.overlap = (bool(overlap) and self.world > 1 and local_apply == self._cuda_apply and not self.fused
                        and not wide_sparse)
        if self.overlap:
            self.g_local, self.g_cols = column_groups(H_local, self.rows_per_rank, self.world, self.rank)
        self._staged = (self.world > 1 and self.device.type == "cuda"
                        and dist.get_backend(group) == dist.Backend.GLOO)

    # ------------------------------------------------------------ fused path
    def _setup_fused(self) -> None:
        """Symmetric-memory X / Y chunks (one per rank, peer-mapped over
        NVLink) for the fused apply: the kernel reads X_C / X_R blocks from
        and reduces Y blocks into the owning rank's chunk directly."""
        import torch.distributed._symmetric_memory as symm_mem

        if self.world > 8:
            raise ValueError("the fused apply supports up to 8 ranks (one NVLink domain)")
        group = self.group if self.group is not None else dist.group.WORLD
        self.Xs = symm_mem.empty(self.rows_per_rank, self.k, dtype=self.dtype, device=self.device)
        self.Ys = symm_mem.empty(self.rows_per_rank, self.k, dtype=self.dtype, device=self.device)
        self.hx = symm_mem.rendezvous(self.Xs, group)
        self.hy = symm_mem.rendezvous(self.Ys, group)
        shape = (self.rows_per_rank, self.k)
        self.x_ptrs = [self.hx.get_remote_tensor(r, shape, self.dtype).data_ptr() for r in range(self.world)]
        self.y_ptrs = [self.hy.get_remote_tensor(r, shape, self.dtype).data_ptr() for r in range(self.world)]

    def _apply_fused(self, xl: torch.Tensor) -> torch.Tensor:
        self.Xs.copy_(xl)
        self.Ys.zero_()
        self.hy.barrier(channel=0)  # every rank's X chunk written and Y chunk zeroed
        sym_spmm_chunked(self.H, self.x_ptrs, self.y_ptrs, self.rows_per_rank, self.k)
        self.hy.barrier(channel=0)  # every rank's reductions into my chunk have landed
        return self.Ys[:, : self.k_user]

    # ------------------------------------------------------------------ build
    @classmethod
    def synthetic(cls, n: int, *, k: int, p: float | None = None, n_off: int | None = None, seed: int = 0,
                  value_seed: int = 0, dtype=torch.float32, device=None, group=None, max_unit: int | None = None,
                  values: str = "h_xor", layout: str | None = None, bands: int | None = 1,
                  fused: bool = False, overlap: bool = False) -> "ShardedSymSpmm":
        """Every rank draws the same global tile pattern (seeded), keeps its
        balanced panel, and generates only its own tile values on its GPU."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        nb = (n + BLOCK - 1) // BLOCK
        if p is None:
            n_pairs = nb * (nb - 1) // 2
            p = 0.0 if n_pairs == 0 else float(n_off or 0) / n_pairs
        rc = synthetic_pattern(nb, p, seed)
        units = plan_units(rc, nb, max_unit)  # None: sized for the global tile count
        _, _, t0, t1 = shard_tile_range(units, world, rank)
        if max_unit is None:
            from .halftiles import auto_max_unit

            max_unit = auto_max_unit(rc.shape[0])
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        H = HalfTiles.synthetic(n, tile_rc=rc[t0:t1], value_seed=value_seed, values=values, dtype=dtype,
                                device=device, max_unit=max_unit, layout=layout, bands=bands)
        H.meta.update(global_tiles=int(rc.shape[0]), global_off_tiles=int(np.count_nonzero(rc[:, 0] != rc[:, 1])),
                      p=p, seed=seed)
        return cls(n, k, dtype, device, H_local=H, group=group, fused=fused, overlap=overlap)

    @classmethod
    def from_halftiles(cls, H: HalfTiles, *, k: int, group=None, fused: bool = False,
                       overlap: bool = False) -> "ShardedSymSpmm":
        """Shard a matrix every rank holds (e.g. built by ``from_basis`` /
        ``from_coo``, dense and sparse tiles): rows are split into panels of
        balanced streamed bytes (``HalfTiles.partition_rows``) and this rank
        keeps its panel (``shard_rows``; views, no copies of dense tiles)."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        b = H.partition_rows(world)
        sub = H.shard_rows(int(b[rank]), int(b[rank + 1]))
        return cls(H.n, k, H.dtype, H.device, H_local=sub, group=group, fused=fused, overlap=overlap)

    def local_tiles(self) -> int:
        """Stored tiles (dense + sparse) in this rank's panel."""
        return self.H.n_tiles + self.H.n_sparse_tiles if self.H is not None else 0

    # ------------------------------------------------------------ exchanges
    def _all_gather(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        if self._staged:  # gloo moves host tensors: stage the CUDA buffers
            o = out.cpu()
            dist.all_gather_into_tensor(o, inp.cpu(), group=self.group)
            out.copy_(o)
            return None
        return dist.all_gather_into_tensor(out, inp, group=self.group, async_op=async_op)

    def _reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if self._staged:
            o = out.cpu()
            dist.reduce_scatter_tensor(o, inp.cpu(), op=dist.ReduceOp.SUM, group=self.group)
            out.copy_(o)
            return
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=self.group)

    def _reduce(self, t: torch.Tensor, dst: int, async_op: bool):
        gdst = dist.get_global_rank(self.group, dst) if self.group is not None else dst
        if self._staged:
            h = t.cpu()
            dist.reduce(h, gdst, op=dist.ReduceOp.SUM, group=self.group)
            if self.rank == dst:
                t.copy_(h)
            return None
        return dist.reduce(t, gdst, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)

    # ------------------------------------------------------------------ apply
    def _cuda_apply(self, X_full: torch.Tensor, Y_part: torch.Tensor) -> None:
        _launch(self.H, X_full[: self.n_pad], Y_part[: self.n_pad], False, None)

    def _launch_ptr(self, H: HalfTiles, x_ptr: int, y: torch.Tensor) -> None:
        """Accumulating apply of a schedule group with X given by its base
        address (global row r at x_ptr + r·k·s)."""
        with torch.cuda.device(self.device):
            check(lib().cim_sym_spmm(H.descriptor(), x_ptr, y.data_ptr(), self.k, self.k, self.k, CIM_ACCUMULATE,
                                     torch.cuda.current_stream(self.device).cuda_stream), "cim_sym_spmm(group)")

    def local_rows(self) -> tuple[int, int]:
        """Global row range [lo, hi) of this rank's X/Y chunk (clipped to n)."""
        lo = self.rank * self.rows_per_rank
        return min(lo, self.n), min(lo + self.rows_per_rank, self.n)

    def apply(self, X_local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Y_local = (A·X)[local rows] given X_local = X[local rows]
        (shape (rows_per_rank, k_user); rows ≥ n must be 0).  ``out``: a
        (rows_per_rank, k_user) buffer to receive Y_local (written in place
        by the kernel / reduce-scatter where the layout allows)."""
        if out is not None:
            if out.shape != (self.rows_per_rank, self.k_user) or out.dtype != self.dtype or out.device != self.device:
                raise ValueError("out must be a (rows_per_rank, k_user) tensor of the operator's dtype and device")
            direct = out.is_contiguous() and self.k == self.k_user and out.data_ptr() % 16 == 0
            if direct and not self.fused and not self.overlap:
                return self._apply_into(X_local, out)
            out.copy_(self.apply(X_local))
            return out
        return self._apply_into(X_local, None)

    def _apply_overlapped(self, xl: torch.Tensor) -> torch.Tensor:
        s = self.X_full.element_size()
        lo = self.rank * self.rows_per_rank
        self.Y_part.zero_()
        work = self._all_gather(self.X_full, xl, async_op=True)
        if self.g_local is not None:  # own-chunk tiles from X_local while the gather is in flight
            self._launch_ptr(self.g_local, xl.data_ptr() - lo * self.k * s, self.Y_part)
        if work is not None:
            work.wait()
        pending = []
        for q in range(self.world - 1, -1, -1):
            g = self.g_cols[q]
            if g is not None:
                self._launch_ptr(g, self.X_full.data_ptr(), self.Y_part)
            sl = self.Y_part[q * self.rows_per_rank:(q + 1) * self.rows_per_rank]
            w = self._reduce(sl, q, async_op=True)  # chunk q is final: reduce it to its owner
            if w is not None:
                pending.append(w)
        for w in pending:
            w.wait()
        return self.Y_part[lo:lo + self.rows_per_rank, : self.k_user]

    def _apply_into(self, X_local: torch.Tensor, out: torch.Tensor | None) -> torch.Tensor:
        if X_local.shape[0] != self.rows_per_rank:
            raise ValueError(f"X_local must have {self.rows_per_rank} rows, got {X_local.shape[0]}")
        if X_local.shape[1] != self.k_user:
            raise ValueError(f"X_local must have {self.k_user} columns, got {X_local.shape[1]}")
        if self.k != self.k_user or not X_local.is_contiguous() or X_local.data_ptr() % 16:
            xl = torch.zeros((self.rows_per_rank, self.k), dtype=self.dtype, device=self.device)
            xl[:, : self.k_user] = X_local
        else:
            xl = X_local
        if self.fused:
            return self._apply_fused(xl)
        if self.overlap:
            return self._apply_overlapped(xl)
        if self.world == 1 and self.local_apply == self._cuda_apply:
            # one rank: the kernel reads X_local and writes Y_local directly
            # (rows_per_rank = n_pad), no staging copies
            Y = self.Y_local if out is None else out
            self._cuda_apply(xl, Y)
            return Y[:, : self.k_user]
        if self.world > 1:
            self._all_gather(self.X_full, xl)
        else:
            self.X_full.copy_(xl)
        self.local_apply(self.X_full, self.Y_part)
        Y = self.Y_local if out is None else out
        if self.world > 1:
            self._reduce_scatter(Y, self.Y_part)
        else:
            Y.copy_(self.Y_part)
        return Y[:, : self.k_user]
