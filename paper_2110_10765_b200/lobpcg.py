"""Block LOBPCG for the lowest eigenpairs of the half-stored symmetric H.

BASELINE.json config 5 / SURVEY.md §8(f) item 1: the eigensolver that wraps
the hot path (Fig. 1 line 15: "LOBPCG ... ⅓–½ of MFDn's
runtime").  The reference itself has no eigensolver, so the
oracle is scipy's ``eigsh`` on the same matrix (tests/test_lobpcg*.py).

Per iteration (Knyazev's LOBPCG, no preconditioner, B = I):

    R  = A X − X Θ                          residuals of the current block
    W  = R ⊥ [X, P]                         (projected, Cholesky-QR)
    AW = A W                                ← the one SpMM of the iteration
    S  = [X, W, P],  AS = [AX, AW, AP]
    G  = Sᵀ AS,  M = Sᵀ S                   (3m × 3m, all-reduced over ranks)
    Rayleigh–Ritz on (G, M) → lowest m Ritz pairs → X, AX, P, AP

The operator is any ``apply(X_local) -> (A X)_local`` on row-distributed
blocks: ``sym_spmm`` on one GPU or ``ShardedSymSpmm.apply`` on N GPUs (rows
sharded as its equal chunks).  Tall-skinny products run on the GPU in the
vector dtype; the 3m × 3m dense problems are solved in float64 on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class LobpcgResult:
    eigenvalues: np.ndarray
    X: torch.Tensor  # local rows of the eigenvector block
    iterations: int
    converged: bool
    residual_norms: np.ndarray
    history: list = field(default_factory=list)
    spmm_calls: int = 0


def _allreduce(t: torch.Tensor, group) -> torch.Tensor:
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


_GRAM_WS: dict = {}


def gram_f64(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """aᵀ·b in float64 on the device through the C-ABI ``cim_gram`` (f32/f64
    tall blocks read once, f64 accumulation, fixed reduction order)."""
    from ._lib import CIM_F32, CIM_F64, check, lib

    if a.shape[0] != b.shape[0] or a.dtype != b.dtype or a.device != b.device:
        raise ValueError("gram operands must share rows, dtype and device")
    if a.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"gram needs float32/float64 blocks, got {a.dtype}")
    if a.stride(1) != 1 or a.stride(0) < a.shape[1]:
        a = a.contiguous()
    if b.stride(1) != 1 or b.stride(0) < b.shape[1]:
        b = b.contiguous()
    rows, ca, cb = a.shape[0], a.shape[1], b.shape[1]
    out = torch.empty((ca, cb), dtype=torch.float64, device=a.device)
    if ca == 0 or cb == 0:
        return out
    L = lib()
    need = int(L.cim_gram_workspace_bytes(rows, ca, cb))
    ws = _GRAM_WS.get(a.device)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=a.device)
        _GRAM_WS[a.device] = ws
    with torch.cuda.device(a.device):
        check(L.cim_gram(a.data_ptr(), a.stride(0), ca, b.data_ptr(), b.stride(0), cb, rows,
                         CIM_F32 if a.dtype == torch.float32 else CIM_F64, out.data_ptr(), ws.data_ptr(), need,
                         torch.cuda.current_stream(a.device).cuda_stream), "cim_gram")
    return out


def _gram(a: torch.Tensor, b: torch.Tensor, group) -> np.ndarray:
    """aᵀ b summed over ranks, in float64 on the host.  CUDA blocks go through
    the native f64-accumulating kernel; CPU blocks (gloo tests, CPU operators)
    through torch in float64."""
    if a.is_cuda:
        g = gram_f64(a, b)
    else:
        g = (a.to(torch.float64).T @ b.to(torch.float64)).contiguous()
    return _allreduce(g, group).cpu().numpy()


def tsmm(A: torch.Tensor, C: torch.Tensor, out: torch.Tensor, alpha: float = 1.0, beta: float = 0.0) -> None:
    """out ← alpha·A·C + beta·out for a tall block A and a small C, writing in
    place into ``out`` (which may be a column-slice view of a wider buffer).
    CUDA float32 goes through the native ``cim_tsmm``; other cases (CPU
    operators in tests, float64) through torch."""
    if A.shape[1] == 0:
        if beta == 0.0:
            out.zero_()
        elif beta != 1.0:
            out.mul_(beta)
        return
    if (A.is_cuda and A.dtype == torch.float32 and A.stride(1) == 1 and out.stride(1) == 1
            and A.shape[1] <= 64 and out.shape[1] <= 64):
        from ._lib import check, lib

        Cd = C.to(A.device, torch.float32).contiguous()
        with torch.cuda.device(A.device):
            check(lib().cim_tsmm(A.data_ptr(), A.stride(0), A.shape[1], Cd.data_ptr(), Cd.shape[1], float(alpha),
                                 float(beta), out.data_ptr(), out.stride(0), A.shape[0],
                                 torch.cuda.current_stream(A.device).cuda_stream), "cim_tsmm")
        return
    prod = A @ C.to(A.device, A.dtype)
    if beta == 0.0:
        out.copy_(prod if alpha == 1.0 else alpha * prod)
    else:
        out.mul_(beta).add_(prod, alpha=alpha)


def _chol_inv_t(M: np.ndarray, eps: float) -> np.ndarray | None:
    """L⁻ᵀ for M = L·Lᵀ when M is numerically positive definite (LAPACK
    condition estimate above ``eps``), else None.  LAPACK's symmetric eigen
    solver costs ~60–80 µs at 24 × 24 on the host — the solver's critical
    path while the GPU waits — where Cholesky, its condition estimate and
    the triangular inverse take ~20 µs."""
    try:
        from scipy.linalg import lapack
    except ImportError:  # the eigenbasis path needs only numpy
        return None
    L, info = lapack.dpotrf(M, lower=1, clean=1)
    if info != 0:
        return None
    rc, info = lapack.dpocon(L, float(np.abs(M).sum(0).max()), uplo="L")
    if info != 0 or not rc > eps:
        return None
    Li, info = lapack.dtrtri(L, lower=1)
    return Li.T if info == 0 else None


def _orth_factor(M: np.ndarray, eps: float = 1e-12) -> np.ndarray:
    """T with (V·T)ᵀ(V·T) = I given M = VᵀV; numerically dependent columns
    are dropped (T has ≤ M.shape[0] columns)."""
    M = 0.5 * (M + M.T)
    T = _chol_inv_t(M, 1e-8)
    if T is not None:
        return T
    w, U = np.linalg.eigh(M)
    keep = w > eps * max(w.max(), 1e-300)
    return U[:, keep] / np.sqrt(w[keep])


def _rayleigh_ritz(G: np.ndarray, M: np.ndarray, m: int, largest: bool, eps: float = 1e-10):
    """Lowest (or largest) m solutions of G c = λ M c with M-orthonormal c.
    Well-conditioned M (the usual case): M = L·Lᵀ, one eigen solve of
    L⁻¹·G·L⁻ᵀ; otherwise M's eigenbasis drops the dependent directions."""
    G = 0.5 * (G + G.T)
    M = 0.5 * (M + M.T)
    T = _chol_inv_t(M, 1e-8)
    if T is None:
        w, U = np.linalg.eigh(M)
        keep = w > eps * w.max()
        T = U[:, keep] / np.sqrt(w[keep])  # Tᵀ M T = I
    lam, Z = np.linalg.eigh(T.T @ G @ T)
    order = np.argsort(lam)[::-1] if largest else np.argsort(lam)
    sel = order[:m]
    return lam[sel], T @ Z[:, sel]


class _Work:
    """Block-major work buffer: six slots [P, X, W, AP, AX, AW], each a
    contiguous (rows × bw) block, bw = m rounded up to a power of two (≥ 4;
    padding columns stay zero).  Slot ranges are handed to the native
    column-blocked kernels (``cim_gram_blocked`` / ``cim_tsmm_blocked``) as
    one operand; a block-major layout keeps every DRAM burst useful, where
    column slices of one wide row-major buffer fetched 4× their bytes."""

    P, X, W, AP, AX, AW = range(6)

    def __init__(self, rows: int, m: int, dtype, device, fast_gram: bool = False):
        self.m, self.rows = m, rows
        self.bw = max(4, 1 << (m - 1).bit_length())
        self.buf = torch.zeros((6, rows, self.bw), dtype=dtype, device=device)
        self.fast_gram = fast_gram and dtype == torch.float32
        # launch state fixed for the solve (the host round trips are on the
        # critical path: no per-call stream / device lookups)
        if self.buf.is_cuda:
            self._stream = torch.cuda.current_stream(self.buf.device).cuda_stream
            self._same_dev = torch.cuda.current_device() == self.buf.device.index
            self._base = self.buf.data_ptr()
            self._slot_bytes = rows * self.bw * self.buf.element_size()
        self._gram_out: dict = {}
        self._vidx: dict = {}

    def _ctx(self):
        import contextlib

        return contextlib.nullcontext() if self._same_dev else torch.cuda.device(self.buf.device)

    def slot(self, s: int, ncols: int | None = None) -> torch.Tensor:
        return self.buf[s][:, : (self.m if ncols is None else ncols)]

    def vidx(self, slots, widths) -> np.ndarray:
        """Virtual column indices (slot-range-relative) of the real columns."""
        key = (len(slots), tuple(widths))
        out = self._vidx.get(key)
        if out is None:
            out = np.concatenate([k * self.bw + np.arange(w) for k, w in enumerate(widths)]).astype(np.int64)
            out.setflags(write=False)
            self._vidx[key] = out
        return out

    def _native(self) -> bool:
        return self.buf.is_cuda and self.buf.dtype in (torch.float32, torch.float64)

    def dense(self, s0: int, s1: int) -> torch.Tensor:
        return self.buf[s0:s1].permute(1, 0, 2).reshape(self.rows, (s1 - s0) * self.bw)

    def gram(self, a0: int, a1: int, b0: int, b1: int, group, block_mask: int = 0) -> np.ndarray:
        """[slots a0..a1)ᵀ·[slots b0..b1) in float64 (virtual columns), summed over ranks.
        ``block_mask`` (bw = 8 only): 8×8 output blocks to compute, bit
        bi·(b1-b0) + bj; 0 = all (the others come back as 0)."""
        ca, cb = (a1 - a0) * self.bw, (b1 - b0) * self.bw
        if self._native() and ca <= 64 and cb <= 64:
            from ._lib import CIM_F32, CIM_F64, CIM_GRAM_FAST, check, lib

            L = lib()
            key = (ca, cb)
            if key not in self._gram_out:
                need = int(L.cim_gram_workspace_bytes(self.rows, ca, cb))
                self._gram_out[key] = (torch.empty((ca, cb), dtype=torch.float64, device=self.buf.device), need,
                                       _workspace(self.buf.device, need))
            out, need, ws = self._gram_out[key]
            if ws.numel() < need or ws is not _WS.get(self.buf.device):
                ws = _workspace(self.buf.device, need)
                self._gram_out[key] = (out, need, ws)
            bs = self.rows * self.bw
            with self._ctx():
                check(L.cim_gram_blocked_ex(self._base + a0 * self._slot_bytes, self.bw, self.bw, bs, ca,
                                            self._base + b0 * self._slot_bytes, self.bw, self.bw, bs, cb, self.rows,
                                            CIM_F32 if self.buf.dtype == torch.float32 else CIM_F64, out.data_ptr(),
                                            ws.data_ptr(), need, block_mask if self.bw == 8 else 0,
                                            CIM_GRAM_FAST if self.fast_gram else 0, self._stream),
                      "cim_gram_blocked_ex")
            return _allreduce(out, group).cpu().numpy()
        if self.buf.is_cuda and (ca > 64 or cb > 64):  # wide blocks: one slot pair at a time, natively
            G = np.zeros((ca, cb))
            for i in range(a0, a1):
                for j in range(b0, b1):
                    G[(i - a0) * self.bw:(i - a0 + 1) * self.bw, (j - b0) * self.bw:(j - b0 + 1) * self.bw] = \
                        self.gram(i, i + 1, j, j + 1, group)
            return G
        return _gram(self.dense(a0, a1), self.dense(b0, b1), group)

    def residual(self, lam: np.ndarray) -> None:
        """W ← AX − X·diag(λ) over the full slots (padding columns of X / AX
        are zero and λ is padded with 0, so W's padding stays zero)."""
        if self._native() and self.buf.dtype == torch.float32:
            from ._lib import check, lib

            lam64 = np.ascontiguousarray(lam, dtype=np.float64)
            with self._ctx():
                check(lib().cim_block_residual(self._base + self.X * self._slot_bytes,
                                               self._base + self.AX * self._slot_bytes, lam64.ctypes.data,
                                               lam64.size, self._base + self.W * self._slot_bytes, self.rows, self.bw,
                                               self._stream), "cim_block_residual")
            return
        lam_p = np.zeros(self.bw)
        lam_p[: lam.size] = lam
        torch.addcmul(self.buf[self.AX], self.buf[self.X], _upload(lam_p, self.buf.dtype, self.buf.device),
                      value=-1.0, out=self.buf[self.W])

    def ritz_update(self, b0: int, CC: np.ndarray, lam: np.ndarray, dst: "_Work") -> bool:
        """dst's [P X] = S·CC, [AP AX] = AS·CC (S = slots b0..AP) and, when
        the fused native kernel runs (bw = 8 f32), also dst's residual
        W = AX − X·diag(λ); returns whether the residual was written."""
        if self._native() and self.buf.dtype == torch.float32 and self.bw == 8 and dst._base != self._base:
            from ._lib import check, lib

            Ch = np.ascontiguousarray(CC, dtype=np.float32)
            lam64 = np.ascontiguousarray(lam, dtype=np.float64)
            with self._ctx():
                check(lib().cim_ritz_update_b8(self._base + b0 * self._slot_bytes,
                                               self._base + (b0 + 3) * self._slot_bytes, self.rows * self.bw,
                                               Ch.shape[0], Ch.ctypes.data, lam64.ctypes.data, lam64.size,
                                               dst._base + self.P * dst._slot_bytes, dst.rows * dst.bw, self.rows,
                                               self._stream), "cim_ritz_update_b8")
            return True
        self.tsmm(b0, self.AP, CC, dst, self.P, self.W)
        self.tsmm(b0 + 3, self.AW + 1, CC, dst, self.AP, self.AW)
        return False

    def tsmm(self, a0: int, a1: int, C: np.ndarray, dst: "_Work", o0: int, o1: int, alpha=1.0, beta=0.0) -> None:
        """dst[slots o0..o1) ← alpha·[slots a0..a1)·C + beta·dst (virtual columns)."""
        q, p = (a1 - a0) * self.bw, (o1 - o0) * self.bw
        if self._native() and self.buf.dtype == torch.float32 and q <= 64 and p <= 64:
            from ._lib import check, lib

            if q * p <= 1024:  # C rides in the kernel parameters: no upload
                Ch = np.ascontiguousarray(C, dtype=np.float32)
                with self._ctx():
                    check(lib().cim_tsmm_blocked_hc(self._base + a0 * self._slot_bytes, self.bw, self.bw,
                                                    self.rows * self.bw, q, Ch.ctypes.data, p, float(alpha),
                                                    float(beta), dst._base + o0 * dst._slot_bytes, self.bw, self.bw,
                                                    self.rows * self.bw, self.rows, self._stream),
                          "cim_tsmm_blocked_hc")
                return
            Cd = _upload(C, torch.float32, self.buf.device)
            with self._ctx():
                check(lib().cim_tsmm_blocked(self._base + a0 * self._slot_bytes, self.bw, self.bw, self.rows * self.bw,
                                             q, Cd.data_ptr(), p, float(alpha), float(beta),
                                             dst._base + o0 * dst._slot_bytes, self.bw, self.bw, self.rows * self.bw,
                                             self.rows, self._stream),
                      "cim_tsmm_blocked")
            return
        prod = self.dense(a0, a1) @ _upload(C, self.buf.dtype, self.buf.device)
        for k, s in enumerate(range(o0, o1)):
            blk = prod[:, k * self.bw:(k + 1) * self.bw]
            if beta == 0.0:
                dst.buf[s].copy_(alpha * blk)
            else:
                dst.buf[s].mul_(beta).add_(blk, alpha=alpha)


_WS: dict = {}
_UP: dict = {}


class _Uploader:
    """Small host → device uploads (the eigensolver's coefficient matrices)
    through a pinned ring, asynchronously: a pageable ``.to(device)`` makes
    torch synchronise the stream, which would stall the host behind every
    queued kernel.  A slot is rewritten only after ``slots`` later uploads,
    and the solver synchronises (Gram read-back) at least once per three
    uploads, so a slot's previous copy has always completed."""

    slots, slot_elems = 16, 64 * 64

    def __init__(self, device):
        self.device = device
        self.host = torch.empty((self.slots, self.slot_elems), dtype=torch.float64, pin_memory=True)
        self.k = 0

    def put(self, a: np.ndarray, dtype) -> torch.Tensor:
        a = np.ascontiguousarray(a)
        if a.size > self.slot_elems:
            return torch.from_numpy(a).to(self.device, dtype)
        h = self.host[self.k % self.slots]
        self.k += 1
        hv = h.view(torch.float32)[: a.size] if dtype == torch.float32 else h[: a.size]
        hv.copy_(torch.from_numpy(a.reshape(-1)).to(hv.dtype))
        return hv.to(self.device, non_blocking=True).view(a.shape)


def _upload(a: np.ndarray, dtype, device) -> torch.Tensor:
    if device.type != "cuda":
        return torch.from_numpy(np.ascontiguousarray(a)).to(device, dtype)
    up = _UP.get(device)
    if up is None:
        up = _UP[device] = _Uploader(device)
    return up.put(a, dtype)


def _workspace(device, nbytes: int) -> torch.Tensor:
    ws = _WS.get(device)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
        _WS[device] = ws
    return ws


_RR_MASKS: dict = {}


def _rr_mask(b0: int) -> int:
    """Block mask of the Sᵀ[S AS] Gram (slots b0..W against P..AW): the 8×8
    slot blocks on and above the diagonals of SᵀS and SᵀAS."""
    mask = _RR_MASKS.get(b0)
    if mask is None:
        ns = _Work.AP - b0
        mask = 0
        for bi in range(ns):
            for bj in range(bi, ns):
                mask |= 1 << (bi * 6 + b0 + bj)
                mask |= 1 << (bi * 6 + b0 + 3 + bj)
        _RR_MASKS[b0] = mask
    return mask


def _embed(M: np.ndarray, rows_idx: np.ndarray, cols_idx: np.ndarray, shape) -> np.ndarray:
    out = np.zeros(shape)
    out[np.ix_(rows_idx, cols_idx)] = M
    return out


def _orthonormalize_slot(work: "_Work", s: int, nv: int, scratch: "_Work", group, passes: int = 2) -> int:
    """Cholesky-QR twice on the first nv columns of slot s (scratch: the same
    slot of another buffer).  Keeps the independent columns, zeroes the rest;
    returns their count."""
    bw = work.bw
    for _ in range(passes):
        T = _orth_factor(work.gram(s, s + 1, s, s + 1, group)[:nv, :nv])
        nk = T.shape[1]
        if nk == 0:
            work.buf[s].zero_()
            return 0
        Tb = _embed(T, np.arange(nv), np.arange(nk), (bw, bw))
        if bw <= 16:  # cim_tsmm reads a row's inputs before writing it when p ≤ 16: in place
            work.tsmm(s, s + 1, Tb, work, s, s + 1)
        else:
            work.tsmm(s, s + 1, Tb, scratch, s, s + 1)
            work.buf[s].copy_(scratch.buf[s])
        nv = nk
    return nv


def lobpcg(apply: Callable[[torch.Tensor], torch.Tensor], X0: torch.Tensor, *, tol: float = 1e-5,
           max_iter: int = 300, largest: bool = False, group=None,
           callback: Callable[[int, np.ndarray, np.ndarray], None] | None = None,
           exact_gram: bool = False, w_orth_passes: int = 1, derived_w_gram: bool = True) -> LobpcgResult:
    """Lowest (default) or largest eigenpairs of the symmetric operator.

    ``X0`` holds this rank's rows of the initial block (n_local × m);
    convergence when every ‖r_j‖ ≤ tol · max(|λ_j|, ‖A‖-scale) where the
    scale is the largest |Ritz value| seen.  ``apply`` maps a contiguous
    (n_local, w) block (w ≤ m) to its image.

    Blocks live in two ping-pong block-major work buffers (``_Work``); Gram
    products run in float64 on the device (``cim_gram_blocked``), block
    updates write in place (``cim_tsmm_blocked``), and only the small
    3m × 3m problems go to the host.  f32 blocks use the fast Gram mode
    (``CIM_GRAM_FAST``: f32 products over ≤ 32-row runs, f64 across runs)
    unless ``exact_gram``.  The projected residual block W gets
    ``w_orth_passes`` Cholesky-QR passes (default one: Rayleigh–Ritz solves
    the generalised problem with the computed SᵀS, so W only needs to be
    well conditioned, not orthonormal to rounding; the initial X gets two).
    With ``derived_w_gram`` (and one pass) the Gram of the projected W is not
    read back from the device: W' = W − B·G with G = BᵀW gives
    W'ᵀW' = WᵀW − 2GᵀG + Gᵀ(BᵀB)G, where WᵀW and G come from the same Gram
    pass as the residual norms and BᵀB = [C_p C]ᵀ(SᵀS)[C_p C] from the last
    Rayleigh–Ritz — one device round trip less per iteration.
    An ``apply`` taking ``out=`` (e.g.
    ``ShardedSymSpmm.apply``) writes AW straight into the work buffer.
    """
    if X0.ndim != 2:
        raise ValueError("X0 must be (n_local, m)")
    rows, m = X0.shape
    dev, dt = X0.device, X0.dtype
    calls = 0
    cur, nxt = _Work(rows, m, dt, dev, not exact_gram), _Work(rows, m, dt, dev, not exact_gram)
    bw = cur.bw
    import inspect

    try:
        apply_out = bw == m and "out" in inspect.signature(apply).parameters
    except (TypeError, ValueError):
        apply_out = False
    Wk = _Work
    cur.slot(Wk.X).copy_(X0)
    if _orthonormalize_slot(cur, Wk.X, m, nxt, group) < m:
        raise ValueError("initial block is rank deficient")
    cur.slot(Wk.AX).copy_(apply(cur.slot(Wk.X).contiguous()))
    calls += 1
    xi = np.arange(m)
    lam, C = _rayleigh_ritz(cur.gram(Wk.X, Wk.X + 1, Wk.AX, Wk.AX + 1, group)[:m, :m],
                            cur.gram(Wk.X, Wk.X + 1, Wk.X, Wk.X + 1, group)[:m, :m], m, largest)
    Cb = _embed(C, xi, xi, (bw, bw))
    cur.tsmm(Wk.X, Wk.X + 1, Cb, nxt, Wk.X, Wk.X + 1)
    cur.tsmm(Wk.AX, Wk.AX + 1, Cb, nxt, Wk.AX, Wk.AX + 1)
    cur, nxt = nxt, cur
    have_p = False
    BtB = None  # [P X]ᵀ[P X] of the current basis (real columns), from the last Rayleigh–Ritz
    history = []
    scale = float(np.abs(lam).max()) or 1.0
    rnorm = np.full(m, np.inf)
    it = 0
    converged = False
    w_ready = False  # W already holds AX − XΛ (written by the fused Ritz update)
    for it in range(1, max_iter + 1):
        # residuals R = AX − X·Λ into the W slot
        # (full bw-wide blocks: padding columns of X / AX are zero, λ padded with 0)
        if not w_ready:
            cur.residual(lam)
        # one Gram pass gives both the residual norms (WᵀW) and the projection
        # coefficients ([P X]ᵀW) — soft locking only selects columns of W
        b0 = Wk.P if have_p else Wk.X
        G_all = cur.gram(b0, Wk.W + 1, Wk.W, Wk.W + 1, group)
        wb = (Wk.W - b0) * bw  # W's rows in G_all
        rnorm = np.sqrt(np.maximum(np.diag(G_all[wb:wb + bw])[:m], 0.0))
        scale = max(scale, float(np.abs(lam).max()))
        history.append((lam.copy(), rnorm.copy()))
        if callback is not None:
            callback(it, lam, rnorm)
        active = rnorm > tol * np.maximum(np.abs(lam), scale)
        if not active.any():
            converged = True
            break
        nw = int(active.sum())
        act = np.flatnonzero(active)
        if nw < m:  # soft locking: keep only the active residual columns
            idx = torch.from_numpy(act).to(dev)
            Wa = cur.slot(Wk.W)[:, idx].clone()
            cur.buf[Wk.W].zero_()
            cur.slot(Wk.W, nw).copy_(Wa)
        # project out the current basis [P X] (or [X]), then orthonormalise
        bidx = cur.vidx(range(b0, Wk.W), [m] * (Wk.W - b0))
        wi = np.arange(nw)
        G_bw = G_all[np.ix_(bidx, act)]
        Gb = _embed(G_bw, bidx, wi, ((Wk.W - b0) * bw, bw))
        if BtB is not None and derived_w_gram and w_orth_passes == 1 and bw <= 16:
            # projection and orthonormalisation in one pass over [P X W]:
            # W ← (W − B·G)·T = W·T − B·(G·T), T from the derived Gram
            WtW = G_all[np.ix_(wb + act, act)]
            T = _orth_factor(WtW - 2.0 * (G_bw.T @ G_bw) + G_bw.T @ BtB @ G_bw)
            nw = T.shape[1]
            if nw > 0:
                Tb = _embed(T, wi, np.arange(nw), (bw, bw))
                cur.tsmm(b0, Wk.W + 1, np.vstack([-Gb @ Tb, Tb]), cur, Wk.W, Wk.W + 1)
        else:
            cur.tsmm(b0, Wk.W, Gb, cur, Wk.W, Wk.W + 1, alpha=-1.0, beta=1.0)
            nw = _orthonormalize_slot(cur, Wk.W, nw, nxt, group, passes=w_orth_passes)
        if nw == 0:
            converged = True
            break
        if apply_out:  # W's unused columns are zero, so A·W over the full block is AW
            apply(cur.buf[Wk.W], out=cur.buf[Wk.AW])
        else:  # the operator takes the solver's m-column blocks; W's columns ≥ nw are zero
            cur.buf[Wk.AW].zero_()
            cur.slot(Wk.AW, m).copy_(apply(cur.slot(Wk.W, m).contiguous()))
        calls += 1
        # Rayleigh–Ritz on S = [P X W] (or [X W]): one Gram pass of S against
        # all six slots gives SᵀS and SᵀAS
        sidx = cur.vidx(range(b0, Wk.AP), [m] * (Wk.W - b0) + [nw])
        # SᵀS and SᵀAS are symmetric: compute the slot blocks on and above
        # their diagonals only (bw = 8: one slot = one 8×8 block), mirror here
        mask = _rr_mask(b0)
        MG = cur.gram(b0, Wk.AP, Wk.P, Wk.AW + 1, group, block_mask=mask)
        if sidx.size == sidx[-1] + 1:  # every column real (m = bw, nothing locked): plain slices
            ns_r = sidx.size
            M = MG[:ns_r, b0 * bw:b0 * bw + ns_r]
            G = MG[:ns_r, (b0 + 3) * bw:(b0 + 3) * bw + ns_r]
        else:
            M = MG[np.ix_(sidx, sidx + b0 * bw)]
            G = MG[np.ix_(sidx, sidx + (b0 + 3) * bw)]
        if bw == 8:
            M = np.triu(M) + np.triu(M, 1).T
            G = np.triu(G) + np.triu(G, 1).T
        lam, C = _rayleigh_ritz(G, M, m, largest)
        # new [P | X] = S·[C_p | C] and [AP | AX] = AS·[C_p | C] into the other buffer,
        # C_p = C with its X rows zeroed (conjugate directions)
        Cp = C.copy()
        xrows = np.flatnonzero((sidx >= (Wk.X - b0) * bw) & (sidx < (Wk.X - b0 + 1) * bw))
        Cp[xrows] = 0.0
        ns = (Wk.AP - b0) * bw
        CC = np.zeros((ns, 2 * bw))
        CC[sidx, :m] = Cp
        CC[sidx, bw:bw + m] = C
        PX = np.hstack([Cp, C])
        BtB = PX.T @ M @ PX
        w_ready = cur.ritz_update(b0, CC, lam, nxt)
        have_p = True
        cur, nxt = nxt, cur
    return LobpcgResult(eigenvalues=lam, X=cur.slot(Wk.X).clone(), iterations=it, converged=converged,
                        residual_norms=rnorm, history=history, spmm_calls=calls)


def lobpcg_sym(H, m: int = 8, *, seed: int = 0, dtype=None, **kw) -> LobpcgResult:
    """LOBPCG on one GPU for a ``HalfTiles`` matrix (apply = sym_spmm)."""
    from .spmm import sym_spmm

    dtype = dtype or H.dtype
    g = torch.Generator(device="cpu").manual_seed(seed)
    X0 = torch.randn((H.n, m), generator=g, dtype=torch.float64).to(H.device, dtype)

    def apply(V: torch.Tensor) -> torch.Tensor:
        return sym_spmm(H, V.to(H.dtype).contiguous()).to(V.dtype)

    return lobpcg(apply, X0, **kw)
