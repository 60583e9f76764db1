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


def _gram(a: torch.Tensor, b: torch.Tensor, group) -> np.ndarray:
    """aᵀ b summed over ranks, in float64 on the host."""
    g = (a.to(torch.float64).T @ b.to(torch.float64)).contiguous()
    return _allreduce(g, group).cpu().numpy()


def _orthonormalize(V: torch.Tensor, group, eps: float = 1e-12) -> torch.Tensor:
    """Cholesky-QR (twice for stability) of a distributed tall block; columns
    that are numerically dependent are dropped."""
    for _ in range(2):
        M = _gram(V, V, group)
        M = 0.5 * (M + M.T)
        w, U = np.linalg.eigh(M)
        keep = w > eps * max(w.max(), 1e-300)
        if not keep.any():
            return V[:, :0]
        T = U[:, keep] / np.sqrt(w[keep])  # V·T has orthonormal columns
        V = V @ torch.from_numpy(T).to(V.device, V.dtype)
    return V


def _rayleigh_ritz(G: np.ndarray, M: np.ndarray, m: int, largest: bool, eps: float = 1e-10):
    """Lowest (or largest) m solutions of G c = λ M c with M-orthonormal c."""
    G = 0.5 * (G + G.T)
    M = 0.5 * (M + M.T)
    w, U = np.linalg.eigh(M)
    keep = w > eps * w.max()
    T = U[:, keep] / np.sqrt(w[keep])  # Tᵀ M T = I
    lam, Z = np.linalg.eigh(T.T @ G @ T)
    order = np.argsort(lam)[::-1] if largest else np.argsort(lam)
    sel = order[:m]
    return lam[sel], T @ Z[:, sel]


def lobpcg(apply: Callable[[torch.Tensor], torch.Tensor], X0: torch.Tensor, *, tol: float = 1e-5,
           max_iter: int = 300, largest: bool = False, group=None,
           callback: Callable[[int, np.ndarray, np.ndarray], None] | None = None) -> LobpcgResult:
    """Lowest (default) or largest eigenpairs of the symmetric operator.

    ``X0`` holds this rank's rows of the initial block (n_local × m);
    convergence when every ‖r_j‖ ≤ tol · max(|λ_j|, ‖A‖-scale) where the
    scale is the largest |Ritz value| seen.
    """
    if X0.ndim != 2:
        raise ValueError("X0 must be (n_local, m)")
    m = X0.shape[1]
    calls = 0
    X = _orthonormalize(X0, group)
    if X.shape[1] < m:
        raise ValueError("initial block is rank deficient")
    AX = apply(X)
    calls += 1
    lam, C = _rayleigh_ritz(_gram(X, AX, group), _gram(X, X, group), m, largest)
    Ct = torch.from_numpy(C).to(X.device, X.dtype)
    X, AX = X @ Ct, AX @ Ct
    P = AP = None
    history = []
    scale = float(np.abs(lam).max()) or 1.0
    rnorm = np.full(m, np.inf)
    it = 0
    converged = False
    for it in range(1, max_iter + 1):
        lam_t = torch.from_numpy(lam).to(X.device, X.dtype)
        R = AX - X * lam_t
        rnorm = np.sqrt(np.maximum(np.diag(_gram(R, R, group)), 0.0))
        scale = max(scale, float(np.abs(lam).max()))
        history.append((lam.copy(), rnorm.copy()))
        if callback is not None:
            callback(it, lam, rnorm)
        active = rnorm > tol * np.maximum(np.abs(lam), scale)
        if not active.any():
            converged = True
            break
        W = R[:, torch.from_numpy(np.flatnonzero(active)).to(R.device)]
        # project out the current basis, then orthonormalise
        basis = [X] if P is None else [X, P]
        for B in basis:
            W = W - B @ torch.from_numpy(_gram(B, W, group)).to(W.device, W.dtype)
        W = _orthonormalize(W, group)
        if W.shape[1] == 0:
            converged = True
            break
        AW = apply(W)
        calls += 1
        S = [X, W] + ([P] if P is not None else [])
        AS = [AX, AW] + ([AP] if AP is not None else [])
        Sm = torch.cat(S, dim=1)
        ASm = torch.cat(AS, dim=1)
        lam, C = _rayleigh_ritz(_gram(Sm, ASm, group), _gram(Sm, Sm, group), m, largest)
        Ct = torch.from_numpy(C).to(X.device, X.dtype)
        Xn = Sm @ Ct
        AXn = ASm @ Ct
        # conjugate directions: the W and P parts of the new Ritz vectors
        Cp = Ct.clone()
        Cp[:m] = 0
        P = Sm @ Cp
        AP = ASm @ Cp
        X, AX = Xn, AXn
    return LobpcgResult(eigenvalues=lam, X=X, iterations=it, converged=converged, residual_norms=rnorm,
                        history=history, spmm_calls=calls)


def lobpcg_sym(H, m: int = 8, *, seed: int = 0, dtype=None, **kw) -> LobpcgResult:
    """LOBPCG on one GPU for a ``HalfTiles`` matrix (apply = sym_spmm)."""
    from .spmm import sym_spmm

    dtype = dtype or H.dtype
    g = torch.Generator(device="cpu").manual_seed(seed)
    X0 = torch.randn((H.n, m), generator=g, dtype=torch.float64).to(H.device, dtype)

    def apply(V: torch.Tensor) -> torch.Tensor:
        return sym_spmm(H, V.to(H.dtype).contiguous()).to(V.dtype)

    return lobpcg(apply, X0, **kw)
