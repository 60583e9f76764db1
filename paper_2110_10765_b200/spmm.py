"""The operator:  Y = H·X + Hᵀ·X  over a half-stored symmetric ``HalfTiles``.

``sym_spmm`` is the B200 drop-in for the reference's pair-walk operator
boundary (``contract_observables``, pkg/src/cimotifs/pipeline.py:534-570):
validate first and raise ``ValueError`` before any compute (:550-555), coerce
inputs to C-contiguous float arrays (:395), write into a caller-owned buffer
or return a fresh array (:569).  Compute happens only in the sm_100a kernel
behind the C-ABI (``cim_sym_spmm``); there is no CPU path.

Layouts: X may be ``(n, k)`` (row-major, what the kernel streams) or
``(k, n)`` — the reference's ``ObservablesInput.c`` layout (n_vec, n),
pipeline.py:387 — selected with ``layout=`` (``"auto"`` prefers (n, k) when
ambiguous).  numpy inputs are copied to the device and the result is returned
as numpy (host buffers in, host buffers out).
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import CIM_ACCUMULATE, CIM_DETERMINISTIC, check, lib
from .halftiles import HalfTiles

LAYOUTS = ("auto", "nk", "kn")


def supported_k(dtype: torch.dtype, k: int, layout: str = "frag") -> bool:
    from .halftiles import LAYOUTS

    code = 0 if dtype == torch.float32 else 1
    return bool(lib().cim_layout_supports(LAYOUTS[layout], code, int(k)))


TC_MAX_K = 64  # f32 vectors per tensor-core apply (N = 2k ≤ 128 TMEM columns per accumulator)
TC_MAX_K_F64 = 64  # f64: one C-ABI call (the DMMA kernel takes ≤ 32; k = 64 runs as two column passes inside)


def tc_max_k(dtype: torch.dtype) -> int:
    return TC_MAX_K if dtype == torch.float32 else TC_MAX_K_F64


def padded_k(dtype: torch.dtype, k: int, layout: str = "frag") -> int:
    """Smallest compiled vector count ≥ k for the layout (extra columns are zero).
    The tensor-core layout takes multiples of 8 up to 64 (f32) / 32 (f64)
    and f64 k = 64 (two column passes of 32 inside the library)."""
    kk = int(k)
    if layout == "tc" and kk > tc_max_k(dtype):
        return -(-kk // tc_max_k(dtype)) * tc_max_k(dtype)
    while kk <= 64 and not supported_k(dtype, kk, layout):
        kk += 1
    if kk > 64:
        raise ValueError(f"k={k} exceeds the largest compiled vector count (64); split X into column blocks")
    return kk


def _launch(H: HalfTiles, Xd: torch.Tensor, Yd: torch.Tensor, accumulate: bool, stream,
            deterministic: bool = False) -> None:
    """Raw C-ABI call on device tensors of shape (n_pad, k) (k compiled)."""
    k = Xd.shape[1]
    s = stream if stream is not None else torch.cuda.current_stream(H.device)
    handle = s.cuda_stream if isinstance(s, torch.cuda.Stream) else int(s)
    if deterministic:
        H.enable_deterministic()
        with torch.cuda.device(H.device):
            rc = lib().cim_sym_spmm(H.descriptor(), Xd.data_ptr(), Yd.data_ptr(), k, Xd.stride(0), Yd.stride(0),
                                    (CIM_ACCUMULATE if accumulate else 0) | CIM_DETERMINISTIC, handle)
        check(rc, "cim_sym_spmm(deterministic)")
        return
    w = tc_max_k(H.dtype)
    if H.layout == "tc" and k > w:
        # column passes of w vectors: each pass streams the tiles once more
        with torch.cuda.stream(s) if isinstance(s, torch.cuda.Stream) else torch.cuda.device(H.device):
            for c0 in range(0, k, w):
                xc = Xd[:, c0:c0 + w].contiguous()
                yc = Yd[:, c0:c0 + w].contiguous() if accumulate else torch.empty_like(xc)
                _launch(H, xc, yc, accumulate, s)
                Yd[:, c0:c0 + w].copy_(yc)
        return
    with torch.cuda.device(H.device):
        rc = lib().cim_sym_spmm(H.descriptor(), Xd.data_ptr(), Yd.data_ptr(), k, Xd.stride(0), Yd.stride(0),
                                CIM_ACCUMULATE if accumulate else 0, handle)
    check(rc, "cim_sym_spmm")


def sym_spmm(H: HalfTiles, X, out=None, *, layout: str = "auto", accumulate: bool = False, stream=None,
             deterministic: bool = False):
    """Y = H·X + Hᵀ·X = A·X for the symmetric A stored as block-half tiles.

    Parameters
    ----------
    H : HalfTiles
    X : torch.Tensor (CUDA or CPU) or numpy array, (n, k) or (k, n), dtype of H
    out : optional tensor/array of X's shape to write into (``accumulate``
        adds to it instead of overwriting)
    layout : "auto" | "nk" | "kn" ("auto" reads the shape; a square X with
        n = k > 1 is ambiguous and raises ValueError)
    stream : torch.cuda.Stream or raw cudaStream_t handle (default: current);
        staging, the kernel and the copy-back all run on it
    deterministic : no float atomics — bitwise reproducible Y (CIM_DETERMINISTIC;
        dense tiles in either layout and sparse tiles; a validation mode, ~2×
        the traffic)
    """
    if not isinstance(H, HalfTiles):
        raise ValueError(f"H must be a HalfTiles, got {type(H).__name__}")
    if stream is not None:
        # stage X, launch and read back Y all on the caller's stream, so the
        # padding copy, the kernel and the copy-back are ordered
        s = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(stream), device=H.device)
        with torch.cuda.stream(s):
            return sym_spmm(H, X, out, layout=layout, accumulate=accumulate, stream=None,
                            deterministic=deterministic)
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}, expected one of {LAYOUTS}")
    is_numpy = isinstance(X, np.ndarray)
    Xt = torch.from_numpy(np.ascontiguousarray(X)) if is_numpy else X
    if not isinstance(Xt, torch.Tensor):
        raise ValueError(f"X must be a torch.Tensor or numpy.ndarray, got {type(X).__name__}")
    if Xt.ndim != 2:
        raise ValueError(f"X must be 2-D (n, k) or (k, n), got shape {tuple(Xt.shape)}")
    if Xt.dtype != H.dtype:
        raise ValueError(f"X dtype {Xt.dtype} does not match the matrix dtype {H.dtype}")
    n = H.n
    if layout == "auto":
        if Xt.shape[0] == n and Xt.shape[1] == n and n > 1:
            raise ValueError(f"X is {n} × {n}: (n, k) and (k, n) are indistinguishable; pass layout='nk' or 'kn'")
        if Xt.shape[0] == n:
            layout = "nk"
        elif Xt.shape[1] == n:
            layout = "kn"
        else:
            raise ValueError(f"X of shape {tuple(Xt.shape)} does not cover the n={n} matrix rows")
    if layout == "nk" and Xt.shape[0] != n:
        raise ValueError(f"X has {Xt.shape[0]} rows, matrix has n={n}")
    if layout == "kn" and Xt.shape[1] != n:
        raise ValueError(f"X covers {Xt.shape[1]} states, matrix has n={n}")
    k = Xt.shape[1] if layout == "nk" else Xt.shape[0]
    if k < 1:
        raise ValueError("X must hold at least one vector")
    if out is not None:
        if tuple(out.shape) != tuple(Xt.shape):
            raise ValueError(f"out has shape {tuple(out.shape)}, expected {tuple(Xt.shape)}")
        if (isinstance(out, np.ndarray) and out.dtype != np.dtype(str(H.dtype).split(".")[-1])) or (
                isinstance(out, torch.Tensor) and out.dtype != H.dtype):
            raise ValueError("out dtype must match the matrix dtype")

    dev = H.device
    kk = padded_k(H.dtype, k, H.layout)
    Xd = Xt.to(dev, non_blocking=True)
    if layout == "kn":
        Xd = Xd.t()
    direct = (Xd.is_contiguous() and kk == k and H.n_pad == n and Xd.data_ptr() % 16 == 0)
    if not direct:
        Xp = torch.zeros((H.n_pad, kk), dtype=H.dtype, device=dev)
        Xp[:n, :k] = Xd
        Xd = Xp
    # output buffer on device, (n_pad, kk) row-major
    out_is_dev_nk = (isinstance(out, torch.Tensor) and out.device == dev and layout == "nk" and direct
                     and out.is_contiguous() and out.data_ptr() % 16 == 0)
    if isinstance(out, torch.Tensor) and out.device == dev and _overlaps(out, Xd):
        raise ValueError("out must not overlap X (Y is zeroed before X is read)")
    if out_is_dev_nk:
        Yd = out
    else:
        Yd = torch.empty((H.n_pad, kk), dtype=H.dtype, device=dev)
        if accumulate and out is not None:
            o = torch.as_tensor(out).to(dev)
            Yd.zero_()
            Yd[:n, :k] = o if layout == "nk" else o.t()
        elif accumulate:
            raise ValueError("accumulate=True needs an `out` buffer to add into")
    _launch(H, Xd, Yd, accumulate, stream, deterministic)
    Y = Yd[:n, :k]
    if layout == "kn":
        Y = Y.t()
    if out_is_dev_nk:
        return out
    if out is not None:
        if isinstance(out, np.ndarray):
            out[...] = Y.cpu().numpy()
        else:
            out.copy_(Y)
        return out
    if is_numpy:
        return Y.cpu().numpy()
    return Y.contiguous() if layout == "kn" else (Y if direct else Y.contiguous())


def _overlaps(a: torch.Tensor, b: torch.Tensor) -> bool:
    """Do the byte ranges of two device tensors intersect?"""
    if a.numel() == 0 or b.numel() == 0:
        return False
    a0 = a.data_ptr()
    a1 = a0 + (sum((s - 1) * st for s, st in zip(a.shape, a.stride())) + 1) * a.element_size()
    b0 = b.data_ptr()
    b1 = b0 + (sum((s - 1) * st for s, st in zip(b.shape, b.stride())) + 1) * b.element_size()
    return a0 < b1 and b0 < a1


def _host_array(A, name: str, n: int, k: int, dtype: torch.dtype) -> torch.Tensor:
    t = torch.from_numpy(A) if isinstance(A, np.ndarray) else A
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a numpy array or CPU tensor, got {type(A).__name__}")
    if t.device.type != "cpu":
        raise ValueError(f"{name} must live in host memory (use sym_spmm for device tensors)")
    if tuple(t.shape) != (n, k):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected ({n}, {k})")
    if t.dtype != dtype:
        raise ValueError(f"{name} dtype {t.dtype} does not match the matrix dtype {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous")
    return t


def sym_spmm_host_batch(H: HalfTiles, Xs, out=None):
    """Y_b = A·X_b for a sequence of HOST (n, k) blocks, pipelined.

    Host copies in, kernel, host copies out of consecutive blocks overlap on
    three streams inside the C-ABI (``cim_sym_spmm_host_batch``): for a
    host-resident workload the apply is PCIe-bound, and steady state costs
    max(H2D, kernel, D2H) per block instead of their sum.  Pass pinned CPU
    tensors (``pin_memory=True``) for asynchronous copies.  Returns the list
    of outputs (``out`` if given, else fresh CPU tensors / numpy arrays
    matching each input).  Synchronous.
    """
    if not isinstance(H, HalfTiles):
        raise ValueError(f"H must be a HalfTiles, got {type(H).__name__}")
    Xs = list(Xs)
    if not Xs:
        return [] if out is None else list(out)
    k = Xs[0].shape[1] if len(Xs[0].shape) == 2 else -1
    if k < 1:
        raise ValueError("each X must be 2-D (n, k) with k >= 1")
    if padded_k(H.dtype, k, H.layout) != k:
        raise ValueError(f"k={k} has no compiled kernel; pad X to k={padded_k(H.dtype, k, H.layout)} vectors")
    xt = [_host_array(X, f"Xs[{b}]", H.n, k, H.dtype) for b, X in enumerate(Xs)]
    if out is None:
        outs = [np.empty((H.n, k), dtype=X.dtype) if isinstance(X, np.ndarray)
                else torch.empty((H.n, k), dtype=H.dtype, pin_memory=X.is_pinned()) for X in Xs]
    else:
        outs = list(out)
        if len(outs) != len(Xs):
            raise ValueError(f"out has {len(outs)} buffers for {len(Xs)} inputs")
    yt = [_host_array(Y, f"out[{b}]", H.n, k, H.dtype) for b, Y in enumerate(outs)]
    import ctypes

    L = lib()
    desc = H.descriptor()
    need = int(L.cim_host_batch_workspace_bytes(desc, k))
    ws = H._workspace(need)
    nb = len(xt)
    xp = (ctypes.c_void_p * nb)(*[t.data_ptr() for t in xt])
    yp = (ctypes.c_void_p * nb)(*[t.data_ptr() for t in yt])
    # the library's streams must not overtake work queued on ours (e.g. the
    # tile-value fill of a matrix built just before this call)
    torch.cuda.current_stream(H.device).synchronize()
    with torch.cuda.device(H.device):
        rc = L.cim_sym_spmm_host_batch(desc, xp, yp, nb, k, ws.data_ptr(), need)
    check(rc, "cim_sym_spmm_host_batch")
    return outs
