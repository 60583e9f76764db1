"""LOBPCG (BASELINE config 5): the algorithm on CPU with a dense operator
(scipy eigh as oracle), the distributed Gram all-reduce on gloo world 2, and
on the GPU through sym_spmm against scipy eigsh of the oracle-assembled
matrix."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2110_10765_b200.lobpcg import lobpcg


def _dense_sym(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    A = A + A.T
    A += np.diag(np.linspace(-20.0, 20.0, n))  # separated spectrum ends
    return A


def test_lobpcg_dense_cpu_matches_eigh():
    n, m = 400, 6
    A = _dense_sym(n, 1)
    At = torch.from_numpy(A)
    X0 = torch.from_numpy(np.random.default_rng(2).standard_normal((n, m)))
    res = lobpcg(lambda V: At @ V, X0, tol=1e-8, max_iter=500)
    want = np.linalg.eigvalsh(A)[:m]
    assert res.converged
    assert np.allclose(res.eigenvalues, want, rtol=1e-8, atol=1e-8)
    # eigenvector residuals
    X = res.X.numpy()
    r = A @ X - X * res.eigenvalues
    assert np.linalg.norm(r, axis=0).max() <= 1e-6 * np.abs(want).max()


def test_lobpcg_largest():
    n, m = 300, 4
    A = _dense_sym(n, 3)
    At = torch.from_numpy(A)
    X0 = torch.from_numpy(np.random.default_rng(4).standard_normal((n, m)))
    res = lobpcg(lambda V: At @ V, X0, tol=1e-8, max_iter=500, largest=True)
    assert np.allclose(np.sort(res.eigenvalues), np.linalg.eigvalsh(A)[-m:], rtol=1e-8, atol=1e-8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m = 360, 5
        A = torch.from_numpy(_dense_sym(n, 7))
        per = n // world
        rows = slice(rank * per, (rank + 1) * per)
        X0_full = torch.from_numpy(np.random.default_rng(8).standard_normal((n, m)))

        def apply(V_local):
            full = [torch.zeros_like(V_local) for _ in range(world)]
            dist.all_gather(full, V_local)
            return A[rows] @ torch.cat(full)

        res = lobpcg(apply, X0_full[rows].clone(), tol=1e-7, max_iter=500)
        q.put((rank, res.eigenvalues, res.converged))
    finally:
        dist.destroy_process_group()


def test_lobpcg_distributed_gram_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.linalg.eigvalsh(_dense_sym(360, 7))[:5]
    for _, lam, conv in out:
        assert conv
        assert np.allclose(lam, want, rtol=1e-8, atol=1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_lobpcg_gpu_vs_eigsh(dtype):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_10765_b200 as pkg
    from paper_2110_10765_b200.lobpcg import lobpcg_sym

    n, m = 4096, 8
    rc = pkg.synthetic_pattern(n // 64, 0.05, seed=5)
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype)
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0).astype(np.float64)
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    A = sp.csr_matrix((v, (i, j)), shape=(n, n))
    want = np.sort(spla.eigsh(A, k=m, which="SA", tol=1e-10)[0])
    tol = 1e-4 if dtype == torch.float32 else 1e-8
    res = lobpcg_sym(H, m, tol=tol, max_iter=1500, dtype=torch.float64)
    got = np.sort(res.eigenvalues)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= (2e-4 if dtype == torch.float32 else 1e-7) * scale, (got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("derived,m", [(True, 8), (False, 8), (True, 5), (True, 3), (True, 12)])
def test_lobpcg_gpu_f32_blocks_vs_eigsh(derived, m):
    """The f32 native path the C5 bench runs (fast Gram, host-coefficient
    tsmm, fused residual, SpMM into the work buffer, derived or read-back W
    Gram) converges to scipy eigsh's lowest eigenvalues."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_10765_b200 as pkg
    from paper_2110_10765_b200.lobpcg import lobpcg
    from paper_2110_10765_b200.sharded import ShardedSymSpmm

    n = 8192  # m = 3 / 5: padded 8-wide slots (fused Ritz update, λ_j = 0 padding); m = 12: 16-wide slots
    rc = pkg.synthetic_pattern(n // 64, 0.03, seed=11)
    S = ShardedSymSpmm(n, m, torch.float32, torch.device("cuda"),
                       H_local=pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=torch.float32))
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0).astype(np.float64)
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    A = sp.csr_matrix((v, (i, j)), shape=(n, n))
    want = np.sort(spla.eigsh(A, k=m, which="SA", tol=1e-10)[0])
    X0 = torch.randn((S.rows_per_rank, m), generator=torch.Generator().manual_seed(3)).cuda()
    X0[n:] = 0
    res = lobpcg(S.apply, X0, tol=2e-4, max_iter=2000, derived_w_gram=derived)
    assert res.converged
    got = np.sort(res.eigenvalues)
    assert np.abs(got - want).max() <= 2e-5 * np.abs(want).max(), (got, want, res.iterations)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(int(os.environ.get("CIM_LOBPCG_CASES", "8"))))
def test_lobpcg_gpu_randomized(case):
    """Seeded random small problems on the GPU operator (dtype, layout, m,
    largest / lowest, density) against numpy's eigvalsh of the assembled
    matrix."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_10765_b200 as pkg
    from paper_2110_10765_b200.lobpcg import lobpcg_sym

    rng = np.random.default_rng(500 + case)
    dtype = torch.float64 if rng.random() < 0.5 else torch.float32
    layout = "tc" if rng.random() < 0.5 else "frag"
    m = int(rng.integers(1, 11))
    largest = bool(rng.random() < 0.3)
    n = int(rng.integers(300, 1200))
    rc = pkg.synthetic_pattern((n + 63) // 64, float(rng.choice([0.1, 0.3, 1.0])), seed=case)
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0).astype(np.float64)
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    A = np.zeros((n, n))
    np.add.at(A, (i, j), v)
    w = np.linalg.eigvalsh(A)
    want = np.sort(w[-m:] if largest else w[:m])
    res = lobpcg_sym(H, m, tol=1e-7, max_iter=3000, largest=largest, dtype=torch.float64)
    got = np.sort(res.eigenvalues)
    tol = (5e-5 if dtype == torch.float32 else 1e-8) * np.abs(w).max()
    assert np.abs(got - want).max() <= tol, (dtype, layout, m, largest, n, got, want)
