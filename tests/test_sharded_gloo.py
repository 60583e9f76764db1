"""Multi-rank row-block sharding on CPU (gloo, world_size 2 and 3).

The per-rank panel product is injected as the f64 oracle (test-only hook); the
partition (native ``cim_partition_units``), the equal X/Y row chunks, the
all-gather and the reduce-scatter are the product code under test.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, p, seed, k, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2110_10765_b200 as pkg
        from paper_2110_10765_b200.sharded import ShardedSymSpmm, shard_tile_range

        nb = (n + 63) // 64
        rc = pkg.synthetic_pattern(nb, p, seed)
        units = pkg.plan_units(rc, nb, max_unit=3)
        _, _, t0, t1 = shard_tile_range(units, world, rank)
        my_rc = rc[t0:t1]
        my_tiles = oracle.synthetic_dense_tiles(n, my_rc, seed=0)

        def local_apply(X_full, Y_part):
            Y = oracle.sym_spmm(n, my_rc, my_tiles, X_full[:n].numpy()) if my_rc.shape[0] else np.zeros((n, k))
            Y_part.zero_()
            Y_part[:n] = torch.from_numpy(Y)

        S = ShardedSymSpmm(n, k, torch.float64, "cpu", group=None, local_apply=local_apply)
        g = torch.Generator().manual_seed(1)
        X = torch.randn((S.rows_total, k), generator=g, dtype=torch.float64)
        X[n:] = 0
        lo = rank * S.rows_per_rank
        Y_local = S.apply(X[lo:lo + S.rows_per_rank].clone())
        # apply(out=): the reduce-scatter lands in the caller's buffer
        out = torch.full((S.rows_per_rank, k), 7.0, dtype=torch.float64)
        Y_out = S.apply(X[lo:lo + S.rows_per_rank].clone(), out=out)
        assert Y_out.data_ptr() == out.data_ptr() and torch.equal(out, Y_local)
        result_q.put((rank, lo, Y_local.numpy().copy(), t1 - t0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_oracle(world):
    n, p, seed, k = 1000, 0.3, 4, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, seed, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    nb = (n + 63) // 64
    import paper_2110_10765_b200 as pkg

    rc = pkg.synthetic_pattern(nb, p, seed)
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0)
    g = torch.Generator().manual_seed(1)
    per = ((nb + world - 1) // world) * 64
    X = torch.randn((per * world, k), generator=g, dtype=torch.float64)
    X[n:] = 0
    Y_ref = oracle.sym_spmm(n, rc, tiles, X[:n].numpy())
    Y = np.zeros((per * world, k))
    counts = []
    for rank, lo, yl, nt in res:
        Y[lo:lo + yl.shape[0]] = yl
        counts.append(nt)
    assert sum(counts) == rc.shape[0]  # every tile owned by exactly one rank
    assert np.abs(Y[:n] - Y_ref).max() <= 1e-12 * np.abs(Y_ref).max()
    assert np.all(Y[n:] == 0)
