"""CPU: the multi-GPU host plumbing (row sharding, the block-cyclic column
maps of the distributed LU, all-gather of shards) with world_size=2 over gloo.  The per-shard compute is
the oracle here (no GPU in this container); on B200s it is the tcgen05 GEMM."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_23565_b200.dist import row_shard
from paper_2509_23565_b200.hpl import global_cols, local_cols_before, local_ncols


def test_row_shard_partitions():
    for m in (1, 7, 100, 16384):
        for world in (1, 2, 3, 8):
            ranges = [row_shard(m, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h - l for l, h in ranges]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n,nb,Q", [(1000, 64, 4), (130, 16, 8), (512, 512, 2), (777, 50, 3),
                                    (262144, 1024, 8)])
def test_block_cyclic_maps_roundtrip(n, nb, Q):
    """The 1 x Q (and, per process row/column, P x Q) maps hpl.py / hpl2d.py
    use: column block b lives on rank b % Q as local block b // Q."""
    cols = [global_cols(n, nb, Q, q) for q in range(Q)]
    assert sum(local_ncols(n, nb, Q, q) for q in range(Q)) == n
    allc = np.sort(np.concatenate(cols))
    assert np.array_equal(allc, np.arange(n))
    for q in range(Q):
        assert len(cols[q]) == local_ncols(n, nb, Q, q)
        assert all(((g // nb) % Q) == q for g in cols[q][:: max(1, len(cols[q]) // 50)])
        for g in range(0, n, max(1, n // 97)):
            # local index of the first of q's columns at or after g
            assert local_cols_before(g, nb, Q, q) == int(np.searchsorted(cols[q], g))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200.dist import gemm_row_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        a = rng.random((37, 50)) - 0.5
        b = rng.random((50, 23)) - 0.5
        c = rng.random((37, 23)) - 0.5

        def compute(_bk, alpha, aa, bb, beta, cc):
            return orc.gemm(alpha, aa, bb, beta, cc, k=7)

        out = gemm_row_sharded(None, -1.0, a, b, 1.0, c, compute=compute)
        q.put((rank, bool(np.array_equal(out, orc.gemm(-1.0, a, b, 1.0, c, k=7)))))
    finally:
        dist.destroy_process_group()


def test_row_sharded_gemm_two_ranks_gloo():
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [root, here] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(2):
            rank, ok = q.get(timeout=90)
            results[rank] = ok
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert results == {0: True, 1: True}
