"""CPU: the multi-GPU host plumbing (row sharding, block-cyclic index maps,
all-gather of shards) with world_size=2 over gloo.  The per-shard compute is
the oracle here (no GPU in this container); on B200s it is the tcgen05 GEMM."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_23565_b200.dist import BlockCyclic, row_shard


def test_row_shard_partitions():
    for m in (1, 7, 100, 16384):
        for world in (1, 2, 3, 8):
            ranges = [row_shard(m, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h - l for l, h in ranges]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n,nb,P,Q", [(1000, 64, 2, 4), (130, 16, 1, 8), (512, 512, 2, 2),
                                      (777, 50, 3, 2)])
def test_block_cyclic_maps_roundtrip(n, nb, P, Q):
    bc = BlockCyclic(n, nb, P, Q)
    counts = np.zeros((P, Q), dtype=np.int64)
    rows_per = [bc.local_shape(bc.rank_of(p, 0))[0] for p in range(P)]
    cols_per = [bc.local_shape(bc.rank_of(0, q))[1] for q in range(Q)]
    assert sum(rows_per) == n and sum(cols_per) == n
    for g in range(n):
        p = (g // nb) % P
        l = bc.g2l(g, P)
        assert bc.l2g(l, p, P) == g
        assert 0 <= l < rows_per[p]
    for gi in range(0, n, 37):
        for gj in range(0, n, 41):
            counts[bc.owner(gi, gj)] += 1
    assert counts.sum() > 0


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
