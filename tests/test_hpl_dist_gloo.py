"""CPU: the distributed HPL driver (hpl.py: 1 x Q block-cyclic LU + solve)
over gloo with world sizes 2 and 3.  The per-rank block operations are the
numpy oracle (tests/hpl_numpy_ops.py); everything else — the block-cyclic
maps, panel and pivot broadcasts, interchange propagation to every rank's
columns, the trailing updates and the distributed triangular solves — is the
product driver.  The assembled factors must equal the single-process oracle
LU bit for bit (the emulated Schur update is per-element independent of the
column partition), pivots and growth included."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_23565_b200.hpl import global_cols, local_cols_before, local_ncols


@pytest.mark.parametrize("n,nb,Q", [(100, 16, 3), (64, 8, 2), (37, 5, 4), (512, 64, 8)])
def test_block_cyclic_column_maps(n, nb, Q):
    seen = np.zeros(n, dtype=int)
    for q in range(Q):
        g = global_cols(n, nb, Q, q)
        assert len(g) == local_ncols(n, nb, Q, q)
        assert np.all(np.diff(g) > 0)
        seen[g] += 1
        for gg in range(0, n + 1, 3):
            assert local_cols_before(gg, nb, Q, q) == int(np.sum(g < gg))
        for b in range(q, -(-n // nb), Q):                       # owner's panel column
            assert g[(b // Q) * nb] == b * nb
    assert np.all(seen == 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, nb, k, seed, out, lookahead=True):
    import torch.distributed as dist

    from hpl_numpy_ops import NumpyOps
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200 import hpl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = orc.hpl_uniform(n, seed)
        comm = hpl.Comm()
        ops = NumpyOps(a, nb, world, rank, k)
        b = a @ np.ones(n)
        ipiv, growth = hpl.factor_block_cyclic(ops, comm, n, nb, lookahead=lookahead)
        factored = ops.slab.copy()
        from paper_2509_23565_b200.solve import ipiv_to_perm
        perm = ipiv_to_perm(ipiv)
        x = hpl.solve_block_cyclic(ops, comm, n, nb, perm, b)
        out.put((rank, factored, ops.gcols, ipiv, growth, x.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nb,world,k,la", [(96, 16, 2, 7, True), (100, 16, 3, 7, True),
                                             (90, 12, 2, None, True), (70, 8, 3, 3, True),
                                             (100, 16, 3, 7, False)])
def test_distributed_lu_matches_oracle(n, nb, world, k, la):
    from oracle import ozaki_oracle as orc
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [root, here] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, k, 5, out, la))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [out.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = orc.hpl_uniform(n, 5)
    lu_ref, perm_ref, growth_ref = orc.lu_factor(a, nb, k)
    lu = np.zeros((n, n))
    for _rank, fac, gcols, ipiv, growth, x in res:
        lu[:, gcols] = fac
        from paper_2509_23565_b200.solve import ipiv_to_perm
        assert np.array_equal(ipiv_to_perm(ipiv), perm_ref)
        assert growth == growth_ref
    assert np.array_equal(lu, lu_ref)
    x_ref = orc.lu_solve(lu_ref, perm_ref, a @ np.ones(n))
    for r in res:
        np.testing.assert_allclose(r[5], x_ref, rtol=1e-9, atol=1e-12)
        assert orc.residual(a, r[5], a @ np.ones(n))[0] < 16.0 or k == 3
