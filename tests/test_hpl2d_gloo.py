"""CPU: the P x Q block-cyclic HPL driver (hpl2d.py) over gloo, P > 1.  The
per-rank block operations are the numpy oracle (tests/hpl_numpy_ops.py
NumpyOps2D); the driver's distributed panel (per-column candidate exchange),
cross-rank row interchanges, U12 broadcasts, trailing updates and the
distributed solve are the product code.  The assembled factors, pivots and
growth must equal the single-process oracle LU bit for bit."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_23565_b200.hpl2d import compose_interchanges, global_rows
from test_hpl_dist_gloo import _free_port


@pytest.mark.parametrize("n,nb,P", [(100, 16, 3), (64, 8, 2), (37, 5, 4)])
def test_row_maps(n, nb, P):
    seen = np.zeros(n, dtype=int)
    for p in range(P):
        seen[global_rows(n, nb, P, p)] += 1
    assert np.all(seen == 1)


def test_compose_interchanges_matches_sequential_swaps():
    rng = np.random.default_rng(3)
    for _ in range(50):
        n, j, jb = 60, 10, 12
        piv = np.array([rng.integers(j + t, n) for t in range(jb)])
        rows = np.arange(n)
        for t in range(jb):
            rows[[j + t, piv[t]]] = rows[[piv[t], j + t]]
        dst, src = compose_interchanges(piv, j)
        moved = np.arange(n)
        moved[dst] = src
        assert np.array_equal(moved, rows)


def _worker(rank, world, P, Q, port, n, nb, k, seed, out, mode="gather", lookahead=True):
    import torch.distributed as dist

    from hpl_numpy_ops import NumpyOps2D
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200 import hpl, hpl2d
    from paper_2509_23565_b200.solve import ipiv_to_perm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = orc.hpl_uniform(n, seed)
        grid = hpl2d.Grid(P, Q, hpl.Comm())
        ops = NumpyOps2D(a, nb, P, Q, grid.p, grid.q, k)
        b = hpl2d.rhs_2d(ops, grid).numpy().copy()
        ipiv, growth = hpl2d.factor_2d(ops, grid, n, nb, mode=mode, lookahead=lookahead)
        factored = ops.slab.copy()
        x = hpl2d.solve_2d(ops, grid, n, nb, ipiv_to_perm(ipiv), b)
        out.put((rank, factored, ops.grows, ops.gcols, ipiv, growth, x.numpy().copy(), b))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,lookahead", [("gather", True), ("column", False)])
@pytest.mark.parametrize("n,nb,P,Q,k", [(96, 16, 2, 1, 7), (100, 16, 2, 2, 7), (70, 8, 3, 1, 3),
                                        (90, 12, 2, 2, None), (130, 16, 2, 3, 7)])
def test_pxq_lu_matches_oracle(n, nb, P, Q, k, mode, lookahead):
    """Both panel modes (one all-gather per panel + the whole panel factored
    on every rank of the column, with the side-stream look-ahead of the next
    panel and the two-phase trailing update; or one exchange per panel
    column) give the oracle's factors, pivots and growth bit for bit."""
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200.solve import ipiv_to_perm
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [root, here] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])
    world = P * Q
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, P, Q, port, n, nb, k, 5, out, mode, lookahead))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = orc.hpl_uniform(n, 5)
    lu_ref, perm_ref, growth_ref = orc.lu_factor(a, nb, k)
    lu = np.full((n, n), np.nan)
    for _rank, fac, grows, gcols, ipiv, growth, x, b in res:
        lu[np.ix_(grows, gcols)] = fac
        assert np.array_equal(ipiv_to_perm(ipiv), perm_ref)
        assert growth == growth_ref
        np.testing.assert_allclose(b, a @ np.ones(n), rtol=1e-14, atol=1e-12)
    assert np.array_equal(lu, lu_ref)
    x_ref = orc.lu_solve(lu_ref, perm_ref, a @ np.ones(n))
    for r in res:
        np.testing.assert_allclose(r[6], x_ref, rtol=1e-9, atol=1e-12)
