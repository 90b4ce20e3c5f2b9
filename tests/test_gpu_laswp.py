"""GPU: oz_laswp (compose the panel's sequential interchanges into one gather
list, apply it to column ranges) against the reference's row swaps replayed
in order (solve.py:80-82, LAPACK dlaswp order), bit for bit.  Pivot patterns
cover self-swaps, rows inside the panel block, rows far below it touched by
several steps, and the full 1024-interchange panel."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _reference(a, k1, piv):
    a = a.copy()
    for t, p in enumerate(piv):
        r = k1 + t
        if p != r:
            a[[r, p], :] = a[[p, r], :]
    return a


def _device(a, k1, piv, c0a, c1a, c0b, c1b):
    import torch

    from paper_2509_23565_b200 import _dev, _lib
    m, n = a.shape
    d = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()   # column-major m x n
    ip = torch.from_numpy(np.asarray(piv, dtype=np.int32)).cuda()
    nb = max(len(piv), 1)
    wsb = int(_lib.query("oz_lu_workspace_bytes", m, nb, 0, 7))
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    _lib.call("oz_lu_ws_init", ws.data_ptr(), wsb, m, nb, 0, _dev.stream())
    _lib.call("oz_laswp", d.data_ptr(), m, c0a, c1a, c0b, c1b, k1, ip.data_ptr(), len(piv),
              ws.data_ptr(), wsb, m, nb, 0, _dev.stream())
    torch.cuda.synchronize()
    return d.cpu().numpy().T


def _pivots(rng, kind, k1, npiv, m):
    t = np.arange(npiv)
    if kind == "random":
        return k1 + t + (rng.random(npiv) * (m - k1 - t)).astype(np.int64)
    if kind == "block":          # pivots inside the panel block only
        return k1 + t + (rng.random(npiv) * (npiv - t)).astype(np.int64)
    if kind == "repeat_far":     # few far rows, each touched by many steps
        far = k1 + npiv + rng.integers(0, 4, size=npiv)
        self_ = rng.random(npiv) < 0.2
        return np.where(self_, k1 + t, far)
    if kind == "identity":
        return k1 + t
    if kind == "general":        # rows above their step too (not getrf output; dlaswp allows it)
        return k1 + (rng.random(npiv) * (m - k1)).astype(np.int64)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["random", "block", "repeat_far", "identity", "general"])
@pytest.mark.parametrize("npiv", [1, 37, 1024])
def test_laswp_matches_sequential_swaps(kind, npiv):
    rng = np.random.default_rng(npiv * 7 + len(kind))
    m, n, k1 = 3000, 24, 500
    a = rng.random((m, n))
    piv = _pivots(rng, kind, k1, npiv, m)
    want = _reference(a, k1, piv)
    got = _device(a, k1, piv, 0, 10, 14, n)           # two column ranges
    assert np.array_equal(got[:, :10], want[:, :10])
    assert np.array_equal(got[:, 14:], want[:, 14:])
    assert np.array_equal(got[:, 10:14], a[:, 10:14])  # columns outside the ranges untouched
