"""GPU: one panel leaf (oz_lu_panel with jb <= the leaf width) against the
reference's unblocked loop (solve.py:75-90) restated in numpy: pivots (np.argmax
order, ties to the first row), factors and the zero-pivot report bit for bit.

Small-integer entries make ties between candidate rows frequent, which is
where a distributed argmax can go wrong.  Heights cover every leaf variant:
register leaf with one cluster of 128-row CTAs (m <= 2048), 256-row CTAs
(m <= 4096), two rows per thread (m <= 8192, 32-column windows), and the
register leaf with the global-memory exchange beyond (256 rows per CTA up to
the SM count, then 512 with 32-column windows, then 1024 / 2048 with 16 / 8
columns on capped grids)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _reference_panel(a):
    """solve.py:75-90 on an m x jb panel (rows swapped within the panel)."""
    a = np.array(a, dtype=np.float64, order="F", copy=True)
    m, jb = a.shape
    piv = np.zeros(jb, dtype=np.int64)
    zero = 0
    for t in range(jb):
        p = t + int(np.argmax(np.abs(a[t:, t])))
        piv[t] = p
        if a[p, t] == 0.0:
            zero = zero or t + 1
            continue
        if p != t:
            a[[t, p], :] = a[[p, t], :]
        if t + 1 < m:
            a[t + 1:, t] /= a[t, t]
            if t + 1 < jb:
                a[t + 1:, t + 1:] -= np.outer(a[t + 1:, t], a[t, t + 1:])
    return a, piv, zero


def _device_panel(a, max_ctas=0):
    import torch

    from paper_2509_23565_b200 import _dev, _lib
    m, jb = a.shape
    d = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()     # column-major m x jb
    wsb = int(_lib.query("oz_lu_workspace_bytes", m, jb, 0, 7))
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    _lib.call("oz_lu_ws_init", ws.data_ptr(), wsb, m, jb, 0, _dev.stream())
    ipiv = torch.zeros((jb,), dtype=torch.int32, device="cuda")
    info = torch.zeros((1,), dtype=torch.int32, device="cuda")
    bits = torch.zeros((2,), dtype=torch.int64, device="cuda")
    _lib.call("oz_lu_panel", d.data_ptr(), m, m, jb, 0, ipiv.data_ptr(), info.data_ptr(),
              bits.data_ptr(), ws.data_ptr(), wsb, m, jb, 0, max_ctas, _dev.stream())
    torch.cuda.synchronize()
    return d.cpu().numpy().T, ipiv.cpu().numpy(), int(info.item())


@pytest.mark.parametrize("m,jb", [(70, 64), (300, 64), (2048, 64), (2049, 64), (4096, 64),
                                  (5000, 32), (8192, 32), (12000, 16), (12000, 64),
                                  (40000, 32)])
def test_leaf_ties_match_reference(m, jb):
    rng = np.random.default_rng(m)
    a = rng.integers(-4, 5, size=(m, jb)).astype(np.float64)
    want, piv, zero = _reference_panel(a)
    got, ipiv, info = _device_panel(a)
    assert zero == 0 and info == 0
    assert np.array_equal(ipiv, piv)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m,jb,ctas", [(12000, 16, 12), (5000, 16, 5)])
def test_tall_leaf_ties_match_reference(m, jb, ctas):
    """The tall register variants on a capped grid (look-ahead side stream):
    1024 rows per CTA with 16-column windows, 2048 with 8-column windows."""
    rng = np.random.default_rng(m + ctas)
    a = rng.integers(-4, 5, size=(m, jb)).astype(np.float64)
    want, piv, zero = _reference_panel(a)
    got, ipiv, info = _device_panel(a, ctas)
    assert zero == 0 and info == 0
    assert np.array_equal(ipiv, piv)
    assert np.array_equal(got, want)


def test_leaf_zero_pivot_reported():
    """An exact zero pivot column (solve.py:78-79): the leaf reports the first
    such column (global index + 1) and keeps going, like the reference's loop
    up to the point where it raises."""
    rng = np.random.default_rng(5)
    m, jb = 1000, 64
    a = rng.random((m, jb)) - 0.5
    a[:, 5] = 0.0                      # stays exactly zero under the updates: zero pivot at t = 5
    want, piv, zero = _reference_panel(a)
    got, ipiv, info = _device_panel(a)
    assert zero != 0 and info == zero
    assert np.array_equal(ipiv[:zero - 1], piv[:zero - 1])
