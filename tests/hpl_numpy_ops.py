"""TEST INFRASTRUCTURE: a numpy stand-in for hpl.DeviceOps, so the
distributed HPL driver (paper_2509_23565_b200/hpl.py) can run its real
host-side logic — block-cyclic maps, panel/pivot broadcasts, interchange
propagation, trailing updates, the distributed solve — over gloo on CPU
ranks.  Every block operation restates the oracle (oracle/ozaki_oracle.py,
i.e. solve.py:66-156 and gemm.py:190-271) on the rank's local columns; the
product never imports this module."""

from __future__ import annotations

import numpy as np
import torch
from scipy.linalg import solve_triangular

from oracle import ozaki_oracle as orc
from paper_2509_23565_b200.hpl import global_cols, local_ncols


class NumpyOps:
    def __init__(self, a_full: np.ndarray, nb: int, Q: int, q: int, k: int | None):
        self.n = a_full.shape[0]
        self.nb, self.Q, self.q, self.k = nb, Q, q, k
        self.full = a_full
        self.ncl = local_ncols(self.n, nb, Q, q)
        self.gcols = global_cols(self.n, nb, Q, q)
        self.slab = np.asfortranarray(a_full[:, self.gcols])
        self.pbuf = [torch.zeros(self.n * nb, dtype=torch.float64) for _ in range(2)]
        self.ipiv_buf = [torch.zeros(nb, dtype=torch.int32) for _ in range(2)]
        self.ipiv = np.zeros(self.n, dtype=np.int32)
        self.flag = 0

    # -- matrix
    def generate(self, *args, **kw):
        self.slab = np.asfortranarray(self.full[:, self.gcols])

    def row_partials(self, x_local=None):
        x = np.ones(self.ncl) if x_local is None else x_local.numpy()
        return (torch.from_numpy(self.slab @ x if self.ncl else np.zeros(self.n)),
                torch.from_numpy(np.abs(self.slab).sum(axis=1)))

    # -- factorization
    def begin(self):
        self.info = 0
        self.seen = 0.0
        self.top = float(np.abs(self.slab).max()) if self.ncl else 0.0

    def panel(self, lc, j, jb, slot=0):
        n = self.n
        a = self.slab
        for t in range(j, j + jb):                               # solve.py:75-90
            c = lc + (t - j)
            p = t + int(np.argmax(np.abs(a[t:, c])))
            if a[p, c] == 0.0 and not self.info:
                self.info = t + 1
            if p != t:
                a[[t, p], lc:lc + jb] = a[[p, t], lc:lc + jb]
            self.ipiv_buf[slot][t - j] = p
            if t + 1 < n:
                a[t + 1:, c] /= a[t, c]
                if t + 1 < j + jb:
                    a[t + 1:, c + 1:lc + jb] -= np.outer(a[t + 1:, c], a[t, c + 1:lc + jb])
                    self.seen = max(self.seen, float(np.abs(a[t + 1:, c + 1:lc + jb]).max()))
        self.seen = max(self.seen, float(np.abs(np.triu(a[j:j + jb, lc:lc + jb])).max()))
        m = n - j
        self.pbuf[slot][:m * jb] = torch.from_numpy(a[j:, lc:lc + jb].ravel(order="F").copy())

    def panel_buffers(self, j, jb, slot=0):
        m = self.n - j
        return self.pbuf[slot][:m * jb], self.ipiv_buf[slot][:jb]

    def record_pivots(self, j, jb, slot=0):
        self.ipiv[j:j + jb] = self.ipiv_buf[slot][:jb].numpy()

    def laswp(self, ranges, j, jb, slot=0):
        cols = np.r_[ranges[0][0]:ranges[0][1], ranges[1][0]:ranges[1][1]].astype(np.int64)
        if cols.size == 0:
            return
        piv = self.ipiv_buf[slot][:jb].numpy()
        for t in range(jb):
            p = int(piv[t])
            if p != j + t:
                tmp = self.slab[j + t, cols].copy()
                self.slab[j + t, cols] = self.slab[p, cols]
                self.slab[p, cols] = tmp

    def _panel(self, j, jb, slot):
        m = self.n - j
        return self.pbuf[slot][:m * jb].numpy().reshape((jb, m)).T   # F-order m x jb

    def trsm_split(self, j, jb, lstart, nt, slot=0):
        pan = self._panel(j, jb, slot)
        a = self.slab
        u12 = solve_triangular(pan[:jb, :jb], a[j:j + jb, lstart:lstart + nt], lower=True,
                               unit_diagonal=True, check_finite=False)
        a[j:j + jb, lstart:lstart + nt] = u12
        self.seen = max(self.seen, float(np.abs(u12).max()))

    def schur_cols(self, j, jb, lstart, nt, c0, c1, slot=0, reserve_sms=0):
        m = self.n - j
        if m - jb <= 0 or c1 <= c0:
            return
        pan = self._panel(j, jb, slot)
        a = self.slab
        cols = slice(lstart + c0, lstart + c1)
        a[j + jb:, cols] = orc.gemm(-1.0, pan[jb:, :], a[j:j + jb, cols], 1.0, a[j + jb:, cols],
                                    k=self.k)
        self.seen = max(self.seen, float(np.abs(a[j + jb:, cols]).max()))

    def finish(self):
        return self.ipiv.copy(), self.info, self.seen, self.top

    # -- solve
    def solve_vector(self, v):
        return torch.from_numpy(np.array(v, dtype=np.float64))

    def trsv(self, lc, j, jb, upper, x):
        blk = self.slab[j:j + jb, lc:lc + jb]
        if upper and np.any(np.diag(blk) == 0.0):
            self.flag = 1
            return
        xs = x[j:j + jb].numpy()
        xs[:] = solve_triangular(blk, xs, lower=not upper, unit_diagonal=not upper,
                                 check_finite=False)

    def gemv_update(self, lc, r0, r1, j, jb, x):
        if r1 > r0:
            xv = x.numpy()
            xv[r0:r1] -= self.slab[r0:r1, lc:lc + jb] @ xv[j:j + jb]

    def zero_diag(self):
        return self.flag
