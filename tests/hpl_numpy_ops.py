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

    def lookahead_sms(self, m, ncols):
        return 16

    def lookahead_cols1(self, m, rest_cols, sms):
        # two-phase split point: exercise both phases of the driver
        return rest_cols // 2

    # -- streams (the device ops run the look-ahead panel on a side stream)
    def side_stream(self):
        import contextlib
        return contextlib.nullcontext()

    def join_side(self):
        pass

    # -- factorization
    def begin(self):
        self.info = 0
        self.seen = 0.0
        self.top = float(np.abs(self.slab).max()) if self.ncl else 0.0

    def panel(self, lc, j, jb, slot=0, max_ctas=0):
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


class NumpyOps2D:
    """The same stand-in for hpl2d.DeviceOps2D (P x Q grid): local rows x
    local columns of the oracle's matrix; every operation restates the
    oracle on those blocks (dpanel.cu's column step = solve.py:75-90)."""

    def __init__(self, a_full: np.ndarray, nb: int, P: int, Q: int, p: int, q: int,
                 k: int | None):
        from paper_2509_23565_b200.hpl2d import global_rows
        self.n = a_full.shape[0]
        self.nb, self.P, self.Q, self.p, self.q, self.k = nb, P, Q, p, q, k
        self.full = a_full
        self.grows = global_rows(self.n, nb, P, p)
        self.gcols = global_rows(self.n, nb, Q, q)
        self.mloc, self.ncl = len(self.grows), len(self.gcols)
        self.slab = np.asfortranarray(a_full[np.ix_(self.grows, self.gcols)])
        self.pbufs = [torch.zeros(max(self.mloc, 1) * nb, dtype=torch.float64)
                      for _ in range(2)]
        self.ubuf = torch.zeros(nb * max(self.ncl, 1), dtype=torch.float64)
        self.ipiv_bufs = [torch.zeros(nb, dtype=torch.int32) for _ in range(2)]
        self.ipiv = np.zeros(self.n, dtype=np.int32)
        self.flag = 0

    def generate(self, *args, **kw):
        self.slab = np.asfortranarray(self.full[np.ix_(self.grows, self.gcols)])

    # -- look-ahead (hpl2d.factor_2d): sizes only matter on the device
    def lookahead_sms(self, m, ncols):
        return 16

    def lookahead_cols1(self, m, rest_cols, sms):
        return rest_cols // 2            # exercise both phases

    def side_stream(self):
        import contextlib
        return contextlib.nullcontext()

    def join_side(self):
        pass

    def vector(self, host=None, n=None):
        if host is None:
            return torch.zeros(n, dtype=torch.float64)
        return torch.from_numpy(np.array(host, dtype=np.float64))

    def row_partials(self, x_local=None):
        x = np.ones(self.ncl) if x_local is None else x_local.numpy()
        ax, asum = np.zeros(self.n), np.zeros(self.n)
        ax[self.grows] = self.slab @ x if self.ncl else 0.0
        asum[self.grows] = np.abs(self.slab).sum(axis=1)
        return torch.from_numpy(ax), torch.from_numpy(asum)

    def begin(self):
        self.info = 0
        self.seen = 0.0
        self.top = float(np.abs(self.slab).max()) if self.slab.size else 0.0

    def dpanel_candidate(self, lc, lr0, t, jb, owns_g):
        rec = np.zeros(3 + 2 * jb)
        col = self.slab[lr0:, lc + t]
        if col.size == 0:
            rec[0] = rec[1] = -1.0
        else:
            i = int(np.argmax(np.abs(col)))
            rec[0], rec[1] = abs(col[i]), self.grows[lr0 + i]
            rec[3:3 + jb] = self.slab[lr0 + i, lc:lc + jb]
        rec[2] = 1.0 if owns_g else 0.0
        if owns_g:
            rec[3 + jb:] = self.slab[lr0, lc:lc + jb]
        return torch.from_numpy(rec)

    def dpanel_apply(self, lc, lr0, t, jb, g, owns_g, recs):
        r = recs.numpy()
        w = 0
        for i in range(1, r.shape[0]):
            if r[i, 0] > r[w, 0] or (r[i, 0] == r[w, 0] >= 0 and r[i, 1] < r[w, 1]):
                w = i
        rw = r[w]
        rg = r[int(np.nonzero(r[:, 2])[0][0])]
        piv = int(rw[1])
        self.ipiv_bufs[0][t] = piv
        if rw[3 + t] == 0.0 and not self.info:
            self.info = g + 1
        a = self.slab
        if piv != g:
            if owns_g:
                a[lr0, lc:lc + jb] = rw[3:3 + jb]
            if (piv // self.nb) % self.P == self.p:
                lrp = ((piv // self.nb) // self.P) * self.nb + piv % self.nb
                a[lrp, lc:lc + jb] = rg[3 + jb:]
        r0 = lr0 + (1 if owns_g else 0)
        pv = rw[3 + t]
        if pv != 0.0 and r0 < self.mloc:
            a[r0:, lc + t] /= pv
            if t + 1 < jb:
                a[r0:, lc + t + 1:lc + jb] -= np.outer(a[r0:, lc + t], rw[3 + t + 1:3 + jb])
                self.seen = max(self.seen, float(np.abs(a[r0:, lc + t + 1:lc + jb]).max()))

    def panel_pack(self, lc, lr_j, jb, R):
        buf = np.zeros((jb, max(R, 1)))
        mine = self.mloc - lr_j
        if mine > 0:
            buf[:, :mine] = self.slab[lr_j:, lc:lc + jb].T
        return torch.from_numpy(buf.ravel().copy())

    def panel_from_gathered(self, allp, lc, lr_j, j, jb, R, slot=0, max_ctas=0):
        """The gathered panel factored by the reference's unblocked loop
        (solve.py:75-90) on the global m x jb panel; own rows written back."""
        from paper_2509_23565_b200.hpl import local_cols_before
        n, nb, P = self.n, self.nb, self.P
        blocks = allp.numpy().reshape((P, jb, max(R, 1)))
        g = np.arange(j, n)
        owner = (g // nb) % P
        lrj = np.array([local_cols_before(j, nb, P, o) for o in range(P)])
        row = ((g // nb) // P) * nb + g % nb - lrj[owner]
        pan = np.asfortranarray(blocks[owner, :, row])          # m x jb
        m = n - j
        for t in range(jb):
            pr = t + int(np.argmax(np.abs(pan[t:, t])))
            self.ipiv_bufs[slot][t] = j + pr
            if pan[pr, t] == 0.0:
                if not self.info:
                    self.info = j + t + 1
                continue
            if pr != t:
                pan[[t, pr], :] = pan[[pr, t], :]
            if t + 1 < m:
                pan[t + 1:, t] /= pan[t, t]
                if t + 1 < jb:
                    pan[t + 1:, t + 1:] -= np.outer(pan[t + 1:, t], pan[t, t + 1:])
                    self.seen = max(self.seen, float(np.abs(pan[t + 1:, t + 1:]).max()))
        mine = self.mloc - lr_j
        if mine > 0:
            self.slab[lr_j:, lc:lc + jb] = pan[self.grows[lr_j:] - j, :]

    def panel_finish(self, lc, lr_j, jb, diag, slot=0):
        if diag:
            self.seen = max(self.seen, float(np.abs(np.triu(
                self.slab[lr_j:lr_j + jb, lc:lc + jb])).max()))
        m = self.mloc - lr_j
        if m > 0:
            self.pbufs[slot][:m * jb] = torch.from_numpy(
                self.slab[lr_j:, lc:lc + jb].ravel(order="F").copy())

    def panel_buffers(self, lr_j, jb, slot=0):
        return self.pbufs[slot][:(self.mloc - lr_j) * jb], self.ipiv_bufs[slot][:jb]

    def record_pivots(self, j, jb, slot=0):
        self.ipiv[j:j + jb] = self.ipiv_bufs[slot][:jb].numpy()
        return self.ipiv[j:j + jb].copy()

    @staticmethod
    def _cols(ranges):
        return np.r_[ranges[0][0]:ranges[0][1], ranges[1][0]:ranges[1][1]].astype(np.int64)

    def gather_rows(self, lrows, ranges):
        blk = self.slab[np.ix_(np.asarray(lrows), self._cols(ranges))]
        return torch.from_numpy(blk.ravel(order="F").copy())

    def rows_buffer(self, nrows, ranges):
        return torch.zeros(nrows * len(self._cols(ranges)), dtype=torch.float64)

    def scatter_rows(self, lrows, ranges, buf, brows, ldb):
        if len(lrows) == 0:
            return
        cols = self._cols(ranges)
        b = buf.numpy().reshape((len(cols), ldb)).T
        self.slab[np.ix_(np.asarray(lrows), cols)] = b[np.asarray(brows), :]

    def _pan(self, lr_j, jb, slot=0):
        m = self.mloc - lr_j
        return self.pbufs[slot][:m * jb].numpy().reshape((jb, m)).T

    def trsm(self, lr_j, jb, lstart, nt, slot=0):
        pan = self._pan(lr_j, jb, slot)
        u12 = solve_triangular(pan[:jb, :jb], self.slab[lr_j:lr_j + jb, lstart:lstart + nt],
                               lower=True, unit_diagonal=True, check_finite=False)
        self.slab[lr_j:lr_j + jb, lstart:lstart + nt] = u12
        self.seen = max(self.seen, float(np.abs(u12).max()))
        self.ubuf[:jb * nt] = torch.from_numpy(u12.ravel(order="F").copy())

    def ubuf_view(self, jb, nt):
        return self.ubuf[:jb * nt]

    def schur(self, lr_j, jb, skip, lstart, nt, slot=0, c0=0, c1=None, reserve_sms=0):
        c1 = nt if c1 is None else c1
        mr = self.mloc - lr_j - skip
        if mr <= 0 or nt <= 0 or c1 <= c0:
            return
        l21 = self._pan(lr_j, jb, slot)[skip:, :]
        u12 = self.ubuf[:jb * nt].numpy().reshape((nt, jb)).T[:, c0:c1]
        cols = slice(lstart + c0, lstart + c1)
        rows = slice(lr_j + skip, self.mloc)
        self.slab[rows, cols] = orc.gemm(-1.0, l21, u12, 1.0, self.slab[rows, cols], k=self.k)
        self.seen = max(self.seen, float(np.abs(self.slab[rows, cols]).max()))

    def finish(self):
        return self.ipiv.copy(), self.info, self.seen, self.top

    def trsv(self, lr, lc, jb, upper, x, j):
        blk = self.slab[lr:lr + jb, lc:lc + jb]
        if upper and np.any(np.diag(blk) == 0.0):
            self.flag = 1
            return
        xs = x[j:j + jb].numpy()
        xs[:] = solve_triangular(blk, xs, lower=not upper, unit_diagonal=not upper,
                                 check_finite=False)

    def gemv_rows(self, lr0, lr1, lc, jb, x, j, out):
        if lr1 > lr0:
            out.numpy()[self.grows[lr0:lr1]] = self.slab[lr0:lr1, lc:lc + jb] @ x.numpy()[j:j + jb]

    def zero_diag(self):
        return self.flag
