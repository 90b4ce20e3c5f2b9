"""Distributed HPL on a P x Q block-cyclic process grid (P > 1), one process
per GPU: the blocked LU of solve.py:94-140, the solve of solve.py:143-156
and the residual of solve.py:181-214.

Layout: nb x nb blocks dealt cyclically in both dimensions.  Rank r is
process (p, q) = (r // Q, r % Q); block (I, J) lives on (I % P, J % Q).  Each
rank stores its local rows x local columns column-major (leading dimension =
local rows); local row lr of process row p is global row
((lr // nb) * P + p) * nb + lr % nb (the same map as the columns, hpl.py).

One step for panel block b (owner process column b % Q, row block b % P):

* panel: the P ranks of the owner process column factor it together, one
  column at a time (oz_dpanel_candidate -> all-gather of P small records
  along the process column -> oz_dpanel_apply): the same arithmetic as the
  reference's unblocked loop, so the pivots are np.argmax's;
* the factored local panel rows and the jb pivots are broadcast along each
  process row;
* the interchanges of all other columns: every rank packs the source rows it
  owns (oz_gather_rows), each process-column rank broadcasts its pack along
  the process column, and every rank writes the destination rows it owns
  (oz_scatter_rows) — "NCCL for the panel/pivot broadcast and row swaps";
* U12: the process row b % P solves its block row (oz_trsm_lunit) and
  broadcasts it along the process column;
* every rank updates its local trailing block through the configured backend
  (oz_schur_split + oz_schur_cols): per element the same Ozaki-INT8 (or
  DGEMM) product as the single-GPU LU, since row exponents come from whole L21
  rows and column exponents from whole U12 columns.

P = 1 grids use hpl.py's 1 x Q driver (panel local to one GPU, look-ahead);
a P > 1 grid pays one all-gather per panel column, which is why 1 x Q is the
default on one NVSwitch node.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .errors import InvalidParamsError, SingularPivotError
from .gemm import BackendKind, GemmBackend, pair_table
from .hpl import Comm, _sm_count, check_scaling, local_cols_before, local_ncols

__all__ = ["Grid", "DeviceOps2D", "compose_interchanges", "factor_2d", "solve_2d", "rhs_2d",
           "residual_2d", "global_rows", "panel_mode", "REC_HDR"]

REC_HDR = 3                                       # dpanel.cu record header


def global_rows(n: int, nb: int, P: int, p: int) -> np.ndarray:
    """Global indices of process row p's local rows, in local order."""
    lr = np.arange(local_ncols(n, nb, P, p), dtype=np.int64)
    return ((lr // nb) * P + p) * nb + lr % nb


def _owner_local(g: np.ndarray, nb: int, P: int):
    """(process row, local row) of global rows g."""
    blk = g // nb
    return blk % P, (blk // P) * nb + g % nb


def compose_interchanges(piv: np.ndarray, j: int):
    """Sequential swaps (j+t <-> piv[t]) -> (dst, src) global rows such that
    afterwards row dst holds the original row src (LAPACK dlaswp order)."""
    pos = {}
    for t, pv in enumerate(piv.tolist()):
        a, b = j + t, int(pv)
        if a != b:
            pos[a], pos[b] = pos.get(b, b), pos.get(a, a)
    moves = sorted((d, s) for d, s in pos.items() if d != s)
    dst = np.array([d for d, _ in moves], dtype=np.int64)
    src = np.array([s for _, s in moves], dtype=np.int64)
    return dst, src


class Grid:
    """The P x Q process grid over torch.distributed: the world, this rank's
    process row (Q ranks, indexed by q) and process column (P ranks, by p)."""

    def __init__(self, P: int, Q: int, world: Comm | None = None):
        import torch.distributed as dist
        self.world = world or Comm()
        if P * Q != self.world.size:
            raise InvalidParamsError(f"grid {P}x{Q} does not match world size {self.world.size}")
        self.P, self.Q = P, Q
        self.p, self.q = divmod(self.world.rank, Q)
        if self.world.size == 1:
            self.row, self.col = self.world, self.world
            return
        backend = dist.get_backend()
        rows = [dist.new_group([pp * Q + qq for qq in range(Q)], backend=backend)
                for pp in range(P)]
        cols = [dist.new_group([pp * Q + qq for pp in range(P)], backend=backend)
                for qq in range(Q)]
        self.row, self.col = Comm(rows[self.p]), Comm(cols[self.q])

    def rank_of(self, p: int, q: int) -> int:
        return p * self.Q + q


class DeviceOps2D:
    """Rank-local block operations of the P x Q driver on the GPU, all through
    the C ABI (include/ozb200.h).  The local matrix is mloc x ncl, column-major,
    leading dimension mloc."""

    def __init__(self, n: int, nb: int, P: int, Q: int, p: int, q: int, backend: GemmBackend):
        t = _lib.require_cuda()
        self.t = t
        self.n, self.nb, self.P, self.Q, self.p, self.q = n, nb, P, Q, p, q
        self.mloc = local_ncols(n, nb, P, p)
        self.ncl = local_ncols(n, nb, Q, q)
        check_scaling(backend, P * Q)
        self.backend = backend
        from .solve import _backend_code
        self.code = _backend_code(backend)
        if backend.kind is BackendKind.EMULATED_INT8:
            self.k, self.qbits = backend.splits, backend.slice_bits
            self.pa, self.pb, self.ps = pair_table(backend)
        else:
            self.k, self.qbits = 0, 7
            self.pa = self.pb = self.ps = np.zeros(1, dtype=np.int32)
        dev = "cuda"
        self.slab = t.empty((max(self.ncl, 1), max(self.mloc, 1)), dtype=t.float64, device=dev)
        self.ld = max(self.mloc, 1)
        # two slots: the look-ahead panel (side stream) fills one while the
        # current step's trsm / Schur update read the other
        self.pbufs = [t.empty((max(self.mloc, 1) * nb,), dtype=t.float64, device=dev)
                      for _ in range(2)]
        self.ubuf = t.empty((nb * max(self.ncl, 1),), dtype=t.float64, device=dev)
        self.rec = t.empty((REC_HDR + 2 * nb,), dtype=t.float64, device=dev)
        self.ipiv_bufs = [t.empty((nb,), dtype=t.int32, device=dev) for _ in range(2)]
        self.side = t.cuda.Stream()   # look-ahead panel beside the update
        self.ipiv = t.empty((n,), dtype=t.int32, device=dev)
        self.info = t.zeros((1,), dtype=t.int32, device=dev)
        self.bits = t.zeros((2,), dtype=t.int64, device=dev)   # [seen, max|A|] IEEE bits
        self.sms = int(_sm_count())
        self.wsb = int(_lib.query("oz_lu_workspace_bytes", n, nb, self.k, self.qbits))
        self.planes = 2 * self.k if self.qbits > 7 else self.k
        self.ws = t.empty((self.wsb,), dtype=t.uint8, device=dev)
        self.tsb = int(_lib.query("oz_lu_solve_workspace_bytes", nb))
        self.tws = t.zeros((self.tsb // 4 + 1,), dtype=t.int32, device=dev)
        self.flag = t.zeros((1,), dtype=t.int32, device=dev)

    def _a(self, lc: int, lr: int) -> int:
        return self.slab.data_ptr() + 8 * (lc * self.ld + lr)

    def _st(self):
        return _dev.stream()

    # -- look-ahead (the 1 x Q driver's: hpl.DeviceOps)
    def lookahead_sms(self, m: int, ncols: int) -> int:
        return int(_lib.query("oz_lookahead_sms", m, ncols, self.nb,
                              len(self.pa) if self.code != 0 else 0))

    def lookahead_cols1(self, m: int, rest_cols: int, sms: int) -> int:
        return int(_lib.query("oz_lookahead_cols1", m, rest_cols, self.nb,
                              len(self.pa) if self.code != 0 else 0, sms))

    def side_stream(self):
        self.side.wait_stream(self.t.cuda.current_stream())
        return self.t.cuda.stream(self.side)

    def join_side(self) -> None:
        self.t.cuda.current_stream().wait_stream(self.side)

    # -- matrix
    def generate(self, kind: int, seed, depth=1, block=1, alpha=1.0) -> None:
        from .matgen import pcg64_state
        state, inc = pcg64_state(seed) if seed is not None else (0, 0)
        m64 = (1 << 64) - 1
        _lib.call("oz_generate_block_cyclic", kind, self.n, depth, block, float(alpha),
                  state >> 64, state & m64, inc >> 64, inc & m64, self.nb, self.P, self.p,
                  self.mloc, self.Q, self.q, self.ncl, self.slab.data_ptr(), self.ld, self._st())

    def local_view(self):
        return self.slab[:self.ncl, :self.mloc].t()

    def vector(self, host=None, n=None):
        t = self.t
        if host is None:
            return t.zeros((n,), dtype=t.float64, device="cuda")
        return t.from_numpy(np.ascontiguousarray(host, dtype=np.float64)).to("cuda")

    def row_partials(self, x_local=None):
        """(A_loc @ x_loc, sum |A_loc|) per local row, scattered into global
        n-vectors (zeros elsewhere)."""
        t = self.t
        ax = t.zeros((self.n,), dtype=t.float64, device="cuda")
        asum = t.zeros((self.n,), dtype=t.float64, device="cuda")
        if self.mloc and self.ncl:
            la = t.empty((self.mloc,), dtype=t.float64, device="cuda")
            ls = t.empty((self.mloc,), dtype=t.float64, device="cuda")
            _lib.call("oz_gemv_partial", self.slab.data_ptr(), self.mloc, self.ncl, 1, self.ld,
                      None if x_local is None else x_local.data_ptr(), la.data_ptr(),
                      ls.data_ptr(), self._st())
            for src, dst in ((la, ax), (ls, asum)):
                _lib.call("oz_scatter_vec", src.data_ptr(), 0, self.mloc, self.nb, self.P, self.p,
                          dst.data_ptr(), self._st())
        return ax, asum

    # -- factorization
    def begin(self) -> None:
        _lib.call("oz_lu_ws_init", self.ws.data_ptr(), self.wsb, self.n, self.nb, self.planes,
                  self._st())
        self.info.zero_()
        self.bits.zero_()
        if self.ncl and self.mloc:
            _lib.call("oz_max_abs_bits", self.slab.data_ptr(), self.mloc, self.ncl, 1, self.ld, 0,
                      self.bits.data_ptr() + 8, self._st())

    def dpanel_candidate(self, lc: int, lr0: int, t: int, jb: int, owns_g: bool):
        rec = self.rec[:REC_HDR + 2 * jb]
        _lib.call("oz_dpanel_candidate", self._a(lc, 0), self.ld, lr0, self.mloc, t, jb,
                  int(owns_g), self.nb, self.P, self.p, rec.data_ptr(), self._st())
        return rec

    def dpanel_apply(self, lc: int, lr0: int, t: int, jb: int, g: int, owns_g: bool, recs):
        _lib.call("oz_dpanel_apply", self._a(lc, 0), self.ld, lr0, self.mloc, t, jb, g,
                  int(owns_g), self.nb, self.P, self.p, recs.data_ptr(),
                  self.ipiv_bufs[0].data_ptr(),
                  self.info.data_ptr(), self.bits.data_ptr(), self._st())

    # -- gathered panel (default): one all-gather per panel, then the
    #    single-GPU recursive panel factorization on every rank of the column
    def panel_pack(self, lc: int, lr_j: int, jb: int, R: int):
        """This rank's panel rows lr_j.. (jb columns) as an R x jb column-major
        block (rows past the local count are zero padding)."""
        t = self.t
        buf = t.zeros((max(R, 1) * jb,), dtype=t.float64, device="cuda")
        mine = self.mloc - lr_j
        if mine > 0:
            _lib.call("oz_copy2d", self._a(lc, lr_j), mine, jb, 1, self.ld, buf.data_ptr(), 1, R,
                      self._st())
        return buf

    def panel_from_gathered(self, allp, lc: int, lr_j: int, j: int, jb: int, R: int,
                            slot: int = 0, max_ctas: int = 0) -> None:
        """Assemble the global m x jb panel (rows j..n) from the P gathered
        blocks, factor it with the single-GPU panel kernels (oz_lu_panel:
        recursive leaves, partial pivoting, interchanges inside the panel),
        and write this rank's rows of the result back into its slab."""
        t = self.t
        n, nb, P = self.n, self.nb, self.P
        m = n - j
        g = np.arange(j, n, dtype=np.int64)
        owner = (g // nb) % P
        lrj = np.array([local_cols_before(j, nb, P, o) for o in range(P)], dtype=np.int64)
        row = ((g // nb) // P) * nb + g % nb - lrj[owner]
        blk_d = self._rows_dev(owner)
        row_d = self._rows_dev(row)
        apan = t.empty((m * jb,), dtype=t.float64, device="cuda")
        _lib.call("oz_assemble_rows", allp.data_ptr(), R, R * jb, blk_d.data_ptr(),
                  row_d.data_ptr(), m, jb, apan.data_ptr(), m, self._st())
        _lib.call("oz_lu_panel", apan.data_ptr(), m, m, jb, j, self.ipiv_bufs[slot].data_ptr(),
                  self.info.data_ptr(), self.bits.data_ptr(), self.ws.data_ptr(), self.wsb,
                  self.n, self.nb, self.planes, max_ctas, self._st())
        mine = self.mloc - lr_j
        if mine > 0:
            back = self._rows_dev(global_rows(n, nb, P, self.p)[lr_j:] - j)
            _lib.call("oz_assemble_rows", apan.data_ptr(), m, 0, None, back.data_ptr(), mine,
                      jb, self._a(lc, lr_j), self.ld, self._st())

    def panel_finish(self, lc: int, lr_j: int, jb: int, diag: bool, slot: int = 0) -> None:
        """Growth over the finalized U rows of the diagonal block; pack the
        local panel rows lr_j.. into the broadcast buffer (F-order)."""
        if diag:
            _lib.call("oz_max_abs_bits", self._a(lc, lr_j), jb, jb, 1, self.ld, 1,
                      self.bits.data_ptr(), self._st())
        m = self.mloc - lr_j
        if m > 0:
            _lib.call("oz_copy2d", self._a(lc, lr_j), m, jb, 1, self.ld,
                      self.pbufs[slot].data_ptr(), 1, m, self._st())

    def panel_buffers(self, lr_j: int, jb: int, slot: int = 0):
        return self.pbufs[slot][:(self.mloc - lr_j) * jb], self.ipiv_bufs[slot][:jb]

    def record_pivots(self, j: int, jb: int, slot: int = 0) -> np.ndarray:
        self.ipiv[j:j + jb].copy_(self.ipiv_bufs[slot][:jb])
        return self.ipiv_bufs[slot][:jb].cpu().numpy()

    def _cols(self, ranges):
        (c0a, c1a), (c0b, c1b) = ranges
        return (c1a - c0a) + (c1b - c0b)

    def _rows_dev(self, rows):
        return self.t.from_numpy(np.ascontiguousarray(rows, dtype=np.int32)).to("cuda")

    def gather_rows(self, lrows: np.ndarray, ranges):
        nr, nc = len(lrows), self._cols(ranges)
        buf = self.t.empty((max(nr * nc, 1),), dtype=self.t.float64, device="cuda")
        (c0a, c1a), (c0b, c1b) = ranges
        rows = self._rows_dev(lrows)          # kept alive until the launch is queued
        _lib.call("oz_gather_rows", self.slab.data_ptr(), self.ld, rows.data_ptr(), nr, c0a, c1a,
                  c0b, c1b, buf.data_ptr(), None, max(nr, 1), self._st())
        return buf[:nr * nc]

    def rows_buffer(self, nrows: int, ranges):
        return self.t.empty((nrows * self._cols(ranges),), dtype=self.t.float64, device="cuda")

    def scatter_rows(self, lrows: np.ndarray, ranges, buf, brows: np.ndarray, ldb: int) -> None:
        if len(lrows) == 0:
            return
        (c0a, c1a), (c0b, c1b) = ranges
        rows, brow = self._rows_dev(lrows), self._rows_dev(brows)   # both alive at the launch
        _lib.call("oz_scatter_rows", self.slab.data_ptr(), self.ld, rows.data_ptr(), len(lrows),
                  c0a, c1a, c0b, c1b, buf.data_ptr(), brow.data_ptr(), ldb, self._st())

    def trsm(self, lr_j: int, jb: int, lstart: int, nt: int, slot: int = 0):
        """U12 <- L11^-1 A12 in place (block row of this process row), copied
        into the U12 broadcast buffer."""
        m = self.mloc - lr_j
        u12 = self._a(lstart, lr_j)
        _lib.call("oz_trsm_lunit", self.pbufs[slot].data_ptr(), m, jb, u12, self.ld, nt,
                  self._st())
        _lib.call("oz_max_abs_bits", u12, jb, nt, 1, self.ld, 0, self.bits.data_ptr(),
                  self._st())
        _lib.call("oz_copy2d", u12, jb, nt, 1, self.ld, self.ubuf.data_ptr(), 1, jb, self._st())

    def ubuf_view(self, jb: int, nt: int):
        return self.ubuf[:jb * nt]

    def schur(self, lr_j: int, jb: int, skip: int, lstart: int, nt: int, slot: int = 0,
              c0: int = 0, c1: int | None = None, reserve_sms: int = 0) -> None:
        """A22 (local rows lr_j+skip.., columns lstart+c0 .. lstart+c1) -= L21 U12.
        The split of L21 and of all of U12 happens with the first column range
        (c0 == 0); later ranges reuse it (per-vector exponents: the product of
        an element does not depend on the column partition)."""
        c1 = nt if c1 is None else c1
        mrem = self.mloc - lr_j
        mr = mrem - skip
        if mr <= 0 or nt <= 0 or c1 <= c0:
            return
        l21 = self.pbufs[slot].data_ptr() + 8 * skip
        u12 = self.ubuf.data_ptr()
        a22 = self._a(lstart, lr_j + skip)
        if c0 == 0:
            _lib.call("oz_schur_split", self.code, mr, nt, jb, l21, mrem, u12, jb, self.k,
                      self.qbits, self.ws.data_ptr(), self.wsb, self.n, self.nb, self._st())
        max_ctas = self.sms - reserve_sms if reserve_sms > 0 else 0
        _lib.call("oz_schur_cols", self.code, mr, nt, jb, l21, mrem, u12, jb, a22, self.ld,
                  self.k, self.qbits, len(self.pa), self.pa.ctypes.data, self.pb.ctypes.data,
                  self.ps.ctypes.data, self.bits.data_ptr(), c0, c1, max_ctas,
                  self.ws.data_ptr(), self.wsb, self.n, self.nb, self._st())

    def finish(self):
        b = self.bits.cpu().numpy().view(np.float64)
        return self.ipiv.cpu().numpy(), int(self.info.item()), float(b[0]), float(b[1])

    # -- solve
    def trsv(self, lr: int, lc: int, jb: int, upper: bool, x, j: int) -> None:
        _lib.call("oz_trsv_block", self._a(lc, lr), self.ld, jb, 1 if upper else 0,
                  x.data_ptr() + 8 * j, self.flag.data_ptr(), self.tws.data_ptr(), self.tsb,
                  self._st())

    def gemv_rows(self, lr0: int, lr1: int, lc: int, jb: int, x, j: int, out) -> None:
        """out[global rows of lr0..lr1] = A_loc[lr0:lr1, lc:lc+jb] @ x[j:j+jb]."""
        if lr1 <= lr0:
            return
        t = self.t
        y = t.empty((lr1 - lr0,), dtype=t.float64, device="cuda")
        _lib.call("oz_gemv_partial", self._a(lc, lr0), lr1 - lr0, jb, 1, self.ld,
                  x.data_ptr() + 8 * j, y.data_ptr(), None, self._st())
        _lib.call("oz_scatter_vec", y.data_ptr(), lr0, lr1 - lr0, self.nb, self.P, self.p,
                  out.data_ptr(), self._st())

    def zero_diag(self) -> int:
        return int(self.flag.item())


# ------------------------------------------------------------ the driver
def panel_mode() -> str:
    """OZ_PANEL_2D: 'gather' (default) or 'column' (the per-column exchange)."""
    import os
    m = os.environ.get("OZ_PANEL_2D", "gather")
    if m not in ("gather", "column"):
        raise InvalidParamsError(f"OZ_PANEL_2D must be gather or column, got {m!r}")
    return m


def factor_2d(ops, grid: Grid, n: int, nb: int, mode: str | None = None,
              lookahead: bool = True):
    """Blocked right-looking LU (solve.py:94-140) on the P x Q grid.
    Returns (ipiv int32[n] global LAPACK-style, growth).

    Panel modes (the P ranks of the owner process column):
    * 'gather' (default): ONE all-gather of the ranks' panel rows per panel,
      then every rank of the column factors the whole m x jb panel with the
      single-GPU recursive panel kernels (identical inputs -> identical
      pivots and factors on every rank) and keeps its own rows -- one host
      round trip per panel instead of jb, and the blocked panel instead of
      the level-2 column loop;
    * 'column': one all-gather of small candidate records per panel column,
      the reference's unblocked loop (solve.py:75-90) distributed.

    Look-ahead (gather mode, depth 1, as hpl.py's 1 x Q driver): the process
    column owning panel b+1 updates that panel's columns first, then gathers
    and factors it on a side stream capped to S SMs (the single-GPU panel_sms
    of the panel's height, so its factors do not depend on the grid), while
    the compute stream updates the rest of its columns: the first cols1 on
    sms - S SMs, the remainder on every SM once the panel is done.  Panel
    buffers alternate between two slots so the look-ahead panel never
    overwrites the L21 the current step is still reading."""
    P, Q, p, q = grid.P, grid.Q, grid.p, grid.q
    ncl = ops.ncl
    nblk = -(-n // nb)
    mode = mode or panel_mode()
    lookahead = lookahead and mode == "gather"
    ops.begin()
    early = set()                                 # panels factored on the side stream
    side_pending = False

    def factor_gathered(jblk, slot, max_ctas):
        j = jblk * nb
        jb = min(nb, n - j)
        lc = (jblk // Q) * nb
        lr_j = local_cols_before(j, nb, P, p)
        R = max(local_ncols(n, nb, P, o) - local_cols_before(j, nb, P, o) for o in range(P))
        allp = grid.col.allgather(ops.panel_pack(lc, lr_j, jb, R))
        ops.panel_from_gathered(allp, lc, lr_j, j, jb, R, slot, max_ctas)
        ops.panel_finish(lc, lr_j, jb, p == jblk % P, slot)

    for jblk in range(nblk):
        j = jblk * nb
        jb = min(nb, n - j)
        pr, pc = jblk % P, jblk % Q
        lc = (jblk // Q) * nb
        lr_j = local_cols_before(j, nb, P, p)
        slot = jblk % 2 if mode == "gather" else 0
        if q == pc and mode == "gather":
            if jblk in early:                         # factored during the previous step
                if side_pending:
                    ops.join_side()
                    side_pending = False
            else:
                factor_gathered(jblk, slot, 0)
        elif q == pc:                                 # panel, one column at a time
            for t in range(jb):
                g = j + t
                owns_g = (g // nb) % P == p
                lr0 = local_cols_before(g, nb, P, p)
                rec = ops.dpanel_candidate(lc, lr0, t, jb, owns_g)
                recs = grid.col.allgather(rec)
                ops.dpanel_apply(lc, lr0, t, jb, g, owns_g, recs)
            ops.panel_finish(lc, lr_j, jb, p == pr)
        pbuf, ipiv = ops.panel_buffers(lr_j, jb, slot)
        grid.row.bcast(pbuf, pc)                      # L of the panel, local rows
        grid.row.bcast(ipiv, pc)
        piv = ops.record_pivots(j, jb, slot)
        # interchanges on every column outside the panel
        ranges = ((0, lc), (lc + jb, ncl)) if q == pc else ((0, ncl), (ncl, ncl))
        dst, src = compose_interchanges(piv, j)
        if len(dst):
            so, sl = _owner_local(src, nb, P)
            do, dl = _owner_local(dst, nb, P)
            packs = []
            for o in range(P):                        # pack every source before any write
                sel = np.nonzero(so == o)[0]
                if len(sel) == 0:
                    packs.append(None)
                    continue
                buf = ops.gather_rows(sl[sel], ranges) if o == p else ops.rows_buffer(len(sel),
                                                                                     ranges)
                packs.append((sel, buf))
            for o in range(P):
                if packs[o] is not None:
                    grid.col.bcast(packs[o][1], o)
            for o in range(P):
                if packs[o] is None:
                    continue
                sel, buf = packs[o]
                mine = np.nonzero(do[sel] == p)[0]
                ops.scatter_rows(dl[sel][mine], ranges, buf, mine, len(sel))
        # U12 and the trailing update
        lstart = local_cols_before(j + jb, nb, Q, q)
        nt = ncl - lstart
        if j + jb < n and nt > 0:
            if p == pr:
                ops.trsm(lr_j, jb, lstart, nt, slot)
            grid.col.bcast(ops.ubuf_view(jb, nt), pr)
            skip = jb if p == pr else 0
            nxt = jblk + 1
            m_next = n - nxt * nb
            jb2 = min(nb, m_next) if nxt < nblk else 0
            S = 0
            if lookahead and nxt < nblk and nxt % Q == q and m_next > jb2:
                S = ops.lookahead_sms(m_next, nt)
            if S > 0:
                ops.schur(lr_j, jb, skip, lstart, nt, slot, 0, jb2)   # the next panel's columns
                with ops.side_stream():
                    factor_gathered(nxt, nxt % 2, S)
                early.add(nxt)
                side_pending = True
                c1 = jb2 + ops.lookahead_cols1(m_next, nt - jb2, S)
                ops.schur(lr_j, jb, skip, lstart, nt, slot, jb2, c1, S)
                if c1 < nt:
                    ops.join_side()
                    side_pending = False
                    ops.schur(lr_j, jb, skip, lstart, nt, slot, c1, nt)
            else:
                ops.schur(lr_j, jb, skip, lstart, nt, slot)
    if side_pending:
        ops.join_side()
    ipiv, info, seen, top = ops.finish()
    info, seen, top = grid.world.allreduce_values([info, seen, top], "max")
    info = int(info)
    if info:
        raise SingularPivotError(f"exact zero pivot column at index {info - 1}")
    return ipiv, (seen / top if top > 0 else 1.0)


def solve_2d(ops, grid: Grid, n: int, nb: int, perm: np.ndarray, b_host: np.ndarray):
    """x = U^-1 L^-1 b[perm] (solve.py:143-156), x replicated: the diagonal
    block's owner solves it and broadcasts the piece; the ranks of that
    process column form their rows' updates, summed over the grid."""
    P, Q, p, q = grid.P, grid.Q, grid.p, grid.q
    x = ops.vector(np.asarray(b_host, dtype=np.float64)[perm])
    nblk = -(-n // nb)
    for upper in (False, True):
        order = reversed(range(nblk)) if upper else range(nblk)
        for jblk in order:
            j = jblk * nb
            jb = min(nb, n - j)
            pr, pc = jblk % P, jblk % Q
            lc = (jblk // Q) * nb
            lr_j = local_cols_before(j, nb, P, p)
            if (p, q) == (pr, pc):
                ops.trsv(lr_j, lc, jb, upper, x, j)
            grid.world.bcast(x[j:j + jb], grid.rank_of(pr, pc))
            r0, r1 = (0, j) if upper else (j + jb, n)
            if r1 <= r0:
                continue
            d = ops.vector(n=n)
            if q == pc:
                lr0 = local_cols_before(r0, nb, P, p)
                lr1 = local_cols_before(r1, nb, P, p)
                ops.gemv_rows(lr0, lr1, lc, jb, x, j, d)
            grid.world.allreduce(d, "sum")
            x[r0:r1] -= d[r0:r1]
    if grid.world.allreduce_values([ops.zero_diag()], "max")[0]:
        raise SingularPivotError("zero diagonal entry in U")
    return x


def rhs_2d(ops, grid: Grid):
    """b = A @ ones (harness.py:126), replicated."""
    ax, _ = ops.row_partials(None)
    grid.world.allreduce(ax, "sum")
    return ax


def residual_2d(ops, grid: Grid, n: int, nb: int, x, b):
    """The scaled residual (solve.py:181-214) with A regenerated in place."""
    from .solve import _report
    xh = x.cpu().numpy()
    gcols = global_rows(n, nb, grid.Q, grid.q)        # same map for the columns
    xl = ops.vector(xh[gcols]) if len(gcols) else None
    ax, asum = ops.row_partials(xl)
    grid.world.allreduce(ax, "sum")
    grid.world.allreduce(asum, "sum")
    r = (ax - b).abs().max().item()
    return _report(float(r), float(asum.max().item()), float(np.abs(xh).max()),
                   float(b.abs().max().item()), n)
