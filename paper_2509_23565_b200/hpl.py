"""Distributed HPL: the blocked LU of solve.py:94-140 and the solve of
solve.py:143-156 over a 1 x Q block-cyclic process grid, one process per GPU.

Layout: column blocks of width nb are dealt round-robin to the
Q ranks (global block b lives on rank b % Q as local block b // Q); every
rank holds all n rows of its columns, column-major, leading dimension n.
With one process row every pivot search is local to the panel owner, so the
only data-path collectives are

* the panel broadcast: the owner factors columns j..j+jb (oz_lu_panel:
  partial pivoting, division, outer-product update — solve.py:66-91) and
  broadcasts the factored panel rows j..n plus its jb pivot rows;
* the triangular-solve broadcasts of the updated right-hand side.

Every rank then applies the panel's interchanges to its own columns
(oz_laswp, whole-row swaps as solve.py:80-82), solves its U12 block
(oz_trsm_lunit, solve.py:123-127) and updates its trailing columns through
the configured backend (oz_schur_update: cuBLAS DGEMM or the Ozaki-INT8
tcgen05 GEMM, solve.py:130-134).  The emulated Schur update is per-element
identical to the single-GPU one (row exponents come from the whole L21,
column exponents from each U12 column), so the distributed factors match the
single-process factors.

The driver only sequences calls: local block operations go through an
``ops`` object (``DeviceOps`` = the C ABI on the local GPU) and collectives
through a ``Comm`` (torch.distributed: NCCL on B200s; gloo stages CUDA
tensors through host memory, which the CPU/1-GPU tests use).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import InvalidParamsError, SingularPivotError
from .gemm import BackendKind, GemmBackend, pair_table

__all__ = ["Comm", "DeviceOps", "HplReport", "HplProblem", "local_cols_before", "local_ncols",
           "global_cols", "factor_block_cyclic", "solve_block_cyclic", "hpl_run"]


# ------------------------------------------------------------ index maps
def local_cols_before(g: int, nb: int, Q: int, q: int) -> int:
    """Number of rank q's columns whose global index is < g (1 x Q grid)."""
    b, off = divmod(g, nb)
    cnt = ((b - q + Q - 1) // Q) * nb if b > q else 0
    if b % Q == q:
        cnt += off
    return cnt


def local_ncols(n: int, nb: int, Q: int, q: int) -> int:
    return local_cols_before(n, nb, Q, q)


def global_cols(n: int, nb: int, Q: int, q: int) -> np.ndarray:
    """Global indices of rank q's local columns, in local order."""
    lc = np.arange(local_ncols(n, nb, Q, q), dtype=np.int64)
    return ((lc // nb) * Q + q) * nb + lc % nb


# ------------------------------------------------------------ collectives
class Comm:
    """torch.distributed over a group.  Under gloo, CUDA tensors are staged
    through host memory (gloo moves host buffers); NCCL moves them in place
    over NVLink."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.size = dist.get_world_size(group)
            self.stage = dist.get_backend(group) == "gloo"
        else:
            self.rank, self.size, self.stage = 0, 1, False

    def _grank(self, r):
        if self.group is None:
            return r
        return self.dist.get_global_rank(self.group, r)

    def bcast(self, t, src: int) -> None:
        if self.size == 1 or t.numel() == 0:
            return
        if self.stage and t.is_cuda:
            import torch
            # gloo stages through the host; only the root's contents matter
            h = t.cpu() if self.rank == src else torch.empty(tuple(t.shape), dtype=t.dtype)
            self.dist.broadcast(h, self._grank(src), group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, self._grank(src), group=self.group)

    def bcast_async(self, t, src: int):
        """Start a broadcast without making the compute stream wait (NCCL);
        returns a handle with .wait(), or None when it already completed."""
        if self.size == 1 or t.numel() == 0:
            return None
        if self.stage and t.is_cuda:
            self.bcast(t, src)
            return None
        return self.dist.broadcast(t, self._grank(src), group=self.group, async_op=True)

    def allgather(self, t):
        """-> (size, *t.shape) tensor of every rank's t, on t's device."""
        import torch
        if self.size == 1:
            return t.reshape((1,) + tuple(t.shape))
        if self.stage and t.is_cuda:
            parts = [torch.empty_like(t, device="cpu") for _ in range(self.size)]
            self.dist.all_gather(parts, t.cpu(), group=self.group)
            return torch.stack(parts).to(t.device)
        if not t.is_cuda:
            parts = [torch.empty_like(t) for _ in range(self.size)]
            self.dist.all_gather(parts, t, group=self.group)
            return torch.stack(parts)
        out = torch.empty((self.size,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def allreduce(self, t, op: str) -> None:
        if self.size == 1:
            return
        rop = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX}[op]
        if self.stage and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, rop, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, rop, group=self.group)

    def allreduce_values(self, vals, op: str) -> list:
        """All-reduce a few host scalars (NCCL needs them on the device)."""
        import torch
        dev = "cpu" if (self.stage or self.size == 1) else "cuda"
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
        self.allreduce(t, op)
        return [float(v) for v in t.cpu().tolist()]

    def barrier(self) -> None:
        if self.size > 1:
            self.dist.barrier(group=self.group)


def _sm_count() -> int:
    out = np.zeros(1, dtype=np.int32)
    _lib.call("oz_sm_count", out.ctypes.data)
    return int(out[0])


def check_scaling(backend: GemmBackend, ranks: int) -> None:
    """GLOBAL scaling takes ONE exponent over a whole operand (split.py:131-134);
    a rank only sees its own A21 rows / U12 columns, so a distributed split
    would pick per-rank exponents and diverge from the reference.  Refuse it
    rather than return different factors."""
    from .split import ScalingMode
    if ranks > 1 and backend.kind is BackendKind.EMULATED_INT8 and \
            backend.scaling is ScalingMode.GLOBAL:
        raise InvalidParamsError("GLOBAL scaling is single-GPU only: the distributed drivers "
                                 "split per rank (use PER_VECTOR or one rank)")


# ------------------------------------------------------------ device ops
class DeviceOps:
    """Rank-local block operations on the GPU, all through the C ABI
    (include/ozb200.h step-level entries).  Owns the local slab (n x ncl,
    column-major), the broadcast buffers and the LU workspace."""

    def __init__(self, n: int, nb: int, Q: int, q: int, backend: GemmBackend):
        t = _lib.require_cuda()
        self.t = t
        self.n, self.nb, self.Q, self.q = n, nb, Q, q
        self.ncl = local_ncols(n, nb, Q, q)
        check_scaling(backend, Q)
        self.backend = backend
        self.emulated = backend.kind is BackendKind.EMULATED_INT8
        from .solve import _backend_code
        self.code = _backend_code(backend)
        if self.emulated:
            self.k, self.qbits = backend.splits, backend.slice_bits
            self.pa, self.pb, self.ps = pair_table(backend)
        else:
            self.k, self.qbits = 0, 7
            self.pa = self.pb = self.ps = np.zeros(1, dtype=np.int32)
        dev = "cuda"
        # local slab: torch (ncl, n) row-major == column-major n x ncl, ld = n
        self.slab = t.empty((max(self.ncl, 1), n), dtype=t.float64, device=dev)
        # two panel slots: panel j+1 is factored (look-ahead) while panel j's
        # L21 still feeds the trailing update
        self.pbuf = [t.empty((n * nb,), dtype=t.float64, device=dev) for _ in range(2)]
        self.ipiv_buf = [t.empty((nb,), dtype=t.int32, device=dev) for _ in range(2)]
        self.sms = int(_sm_count())
        self.ipiv = t.empty((n,), dtype=t.int32, device=dev)
        self.info = t.zeros((1,), dtype=t.int32, device=dev)
        self.bits = t.zeros((2,), dtype=t.int64, device=dev)   # [seen, max|A|] as IEEE bits
        self.wsb = int(_lib.query("oz_lu_workspace_bytes", n, nb, self.k, self.qbits))
        self.planes = 2 * self.k if self.qbits > 7 else self.k   # workspace int8 planes
        self.ws = t.empty((self.wsb,), dtype=t.uint8, device=dev)
        self.tsb = int(_lib.query("oz_lu_solve_workspace_bytes", nb))
        self.tws = t.zeros((self.tsb // 4 + 1,), dtype=t.int32, device=dev)
        self.flag = t.zeros((1,), dtype=t.int32, device=dev)
        self.side = t.cuda.Stream()   # look-ahead panel (+ its broadcast) beside the update

    def lookahead_sms(self, m: int, ncols: int) -> int:
        """Look-ahead SMs for the panel of an m-row trailing matrix (the
        single-GPU driver's value for the same panel: equal SM caps keep the
        panel's factors bit-identical)."""
        return int(_lib.query("oz_lookahead_sms", m, ncols, self.nb,
                              len(self.pa) if self.emulated else 0))

    def lookahead_cols1(self, m: int, rest_cols: int, sms: int) -> int:
        """Two-phase look-ahead: how many of this rank's rest_cols columns to
        update beside the panel on the other SMs (the rest after it, on all)."""
        return int(_lib.query("oz_lookahead_cols1", m, rest_cols, self.nb,
                              len(self.pa) if self.emulated else 0, sms))

    # -- streams
    def side_stream(self):
        """Context: run the enclosed calls on the side stream, after the work
        already queued on the compute stream."""
        self.side.wait_stream(self.t.cuda.current_stream())
        return self.t.cuda.stream(self.side)

    def join_side(self) -> None:
        self.t.cuda.current_stream().wait_stream(self.side)

    # -- addressing
    def _a(self, lc: int, row: int) -> int:
        return self.slab.data_ptr() + 8 * (lc * self.n + row)

    def _st(self):
        return _dev.stream()

    # -- matrix
    def generate(self, kind: int, seed, depth=1, block=1, alpha=1.0) -> None:
        from .matgen import pcg64_state
        state, inc = pcg64_state(seed) if seed is not None else (0, 0)
        m64 = (1 << 64) - 1
        _lib.call("oz_generate_cyclic", kind, self.n, depth, block, float(alpha), state >> 64,
                  state & m64, inc >> 64, inc & m64, self.nb, self.Q, self.q, self.ncl,
                  self.slab.data_ptr(), self.n, self._st())

    def row_partials(self, x_local=None):
        """(A_local @ x_local, sum |A_local| per row) over this rank's columns."""
        t = self.t
        ax = t.empty((self.n,), dtype=t.float64, device="cuda")
        asum = t.empty((self.n,), dtype=t.float64, device="cuda")
        _lib.call("oz_gemv_partial", self.slab.data_ptr(), self.n, self.ncl, 1, self.n,
                  None if x_local is None else x_local.data_ptr(), ax.data_ptr(),
                  asum.data_ptr(), self._st())
        return ax, asum

    def local_view(self):
        """The local slab as an (n, ncl) column-major tensor view."""
        return self.slab[:self.ncl].t()

    # -- factorization steps
    def begin(self) -> None:
        _lib.call("oz_lu_ws_init", self.ws.data_ptr(), self.wsb, self.n, self.nb, self.planes,
                  self._st())
        self.info.zero_()
        self.bits.zero_()
        if self.ncl:
            _lib.call("oz_max_abs_bits", self.slab.data_ptr(), self.n, self.ncl, 1, self.n, 0,
                      self.bits.data_ptr() + 8, self._st())

    def panel(self, lc: int, j: int, jb: int, slot: int = 0, max_ctas: int = 0) -> None:
        _lib.call("oz_lu_panel", self._a(lc, j), self.n, self.n - j, jb, j,
                  self.ipiv_buf[slot].data_ptr(), self.info.data_ptr(), self.bits.data_ptr(),
                  self.ws.data_ptr(), self.wsb, self.n, self.nb, self.planes, max_ctas,
                  self._st())
        # triu of the panel's diagonal block: finalized U rows (solve.py:135-137)
        _lib.call("oz_max_abs_bits", self._a(lc, j), jb, jb, 1, self.n, 1,
                  self.bits.data_ptr(), self._st())
        m = self.n - j
        _lib.call("oz_copy2d", self._a(lc, j), m, jb, 1, self.n, self.pbuf[slot].data_ptr(), 1,
                  m, self._st())

    def panel_buffers(self, j: int, jb: int, slot: int = 0):
        m = self.n - j
        return self.pbuf[slot][:m * jb], self.ipiv_buf[slot][:jb]

    def record_pivots(self, j: int, jb: int, slot: int = 0) -> None:
        self.ipiv[j:j + jb].copy_(self.ipiv_buf[slot][:jb])

    def laswp(self, ranges, j: int, jb: int, slot: int = 0) -> None:
        (c0a, c1a), (c0b, c1b) = ranges
        _lib.call("oz_laswp", self.slab.data_ptr(), self.n, c0a, c1a, c0b, c1b, j,
                  self.ipiv_buf[slot].data_ptr(), jb, self.ws.data_ptr(), self.wsb, self.n,
                  self.nb, self.planes, self._st())

    def trsm_split(self, j: int, jb: int, lstart: int, nt: int, slot: int = 0) -> None:
        """U12 <- L11^-1 A12 on local columns lstart..lstart+nt, then split
        L21 / U12 for the trailing update."""
        m = self.n - j
        pb = self.pbuf[slot].data_ptr()
        u12 = self._a(lstart, j)
        _lib.call("oz_trsm_lunit", pb, m, jb, u12, self.n, nt, self._st())
        _lib.call("oz_max_abs_bits", u12, jb, nt, 1, self.n, 0, self.bits.data_ptr(),
                  self._st())
        if m - jb > 0:
            _lib.call("oz_schur_split", self.code, m - jb, nt, jb, pb + 8 * jb, m,
                      u12, self.n, self.k, self.qbits, self.ws.data_ptr(), self.wsb, self.n,
                      self.nb, self._st())

    def schur_cols(self, j: int, jb: int, lstart: int, nt: int, c0: int, c1: int,
                   slot: int = 0, reserve_sms: int = 0) -> None:
        """A22 -= L21 U12 on trailing local columns lstart+c0 .. lstart+c1."""
        m = self.n - j
        if m - jb <= 0 or c1 <= c0:
            return
        max_ctas = self.sms - reserve_sms if reserve_sms > 0 else 0
        _lib.call("oz_schur_cols", self.code, m - jb, nt, jb,
                  self.pbuf[slot].data_ptr() + 8 * jb, m, self._a(lstart, j), self.n,
                  self._a(lstart, j + jb), self.n, self.k, self.qbits, len(self.pa),
                  self.pa.ctypes.data, self.pb.ctypes.data, self.ps.ctypes.data,
                  self.bits.data_ptr(), c0, c1, max_ctas, self.ws.data_ptr(), self.wsb, self.n,
                  self.nb, self._st())

    def finish(self):
        """-> (ipiv host int32[n], info, seen, max|A|) of this rank."""
        b = self.bits.cpu().numpy().view(np.float64)
        return self.ipiv.cpu().numpy(), int(self.info.item()), float(b[0]), float(b[1])

    # -- triangular solves
    def solve_vector(self, vec_host: np.ndarray):
        return self.t.from_numpy(np.ascontiguousarray(vec_host, dtype=np.float64)).to("cuda")

    def trsv(self, lc: int, j: int, jb: int, upper: bool, x) -> None:
        _lib.call("oz_trsv_block", self._a(lc, j), self.n, jb, 1 if upper else 0,
                  x.data_ptr() + 8 * j, self.flag.data_ptr(), self.tws.data_ptr(), self.tsb,
                  self._st())

    def gemv_update(self, lc: int, r0: int, r1: int, j: int, jb: int, x) -> None:
        """x[r0:r1] -= A[r0:r1, local cols lc..lc+jb] @ x[j:j+jb]."""
        if r1 <= r0:
            return
        _lib.call("oz_dgemm", 0, 0, r1 - r0, 1, jb, -1.0, self._a(lc, r0), self.n,
                  x.data_ptr() + 8 * j, jb, 1.0, x.data_ptr() + 8 * r0, r1 - r0, self._st())

    def zero_diag(self) -> int:
        return int(self.flag.item())


# ------------------------------------------------------------ the driver
def factor_block_cyclic(ops, comm, n: int, nb: int, lookahead: bool = True,
                        reserve_sms: int | None = None):
    """Blocked right-looking LU (solve.py:94-140) of the distributed matrix in
    ops' local slabs.  Returns (ipiv int32[n] global LAPACK-style, growth).

    Look-ahead (depth 1): the owner of panel b+1 updates that panel's columns
    first, then factors it on a side stream with S CTAs and starts its
    broadcast from there (asynchronously on NCCL), while its compute stream
    updates the rest of its columns on sms - S CTAs; the other ranks find
    panel b+1 ready when they finish step b.  S (reserve_sms, default: the
    look-ahead model for this rank's share of the update, oz_lookahead_sms)
    also caps the panel's own kernels; on one rank it is the single-GPU
    driver's split, so the factors equal the single-GPU LU's bit for bit.  The
    last panel is factored after the update, as there."""
    Q, q = comm.size, comm.rank
    ncl = local_ncols(n, nb, Q, q)
    nblk = -(-n // nb)
    ops.begin()
    sends = {}                                   # slot -> in-flight early broadcast handles
    early = set()                                # panels already factored and sent
    side_pending = False                         # side-stream panel not yet joined

    def factor_and_send(b, lc, slot, async_ok, max_ctas=0):
        jj = b * nb
        jjb = min(nb, n - jj)
        for h in sends.pop(slot, ()):            # the slot's previous send must be done
            h.wait()
        ops.panel(lc, jj, jjb, slot, max_ctas)
        if async_ok:
            pb, ip = ops.panel_buffers(jj, jjb, slot)
            sends[slot] = [h for h in (comm.bcast_async(pb, q), comm.bcast_async(ip, q)) if h]
            early.add(b)

    if q == 0:
        factor_and_send(0, 0, 0, False)
    for jblk in range(nblk):
        j = jblk * nb
        jb = min(nb, n - j)
        owner = jblk % Q
        slot = jblk % 2
        lc = (jblk // Q) * nb                   # the panel's local column on its owner
        if side_pending:                         # this panel came from the side stream
            ops.join_side()
            side_pending = False
        if jblk not in early:                    # receive (or, on the owner, send) now
            pbuf, ipiv = ops.panel_buffers(j, jb, slot)
            comm.bcast(pbuf, owner)              # L11/L21 of the factored panel
            comm.bcast(ipiv, owner)              # its jb pivot rows
        ops.record_pivots(j, jb, slot)
        if q == owner:
            ranges = ((0, lc), (lc + jb, ncl))
        else:
            ranges = ((0, ncl), (ncl, ncl))
        ops.laswp(ranges, j, jb, slot)
        lstart = local_cols_before(j + jb, nb, Q, q)
        nt = ncl - lstart
        nxt = jblk + 1
        mine_next = nxt < nblk and nxt % Q == q
        if nt > 0:
            ops.trsm_split(j, jb, lstart, nt, slot)
            if mine_next:
                jb2 = min(nb, n - nxt * nb)       # the next panel = my first trailing columns
                ops.schur_cols(j, jb, lstart, nt, 0, jb2, slot)
                m_next = n - nxt * nb
                S = 0
                if lookahead and m_next > jb2:
                    S = (ops.lookahead_sms(m_next, nt) if reserve_sms is None
                         else reserve_sms)
                if S > 0:
                    with ops.side_stream():
                        factor_and_send(nxt, lstart, nxt % 2, Q > 1, S)
                    side_pending = True
                    # two-phase: the first cols1 columns beside the panel on
                    # sms - S SMs, the rest on every SM once the panel is done
                    c1 = jb2 + ops.lookahead_cols1(m_next, nt - jb2, S)
                    ops.schur_cols(j, jb, lstart, nt, jb2, c1, slot, S)
                    if c1 < nt:
                        ops.join_side()
                        side_pending = False
                        ops.schur_cols(j, jb, lstart, nt, c1, nt, slot)
                else:
                    ops.schur_cols(j, jb, lstart, nt, jb2, nt, slot)
                    factor_and_send(nxt, lstart, nxt % 2, False)
            else:
                ops.schur_cols(j, jb, lstart, nt, 0, nt, slot)
        elif mine_next:                          # pragma: no cover (no trailing columns)
            factor_and_send(nxt, lstart, nxt % 2, False)
    if side_pending:
        ops.join_side()
    for hs in sends.values():
        for h in hs:
            h.wait()
    ipiv, info, seen, top = ops.finish()
    info, seen, top = comm.allreduce_values([info, seen, top], "max")
    info = int(info)
    if info:
        raise SingularPivotError(f"exact zero pivot column at index {info - 1}")
    return ipiv, (seen / top if top > 0 else 1.0)


def solve_block_cyclic(ops, comm, n: int, nb: int, perm: np.ndarray, b_host: np.ndarray):
    """x = U^-1 L^-1 b[perm] with the factors distributed by column blocks
    (solve.py:143-156).  Block b's owner solves its diagonal block and
    updates the remaining right-hand side, then broadcasts it."""
    Q, q = comm.size, comm.rank
    x = ops.solve_vector(np.asarray(b_host, dtype=np.float64)[perm])
    nblk = -(-n // nb)
    for jblk in range(nblk):                       # unit lower, forward
        j = jblk * nb
        jb = min(nb, n - j)
        owner = jblk % Q
        if q == owner:
            lc = (jblk // Q) * nb
            ops.trsv(lc, j, jb, False, x)
            ops.gemv_update(lc, j + jb, n, j, jb, x)
        comm.bcast(x[j:], owner)
    for jblk in reversed(range(nblk)):             # upper, backward
        j = jblk * nb
        jb = min(nb, n - j)
        owner = jblk % Q
        if q == owner:
            lc = (jblk // Q) * nb
            ops.trsv(lc, j, jb, True, x)
            ops.gemv_update(lc, 0, j, j, jb, x)
        comm.bcast(x[:j + jb], owner)
    if comm.allreduce_values([ops.zero_diag()], "max")[0]:
        raise SingularPivotError("zero diagonal entry in U")
    return x


@dataclass
class HplReport:
    """One distributed HPL run (the reference's SolveReport fields plus timing)."""
    n: int
    nb: int
    grid: str
    backend: str
    scaled_residual: float
    raw_residual_inf: float
    norm_a_inf: float
    norm_x_inf: float
    norm_b_inf: float
    growth: float
    seconds_factor: float
    seconds_solve: float
    tflops: float

    @property
    def passed(self) -> bool:
        from .solve import PASS_THRESHOLD
        return self.scaled_residual < PASS_THRESHOLD


def _replicated_rhs(ops, comm):
    ax, _ = ops.row_partials(None)                # b = A @ ones (harness.py:126)
    comm.allreduce(ax, "sum")
    return ax


def _residual(ops, comm, n, nb, x, b):
    """||Ax-b||_inf / ((||A||_inf ||x||_inf + ||b||_inf) n eps) with A
    regenerated in the slabs (solve.py:181-214)."""
    from .solve import _report
    gcols = global_cols(n, nb, comm.size, comm.rank)
    xh = x.cpu().numpy()
    xl = ops.solve_vector(xh[gcols]) if len(gcols) else None
    ax, asum = ops.row_partials(xl)
    comm.allreduce(ax, "sum")
    comm.allreduce(asum, "sum")
    r = (ax - b).abs().max().item()
    return _report(float(r), float(asum.max().item()), float(np.abs(xh).max()),
                   float(b.abs().max().item()), n)


class HplProblem:
    """One distributed HPL problem kept resident: the generated matrix (a
    pristine copy of every rank's slab), the replicated b = A @ 1, and the
    buffers of the factorization.  ``step()`` = restore + factor + solve.
    grid = (P, Q) with P * Q = world size; P = 1 (default) runs the 1 x Q
    driver of this module, P > 1 the 2-D driver of hpl2d.py."""

    def __init__(self, n: int, nb: int, backend: GemmBackend | None = None, *,
                 matrix: str = "uniform", seed: int = 99, depth: int = 4, block: int = 15,
                 alpha: float = 0.5, comm: Comm | None = None, ops=None,
                 grid: tuple[int, int] | None = None, keep_copy: bool | None = None):
        from .matgen import GEN_PARAWILK_RANDOMIZED, GEN_UNIFORM
        self.backend = backend or GemmBackend.native()
        self.comm = comm or Comm()
        check_scaling(self.backend, self.comm.size)
        if not 1 <= nb <= min(n, 1024):
            raise InvalidParamsError(f"nb must be in 1..{min(n, 1024)}, got {nb}")
        P, Q = grid if grid is not None else (1, self.comm.size)
        if P < 1 or Q < 1 or P * Q != self.comm.size:
            raise InvalidParamsError(f"grid {P}x{Q} does not match {self.comm.size} ranks")
        self.n, self.nb, self.P, self.Q = n, nb, P, Q
        self.grid = None
        if P > 1:
            from .hpl2d import DeviceOps2D, Grid
            self.grid = Grid(P, Q, self.comm)
            self.ops = ops or DeviceOps2D(n, nb, P, Q, self.grid.p, self.grid.q, self.backend)
        else:
            self.ops = ops or DeviceOps(n, nb, self.comm.size, self.comm.rank, self.backend)
        self.gen = (GEN_UNIFORM if matrix == "uniform" else GEN_PARAWILK_RANDOMIZED, seed, depth,
                    block, alpha)
        self.ops.generate(*self.gen)
        if self.grid is not None:
            from .hpl2d import rhs_2d
            self.b = rhs_2d(self.ops, self.grid)
        else:
            self.b = _replicated_rhs(self.ops, self.comm)
        # pristine copy of the slab for restore(); large slabs (configs[3]/[4]:
        # 68.7 GB per GPU) are regenerated instead (the PCG64 generator writes
        # at HBM speed), which halves the footprint
        slab = getattr(self.ops, "slab", None)
        big = slab is not None and hasattr(slab, "numel") and slab.numel() * 8 > 32 << 30
        keep = (not big) if keep_copy is None else keep_copy
        self.a0 = slab.clone() if keep and slab is not None and hasattr(slab, "clone") else None
        self.growth = None

    def restore(self) -> None:
        if self.a0 is not None:
            self.ops.slab.copy_(self.a0)
        else:
            self.ops.generate(*self.gen)

    def factor(self):
        if self.grid is not None:
            from .hpl2d import factor_2d
            ipiv, self.growth = factor_2d(self.ops, self.grid, self.n, self.nb)
        else:
            ipiv, self.growth = factor_block_cyclic(self.ops, self.comm, self.n, self.nb)
        return ipiv

    def solve(self, ipiv):
        from .solve import ipiv_to_perm
        perm, bh = ipiv_to_perm(ipiv), self.b.cpu().numpy()
        if self.grid is not None:
            from .hpl2d import solve_2d
            return solve_2d(self.ops, self.grid, self.n, self.nb, perm, bh)
        return solve_block_cyclic(self.ops, self.comm, self.n, self.nb, perm, bh)

    def factor_solve(self):
        return self.solve(self.factor())

    def step(self):
        self.restore()
        return self.factor_solve()

    def verify(self, x):
        self.restore()
        if self.grid is not None:
            from .hpl2d import residual_2d
            return residual_2d(self.ops, self.grid, self.n, self.nb, x, self.b)
        return _residual(self.ops, self.comm, self.n, self.nb, x, self.b)


def hpl_run(n: int, nb: int, backend: GemmBackend | None = None, *, matrix: str = "uniform",
            seed: int = 99, depth: int = 4, block: int = 15, alpha: float = 0.5,
            comm: Comm | None = None, ops=None, grid: tuple[int, int] | None = None) -> HplReport:
    """Generate the matrix distributed (hpl_uniform or randomized ParaWilk,
    matgen.py:149-171), b = A @ 1, factor, solve and verify on a P x Q grid
    (default 1 x world).  Times factor and solve with device events, max over
    ranks."""
    import torch
    prob = HplProblem(n, nb, backend, matrix=matrix, seed=seed, depth=depth, block=block,
                      alpha=alpha, comm=comm, ops=ops, grid=grid)
    comm, backend = prob.comm, prob.backend
    prob.restore()
    comm.barrier()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    ipiv = prob.factor()
    growth = prob.growth
    e1.record()
    x = prob.solve(ipiv)
    e2.record()
    torch.cuda.synchronize()
    tf, ts = comm.allreduce_values([e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3],
                                   "max")
    rep = prob.verify(x)
    return HplReport(n=n, nb=nb, grid=f"{prob.P}x{prob.Q}", backend=backend.describe(),
                     scaled_residual=rep.scaled_residual, raw_residual_inf=rep.raw_residual_inf,
                     norm_a_inf=rep.norm_a_inf, norm_x_inf=rep.norm_x_inf,
                     norm_b_inf=rep.norm_b_inf, growth=growth, seconds_factor=tf,
                     seconds_solve=ts, tflops=2.0 * n ** 3 / 3.0 / (tf + ts) / 1e12)


del math, time
