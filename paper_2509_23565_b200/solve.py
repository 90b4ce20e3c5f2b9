"""Blocked right-looking LU with partial pivoting and residual verification,
on B200 (drop-in for /root/reference/pkg/src/ozemu/solve.py).

Panel factorization, interchanges, trsm and the triangular solves are FP64
CUDA kernels (csrc/lu.cu); the trailing Schur update A22 <- A22 - A21 @ U12
goes through the configured GEMM backend exactly where the reference calls it
(solve.py:130-134): cuBLAS DGEMM for the native comparator, the fused
Ozaki-INT8 tcgen05 GEMM (csrc/gemm_emu.cu) for the emulated backend.  The
whole factorization is one call into the C ABI (`oz_lu_factor`) and runs
asynchronously on the current stream.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .errors import (InvalidParamsError, NonFiniteEntryError, NonSquareError,
                     ShapeMismatchError, SingularPivotError)
from .gemm import BackendKind, FlopCounter, GemmBackend, pair_table, retained_pairs

__all__ = ["PASS_THRESHOLD", "EPSILON", "LuFactors", "SolveReport", "lu_factor", "lu_solve",
           "scaled_residual", "solve_system"]

#: HPL verdict boundary: a run passes when the scaled residual is strictly below.
PASS_THRESHOLD = 16.0
EPSILON = 2.0**-52


@dataclass(frozen=True)
class LuFactors:
    """Packed LU factorization PA = LU (solve.py:41-63).

    ``lu`` holds L strictly below the diagonal (unit diagonal implied) and U
    on and above; ``pivots[i]`` is the original row index at position i.
    When the input was a CUDA tensor, ``lu``/``pivots`` are CUDA tensors
    (``lu`` a column-major view); otherwise frozen numpy arrays.
    """

    lu: object
    pivots: object
    lu_block: int
    growth: float
    _device_lu: object = field(default=None, repr=False, compare=False)
    _device_perm: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if isinstance(self.lu, np.ndarray):
            self.lu.setflags(write=False)
        if isinstance(self.pivots, np.ndarray):
            self.pivots.setflags(write=False)

    @property
    def n(self) -> int:
        return int(self.lu.shape[0])


@dataclass
class SolveReport:
    """Residual metrics plus run metadata for one linear solve (solve.py:159-178)."""

    scaled_residual: float
    raw_residual_inf: float
    norm_a_inf: float
    norm_x_inf: float
    norm_b_inf: float
    n: int
    epsilon: float = EPSILON
    backend: str = ""
    lu_block: int | None = None
    growth: float | None = None
    flops: FlopCounter | None = None
    seconds: float | None = None

    @property
    def passed(self) -> bool:
        return self.scaled_residual < PASS_THRESHOLD


# ------------------------------------------------------------------ helpers
def _as_square_device(a, what="matrix"):
    """-> (device tensor, host_io flag).  Validates 2-D square, nonempty."""
    if _dev.is_device(a):
        x, _ = _dev.to_device_f64(a)
        host = False
    else:
        arr = a if _is_host_tensor(a) else np.asarray(a, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise NonSquareError(f"expected a square matrix, got shape {tuple(arr.shape)}")
        if arr.shape[0] == 0:
            raise InvalidParamsError("empty matrices are not supported")
        x = _upload(arr)
        host = True
    if x.ndim != 2 or x.shape[0] != x.shape[1]:
        raise NonSquareError(f"expected a square matrix, got shape {tuple(x.shape)}")
    if x.shape[0] == 0:
        raise InvalidParamsError("empty matrices are not supported")
    return x, host


def _is_host_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor) and not x.is_cuda
    except ImportError:  # pragma: no cover
        return False


def _host_row_major(a):
    """A square, C-contiguous float64 host matrix (numpy or CPU tensor) the
    overlapped upload can read in place; None otherwise (device inputs and
    other layouts take the plain path)."""
    t = _dev.torch()
    if _dev.is_device(a):
        return None
    if isinstance(a, t.Tensor):
        if (a.dtype != t.float64 or a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] == 0
                or not a.is_contiguous()):
            return None
        return a
    if isinstance(a, np.ndarray) and a.dtype == np.float64 and a.ndim == 2 and \
            a.shape[0] == a.shape[1] and a.shape[0] > 0 and a.flags.c_contiguous:
        return a
    return None


def _upload(x):
    """numpy array or (pinned) CPU tensor -> CUDA float64 tensor."""
    t = _dev.torch()
    if isinstance(x, t.Tensor):
        return x.to(device="cuda", dtype=t.float64, non_blocking=True)
    return t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to("cuda")


def _vector_device(v, n, what):
    t = _dev.torch()
    if _dev.is_device(v):
        x = v.to(t.float64)
    else:
        arr = v if _is_host_tensor(v) else np.asarray(v, dtype=np.float64)
        x = _upload(arr)
    if tuple(x.shape) != (n,):
        raise ShapeMismatchError(f"{what} has shape {tuple(x.shape)}, expected ({n},)")
    return x.contiguous()


def _col_major_copy(x):
    """Column-major (LAPACK order) working copy of a square CUDA matrix."""
    t = _dev.torch()
    n = int(x.shape[0])
    out = t.empty((n, n), dtype=t.float64, device="cuda").t()   # strides (1, n)
    rs, cs = _dev.strides2d(x)
    _lib.call("oz_copy2d", x.data_ptr(), n, n, rs, cs, out.data_ptr(), 1, n, _dev.stream())
    return out


def _count_flops(counter: FlopCounter, n: int, nb: int, backend: GemmBackend) -> None:
    """Same nominal counts as the reference (solve.py:88-90,128-129; gemm.py:224-228,262)."""
    npairs = (len(retained_pairs(backend.splits, backend.truncation))
              if backend.kind is BackendKind.EMULATED_INT8 else 0)
    for j in range(0, n, nb):
        jb = min(nb, n - j)
        t = np.arange(j, j + jb, dtype=np.int64)
        rows = n - t - 1
        counter.add_f64(int((rows + rows * np.maximum(j + jb - t - 1, 0)).sum()))
        rest = n - j - jb
        if rest > 0:
            counter.add_f64(jb * (jb - 1) // 2 * rest)
            if backend.kind is BackendKind.NATIVE_F64:
                counter.add_f64(rest * jb * rest)
            else:
                k = backend.splits
                counter.add_emulated(macs=npairs * rest * jb * rest, pairs=npairs)
                counter.add_f64(npairs * rest * rest + 2 * k * (rest * jb + jb * rest))


def _backend_code(backend: GemmBackend) -> int:
    """C-ABI Schur backend: 0 native, 1 emulated per-vector, 2 emulated GLOBAL
    scaling (split.py:131-134)."""
    if backend.kind is not BackendKind.EMULATED_INT8:
        return 0
    from .split import ScalingMode
    return 2 if backend.scaling is ScalingMode.GLOBAL else 1


def factor_device(a_cm, nb: int, backend: GemmBackend, chunks=None):
    """In-place LU of a column-major CUDA matrix.  Returns (ipiv tensor,
    stats tensor, info tensor) without synchronizing.  chunks = (events,
    width): the matrix is still being uploaded; events[c] (torch.cuda.Event)
    fires once columns [c*width, (c+1)*width) are in place."""
    t = _dev.torch()
    n = int(a_cm.shape[0])
    emulated = backend.kind is BackendKind.EMULATED_INT8
    k = backend.splits if emulated else 0
    if emulated:
        if nb << (2 * backend.slice_bits) >= 1 << 53:
            from .errors import AccumulatorOverflowError
            raise AccumulatorOverflowError("lu_block too large for exact accumulation")
        pa, pb, sh = pair_table(backend)
    else:
        pa = pb = sh = np.zeros(1, dtype=np.int32)
    ws_bytes = int(_lib.query("oz_lu_workspace_bytes", n, nb, k, backend.slice_bits))
    ws = t.empty((ws_bytes,), dtype=t.uint8, device="cuda")
    ipiv = t.empty((n,), dtype=t.int32, device="cuda")
    stats = t.zeros((4,), dtype=t.float64, device="cuda")
    info = t.zeros((1,), dtype=t.int32, device="cuda")
    if chunks is None:
        _lib.call("oz_lu_factor", a_cm.data_ptr(), n, int(a_cm.stride(1)), nb,
                  _backend_code(backend), k, backend.slice_bits, len(pa), pa.ctypes.data,
                  pb.ctypes.data, sh.ctypes.data, ipiv.data_ptr(), stats.data_ptr(),
                  info.data_ptr(), ws.data_ptr(), ws_bytes, _dev.stream())
    else:
        events, width = chunks
        handles = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
        _lib.call("oz_lu_factor_overlapped", a_cm.data_ptr(), n, int(a_cm.stride(1)), nb,
                  _backend_code(backend), k, backend.slice_bits, len(pa), pa.ctypes.data,
                  pb.ctypes.data, sh.ctypes.data, ipiv.data_ptr(), stats.data_ptr(),
                  info.data_ptr(), ws.data_ptr(), ws_bytes, handles, width, _dev.stream())
    return ipiv, stats, info, ws


_UPLOAD_STREAMS = {}


def _upload_overlapped(host, nb: int):
    """Row-major host matrix -> (row-major device copy, column-major working
    copy, (per-block events, block width), non-finite flag) in column blocks:
    a copy stream moves block c over PCIe (cudaMemcpy2DAsync) while a second
    stream transposes block c-1 and checks it for NaN/inf; oz_lu_factor_
    overlapped waits on each block's event just before it first touches it."""
    t = _dev.torch()
    n = int(host.shape[0])
    dev = t.cuda.current_device()
    if dev not in _UPLOAD_STREAMS:
        _UPLOAD_STREAMS[dev] = (t.cuda.Stream(), t.cuda.Stream())
    cs, ts = _UPLOAD_STREAMS[dev]
    cur = t.cuda.current_stream()
    ad = t.empty((n, n), dtype=t.float64, device="cuda")
    work = t.empty((n, n), dtype=t.float64, device="cuda").t()
    bad = t.zeros((1,), dtype=t.int32, device="cuda")
    cs.wait_stream(cur)
    ts.wait_stream(cur)
    w = max(int(os.environ.get("OZ_UPLOAD_BLOCK", "2048")), nb)   # measured best at n = 32768
    w = (w // nb) * nb
    hptr = host.data_ptr() if isinstance(host, t.Tensor) else host.ctypes.data
    events = []
    for c0 in range(0, n, w):
        c1 = min(n, c0 + w)
        _lib.call("oz_memcpy2d_h2d", ad.data_ptr() + 8 * c0, 8 * n, hptr + 8 * c0, 8 * n,
                  8 * (c1 - c0), n, cs.cuda_stream)
        copied = t.cuda.Event()
        copied.record(cs)
        ts.wait_event(copied)
        _lib.call("oz_copy2d", ad.data_ptr() + 8 * c0, n, c1 - c0, n, 1,
                  work.data_ptr() + 8 * n * c0, 1, n, ts.cuda_stream)
        _lib.call("oz_nonfinite_flag", ad.data_ptr() + 8 * c0, n, c1 - c0, n, 1,
                  bad.data_ptr(), ts.cuda_stream)
        done = t.cuda.Event()
        done.record(ts)
        events.append(done)
    return ad, work, (events, w), bad


def ipiv_to_perm(ipiv_host: np.ndarray) -> np.ndarray:
    ipiv_host = np.ascontiguousarray(ipiv_host, dtype=np.int32)
    n = ipiv_host.shape[0]
    perm = np.empty(n, dtype=np.int64)
    _lib.call("oz_ipiv_to_perm", ipiv_host.ctypes.data, n, perm.ctypes.data)
    return perm


def _finish_factor(ipiv, stats, info):
    inf = int(info.item())
    if inf:
        raise SingularPivotError(f"exact zero pivot column at index {inf - 1}")
    st = stats.cpu().numpy()
    growth = float(st[0] / st[1]) if st[1] > 0 else 1.0
    perm = ipiv_to_perm(ipiv.cpu().numpy())
    return perm, growth


# ------------------------------------------------------------------ public API
def lu_factor(a, lu_block: int = 64, schur_backend: GemmBackend | None = None,
              counter: FlopCounter | None = None) -> LuFactors:
    """Factor a square matrix as PA = LU with panel width ``lu_block`` (solve.py:94-140)."""
    x, host = _as_square_device(a)
    n = int(x.shape[0])
    if not bool(_dev.torch().isfinite(x).all().item()):
        raise NonFiniteEntryError("matrix contains NaN or infinite entries")
    if not 1 <= lu_block <= n:
        raise InvalidParamsError(f"lu_block must be in 1..{n}, got {lu_block}")
    if schur_backend is None:
        schur_backend = GemmBackend.native()
    work = _col_major_copy(x)
    ipiv, stats, info, _ws = factor_device(work, lu_block, schur_backend)
    perm, growth = _finish_factor(ipiv, stats, info)
    if counter is not None:
        _count_flops(counter, n, lu_block, schur_backend)
    t = _dev.torch()
    dperm = t.from_numpy(perm).to("cuda")
    if host:
        lu_host = np.asfortranarray(work.t().cpu().numpy().T)
        return LuFactors(lu=lu_host, pivots=perm, lu_block=lu_block, growth=growth,
                         _device_lu=work, _device_perm=dperm)
    return LuFactors(lu=work, pivots=dperm, lu_block=lu_block, growth=growth,
                     _device_lu=work, _device_perm=dperm)


def _solve_device(lu_cm, dperm, b_dev):
    t = _dev.torch()
    n = int(lu_cm.shape[0])
    x = t.empty((n,), dtype=t.float64, device="cuda")
    nbytes = int(_lib.query("oz_lu_solve_workspace_bytes", n))
    ws = t.zeros((nbytes // 4 + 1,), dtype=t.int32, device="cuda")
    _lib.call("oz_lu_solve", lu_cm.data_ptr(), n, int(lu_cm.stride(1)), dperm.data_ptr(),
              b_dev.data_ptr(), x.data_ptr(), ws.data_ptr(), nbytes, _dev.stream())
    return x, ws


def lu_solve(factors: LuFactors, rhs):
    """Solve Ax = b from packed factors (solve.py:143-156)."""
    n = factors.n
    host = not _dev.is_device(rhs)
    b = _vector_device(rhs, n, "rhs")
    t = _dev.torch()
    lu_cm = factors._device_lu
    dperm = factors._device_perm
    if lu_cm is None:
        src = factors.lu
        src_dev = src if _dev.is_device(src) else t.from_numpy(
            np.ascontiguousarray(np.asarray(src, dtype=np.float64))).to("cuda")
        lu_cm = _col_major_copy(src_dev)
    if dperm is None:
        pv = factors.pivots
        dperm = pv.to(t.int64) if _dev.is_device(pv) else t.from_numpy(
            np.asarray(pv, dtype=np.int64)).to("cuda")
    x, flag = _solve_device(lu_cm, dperm, b)
    if int(flag[0].item()):
        raise SingularPivotError("zero diagonal entry in U")
    return x.cpu().numpy() if host else x


def _norms(a_dev, x_dev, b_dev):
    t = _dev.torch()
    n = int(a_dev.shape[0])
    out = t.zeros((4,), dtype=t.float64, device="cuda")
    rs, cs = _dev.strides2d(a_dev)
    _lib.call("oz_residual_norms", a_dev.data_ptr(), n, rs, cs, x_dev.data_ptr(),
              b_dev.data_ptr(), out.data_ptr(), _dev.stream())
    return [float(v) for v in out.cpu().numpy()]


def _report(raw, norm_a, norm_x, norm_b, n, **metadata) -> SolveReport:
    denom = (norm_a * norm_x + norm_b) * n * EPSILON                  # solve.py:198-205
    if raw == 0.0:
        resid = 0.0
    elif denom == 0.0:
        resid = float("inf")
    else:
        resid = raw / denom
    return SolveReport(scaled_residual=resid, raw_residual_inf=raw, norm_a_inf=norm_a,
                       norm_x_inf=norm_x, norm_b_inf=norm_b, n=n, **metadata)


def scaled_residual(a, x, b, **metadata) -> SolveReport:
    """HPL scaled residual ||Ax-b||_inf / ((||A||_inf ||x||_inf + ||b||_inf) n eps)
    with Ax evaluated in FP64 on the device (solve.py:181-214)."""
    ad, _ = _as_square_device(a)
    n = int(ad.shape[0])
    try:
        xd = _vector_device(x, n, "x")
        bd = _vector_device(b, n, "b")
    except ShapeMismatchError:
        raise ShapeMismatchError("x and b must be length-n vectors") from None
    raw, na, nx, nbv = _norms(ad, xd, bd)
    return _report(raw, na, nx, nbv, n, **metadata)


def solve_system(a, b, lu_block: int = 64, backend: GemmBackend | None = None):
    """Factor, solve and verify in one call; wall time covers factor + solve
    (solve.py:217-239).  Device work is synchronized before the clock stops.

    Errors surface in the reference's order: lu_factor's checks (square,
    empty, non-finite, lu_block, singular pivot) before lu_solve's rhs shape
    check (solve.py:227-228)."""
    if backend is None:
        backend = GemmBackend.native()
    t = _dev.torch()
    counter = FlopCounter()
    t0 = time.perf_counter()
    src = _host_row_major(a)
    if src is not None:
        # host matrix: overlapped upload (column blocks over PCIe while the
        # first panels are factored); non-finite entries are caught by a flag
        # folded into the upload, before any result is returned
        n = int(src.shape[0])
        host = True
        if not 1 <= lu_block <= n:
            hv = src.numpy() if isinstance(src, t.Tensor) else src
            if not np.isfinite(hv).all():
                raise NonFiniteEntryError("matrix contains NaN or infinite entries")
            raise InvalidParamsError(f"lu_block must be in 1..{n}, got {lu_block}")
        try:
            ad, work, chunks, bad = _upload_overlapped(src, lu_block)
            ipiv, stats, info, _ws = factor_device(work, lu_block, backend, chunks=chunks)
            if int(bad.item()):
                raise NonFiniteEntryError("matrix contains NaN or infinite entries")
        except BaseException:
            # the copy/transpose side streams may still be writing into
            # ad/work/bad (and reading the host matrix): drain the device
            # before those buffers go back to the caching allocator
            t.cuda.synchronize()
            raise
    else:
        ad, host = _as_square_device(a)
        n = int(ad.shape[0])
        if not bool(t.isfinite(ad).all().item()):
            raise NonFiniteEntryError("matrix contains NaN or infinite entries")
        if not 1 <= lu_block <= n:
            raise InvalidParamsError(f"lu_block must be in 1..{n}, got {lu_block}")
        work = _col_major_copy(ad)
        ipiv, stats, info, _ws = factor_device(work, lu_block, backend)
    perm, growth = _finish_factor(ipiv, stats, info)
    bd = _vector_device(b, n, "rhs")                       # lu_solve's check (solve.py:147-148)
    dperm = t.from_numpy(perm).to("cuda", non_blocking=True)
    x, flag = _solve_device(work, dperm, bd)
    if int(flag[0].item()):
        raise SingularPivotError("zero diagonal entry in U")
    t.cuda.current_stream().synchronize()   # this call's stream only (concurrent callers)
    seconds = time.perf_counter() - t0
    _count_flops(counter, n, lu_block, backend)
    raw, na, nx, nbv = _norms(ad, x, bd)
    report = _report(raw, na, nx, nbv, n, backend=backend.describe(), lu_block=lu_block,
                     growth=growth, flops=counter, seconds=seconds)
    return (x.cpu().numpy() if host else x), report
