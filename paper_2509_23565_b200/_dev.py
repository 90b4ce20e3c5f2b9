"""Device-side plumbing shared by the drop-in modules: host<->device
conversion, workspaces and thin wrappers over the C ABI.

Inputs may be numpy arrays (copied to the GPU; results come back as numpy,
exactly like the reference) or CUDA torch tensors (zero-copy; results stay on
the device).  PyTorch is used only for device memory and streams.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import InvalidParamsError, NonFiniteEntryError


def torch():
    return _lib.require_cuda()


def is_device(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor) and x.is_cuda


def to_device_f64(x):
    """Return (tensor float64 on cuda, was_numpy)."""
    t = torch()
    if isinstance(x, t.Tensor):
        if not x.is_cuda:
            x = x.to("cuda")
        if x.dtype != t.float64:
            x = x.to(t.float64)
        return x, False
    arr = np.asarray(x, dtype=np.float64)
    return t.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False), True


def stream() -> int:
    return _lib.stream_handle()


def strides2d(x):
    """(row_stride, col_stride) in elements of a 2-D tensor."""
    return int(x.stride(0)), int(x.stride(1))


class SplitResult:
    """Device slice stack: slices [planes, nvec, ld] int8 (K-major; planes = k,
    or 2k (hi, lo) planes for q > 7), exps int32[nvec]."""

    __slots__ = ("slices", "exps", "ld", "nvec", "inner", "k")

    def __init__(self, slices, exps, ld, nvec, inner, k):
        self.slices, self.exps, self.ld, self.nvec, self.inner, self.k = (
            slices, exps, ld, nvec, inner, k)


def split_device(a, k: int, q: int, orientation: int, mode: int) -> SplitResult:
    """oz_split on a 2-D float64 CUDA tensor (any strides)."""
    t = torch()
    rows, cols = int(a.shape[0]), int(a.shape[1])
    nvec, inner = (rows, cols) if orientation == 0 else (cols, rows)
    ld = max(16, -(-inner // 16) * 16)
    planes = 2 * k if q > 7 else k   # q > 7: (hi, lo) int8 planes per int16 slice
    slices = t.empty((planes, nvec, ld), dtype=t.int8, device=a.device)
    exps = t.empty((nvec,), dtype=t.int32, device=a.device)
    aux = t.empty((4,), dtype=t.int32, device=a.device)
    rs, cs = strides2d(a)
    _lib.call("oz_split", a.data_ptr(), rows, cols, rs, cs, orientation, mode, k, q,
              slices.data_ptr(), ld, nvec * ld, exps.data_ptr(), aux.data_ptr(), stream())
    if int(aux[0].item()) != 0:
        raise NonFiniteEntryError("matrix contains NaN or infinite entries")
    return SplitResult(slices, exps, ld, nvec, inner, k)


def check_finite_device(a, name: str = "matrix") -> None:
    t = torch()
    if not bool(t.isfinite(a).all().item()):
        raise NonFiniteEntryError(f"{name} contains NaN or infinite entries")


def require_2d(a, err=InvalidParamsError, what="matrix"):
    if a.ndim != 2:
        raise err(f"expected a 2-D {what}, got ndim={a.ndim}")
