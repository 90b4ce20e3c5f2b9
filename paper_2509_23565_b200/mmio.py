"""MatrixMarket array-format I/O for dense FP64 matrices (drop-in for
/root/reference/pkg/src/ozemu/mmio.py:16-48).  Interchange only: values are
written with 17 significant digits, so a round trip is exact."""

from __future__ import annotations

import io
from pathlib import Path

import numpy as np
import scipy.io

__all__ = ["MM_HEADER", "write_matrix_market", "read_matrix_market", "matrix_market_bytes"]

MM_HEADER = "%%MatrixMarket matrix array real general"


def _host(a) -> np.ndarray:
    if hasattr(a, "detach") and hasattr(a, "cpu"):          # torch tensor (any device)
        a = a.detach().cpu().numpy()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def write_matrix_market(target, a, comment: str = "") -> None:
    """Dense array format, column-major value order; `target` is a path or a
    binary file object."""
    a = _host(a)
    kw = dict(comment=comment, field="real", precision=17, symmetry="general")
    if isinstance(target, (str, Path)):
        with open(target, "wb") as fh:
            scipy.io.mmwrite(fh, a, **kw)
    else:
        scipy.io.mmwrite(target, a, **kw)


def read_matrix_market(source) -> np.ndarray:
    return np.asarray(scipy.io.mmread(source), dtype=np.float64)


def matrix_market_bytes(a, comment: str = "") -> bytes:
    buf = io.BytesIO()
    write_matrix_market(buf, a, comment)
    return buf.getvalue()
