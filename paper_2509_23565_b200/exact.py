"""Exact matrix products on the host, the checker behind ``gemm_error_profile``
(drop-in for /root/reference/pkg/src/ozemu/oracle.py:1-108, exported there as
``ozemu.oracle``).

Every finite FP64 value is a dyadic rational m * 2^e with |m| < 2^53, so a
whole matrix is one integer matrix times a single power of two (the smallest
exponent present).  The product of two such matrices is then an exact integer
matrix times 2^(sa + sb), computed here with Python integers through numpy's
object-dtype matmul.  This is error-study tooling for small shapes (inner
dimension of a few hundred): it checks the GPU output, it is never on the
solve path, and it shares no arithmetic with the emulated GEMM it checks.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from .errors import ShapeMismatchError

__all__ = ["exact_gemm_scaled", "exact_gemm_fractions", "exact_gemm_float",
           "abs_error_vs_exact", "rel_error_vs_exact"]


def _as_dyadic(m) -> tuple[np.ndarray, int]:
    """m (FP64, finite) -> (object array of Python ints N, s) with m == N * 2**s."""
    m = np.asarray(m, dtype=np.float64)
    frac, ex = np.frexp(m)
    sig = np.ldexp(frac, 53).astype(np.int64)          # |sig| < 2^53, exact
    ex = ex.astype(np.int64) - 53
    live = sig != 0
    s = int(ex[live].min()) if live.any() else 0
    shifts = np.where(live, ex - s, 0)
    ints = np.empty(m.shape, dtype=object)
    flat_i, flat_sig, flat_sh = ints.reshape(-1), sig.reshape(-1), shifts.reshape(-1)
    for t in range(flat_i.size):
        flat_i[t] = int(flat_sig[t]) << int(flat_sh[t])
    return ints, s


def _product(a, b) -> tuple[np.ndarray, int]:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeMismatchError(f"cannot multiply {a.shape} by {b.shape}")
    ai, sa = _as_dyadic(a)
    bi, sb = _as_dyadic(b)
    if a.shape[1] == 0:
        prod = np.empty((a.shape[0], b.shape[1]), dtype=object)
        prod.fill(0)
    else:
        prod = ai.dot(bi)                                  # Python-int dot products: exact
    return prod, sa + sb


def _frac(v: int, s: int) -> Fraction:
    return Fraction(v << s) if s >= 0 else Fraction(v, 1 << -s)


def exact_gemm_scaled(a, b) -> tuple[list[list[int]], int]:
    """A @ B exactly, as (integer rows, s) with C[i][j] == ints[i][j] * 2**s."""
    prod, s = _product(a, b)
    return [[int(v) for v in row] for row in prod], s


def exact_gemm_fractions(a, b) -> list[list[Fraction]]:
    """A @ B exactly, as nested lists of Fractions."""
    prod, s = _product(a, b)
    return [[_frac(int(v), s) for v in row] for row in prod]


def exact_gemm_float(a, b) -> np.ndarray:
    """A @ B rounded once per element to the nearest FP64 value."""
    prod, s = _product(a, b)
    out = np.empty(prod.shape, dtype=np.float64)
    for idx, v in np.ndenumerate(prod):
        out[idx] = float(_frac(int(v), s))
    return out


def _diffs(approx, a, b):
    approx = np.asarray(approx, dtype=np.float64)
    prod, s = _product(a, b)
    if approx.shape != prod.shape:
        raise ShapeMismatchError(f"approx has shape {approx.shape}, product is {prod.shape}")
    for idx, v in np.ndenumerate(prod):
        exact = _frac(int(v), s)
        yield idx, abs(Fraction(float(approx[idx])) - exact), exact


def abs_error_vs_exact(approx, a, b) -> np.ndarray:
    """|approx - A@B| per element; the difference is exact, rounded once."""
    out = np.empty(np.shape(approx), dtype=np.float64)
    for idx, diff, _ in _diffs(approx, a, b):
        out[idx] = float(diff)
    return out


def rel_error_vs_exact(approx, a, b) -> np.ndarray:
    """|approx - A@B| / |A@B| per element; 0/0 -> 0, x/0 -> inf."""
    out = np.empty(np.shape(approx), dtype=np.float64)
    for idx, diff, exact in _diffs(approx, a, b):
        if exact == 0:
            out[idx] = 0.0 if diff == 0 else np.inf
        else:
            out[idx] = float(diff / abs(exact))
    return out
