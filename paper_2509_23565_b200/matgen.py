"""Test-matrix generators on the GPU (drop-in for
/root/reference/pkg/src/ozemu/matgen.py:39-171).

The ParaWilk pattern, the randomized 2*U(0,1)^2 overlay and the HPL
U(-1/2, 1/2) matrix are produced by the sm_100a generator kernel
(csrc/matgen.cu), bit-identical with numpy's ``default_rng(seed).random``
stream (element (i, j) = stream position i*n + j).  numpy is used only to
derive the 128-bit PCG64 seed state from the integer seed (SeedSequence).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import (InvalidDimError, InvalidParamsError, InvalidPermutationError,
                     NonPowerOfTwoScaleError, ShapeMismatchError)

__all__ = ["ParaWilkParams", "parawilk", "parawilk_randomized", "hpl_uniform", "wilkinson",
           "turing", "turing_inverse", "generalized_fibonacci", "nnz_pattern", "DiagonalScale",
           "Permutation", "apply_scaling", "generate_device", "pcg64_state"]

GEN_UNIFORM, GEN_PARAWILK, GEN_PARAWILK_RANDOMIZED = 0, 1, 2


@dataclass(frozen=True)
class ParaWilkParams:
    """Parameters of the ParaWilk family (matgen.py:39-72)."""

    n: int
    depth: int
    block: int
    alpha: float = 1.0
    randomize: bool = False
    seed: int | None = None

    def __post_init__(self):
        if self.n < 2:
            raise InvalidDimError("n must be >= 2")
        if self.depth < 1:
            raise InvalidParamsError("depth must be >= 1")
        if self.block < 1:
            raise InvalidParamsError("block must be >= 1")
        if not np.isfinite(self.alpha) or self.alpha == 0.0:
            raise InvalidParamsError("alpha must be finite and nonzero")
        if self.depth > self.n - 1:
            object.__setattr__(self, "depth", self.n - 1)

    def describe(self) -> str:
        tag = f"parawilk[n={self.n},d={self.depth},b={self.block},alpha={self.alpha!r}"
        if self.randomize:
            tag += f",randomized,seed={self.seed}"
        return tag + "]"


def pcg64_state(seed: int) -> tuple[int, int]:
    """(state, inc) of numpy's PCG64 after SeedSequence(seed) seeding."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def generate_device(kind: int, n: int, seed: int | None = None, depth: int = 1, block: int = 1,
                    alpha: float = 1.0, layout: str = "C", out=None):
    """Generate an n x n matrix directly in HBM.  layout 'C' = row-major
    (numpy order), 'F' = column-major (LU order)."""
    t = _dev.torch()
    if out is None:
        out = t.empty((n, n), dtype=t.float64, device="cuda")
        if layout == "F":
            out = out.t()  # column-major view of the same shape
    rs, cs = _dev.strides2d(out)
    state, inc = pcg64_state(seed) if seed is not None else (0, 0)
    m64 = (1 << 64) - 1
    _lib.call("oz_generate", kind, n, depth, block, float(alpha), state >> 64, state & m64,
              inc >> 64, inc & m64, out.data_ptr(), rs, cs, _dev.stream())
    return out


def _to_host(x) -> np.ndarray:
    return x.cpu().numpy()


def parawilk(params: ParaWilkParams) -> np.ndarray:
    """Deterministic ParaWilk pattern (matgen.py:133-146)."""
    return _to_host(generate_device(GEN_PARAWILK, params.n, None, params.depth, params.block,
                                    params.alpha))


def parawilk_randomized(params: ParaWilkParams) -> np.ndarray:
    """ParaWilk pattern with the zero positions filled by 2*U(0,1)**2 (matgen.py:149-161)."""
    if params.seed is None:
        raise InvalidParamsError("a seed is required for randomized generation")
    return _to_host(generate_device(GEN_PARAWILK_RANDOMIZED, params.n, params.seed, params.depth,
                                    params.block, params.alpha))


def hpl_uniform(n: int, seed: int) -> np.ndarray:
    """n-by-n i.i.d. U(-1/2, 1/2), row-major fill order (matgen.py:164-171)."""
    if n < 1:
        raise InvalidDimError("n must be >= 1")
    if seed is None:
        raise InvalidParamsError("a seed is required")
    return _to_host(generate_device(GEN_UNIFORM, n, seed))


def wilkinson(n: int) -> np.ndarray:
    """Unit diagonal, -1 below, ones in the last column (matgen.py:75-83) —
    the ParaWilk pattern with depth n-1 and one alpha=1 column at n-1."""
    if n < 2:
        raise InvalidDimError("n must be >= 2")
    return _to_host(generate_device(GEN_PARAWILK, n, None, n - 1, n - 1, 1.0))


def turing(n: int, depth: int) -> np.ndarray:
    """Unit lower triangular with -1 on subdiagonals 1..depth (matgen.py:86-95)."""
    if n < 2:
        raise InvalidDimError("n must be >= 2")
    if not 1 <= depth <= n - 1:
        raise InvalidDimError(f"depth must be in 1..{n - 1}")
    return _to_host(generate_device(GEN_PARAWILK, n, None, depth, n, 1.0))


# ---------------------------------------------------------------------------
# Host test-matrix utilities (matgen.py:98-130, 174-251).  Tiny exact-integer
# and exact-scaling helpers the reference exports next to its generators; no
# configuration of the hot path uses them, so they stay host code.

def generalized_fibonacci(order: int, count: int) -> list[int]:
    """f[0] = 1, f[i] = f[i-1] + ... + f[i-order] (missing terms count as 0)
    (matgen.py:116-130); order 2 is Fibonacci."""
    if order < 1:
        raise InvalidParamsError("order must be >= 1")
    if count < 1:
        raise InvalidParamsError("count must be >= 1")
    f = [1]
    window = 1                      # running sum of the last `order` terms
    for i in range(1, count):
        f.append(window)
        window += f[i]
        if i - order >= 0:
            window -= f[i - order]
    return f


def turing_inverse(n: int, depth: int) -> np.ndarray:
    """Exact inverse of turing(n, depth) as an object array of Python ints
    (matgen.py:98-113).  turing() is unit lower triangular Toeplitz with -1 on
    subdiagonals 1..depth, so its inverse is lower triangular Toeplitz with
    the order-`depth` generalized Fibonacci numbers down each column."""
    if n < 2:
        raise InvalidDimError("n must be >= 2")
    if not 1 <= depth <= n - 1:
        raise InvalidDimError(f"depth must be in 1..{n - 1}")
    f = generalized_fibonacci(depth, n)
    inv = np.empty((n, n), dtype=object)
    for i in range(n):
        for j in range(n):
            inv[i, j] = f[i - j] if i >= j else 0
    return inv


def nnz_pattern(a) -> np.ndarray:
    """uint8 indicator of the nonzero entries (matgen.py:174-176)."""
    return np.not_equal(a, 0).astype(np.uint8)


@dataclass(frozen=True)
class DiagonalScale:
    """Diagonal scaling by signed powers of two, exact in FP64 (matgen.py:179-195)."""

    entries: np.ndarray

    def __post_init__(self):
        e = np.atleast_1d(np.asarray(self.entries, dtype=np.float64))
        if e.ndim != 1 or e.size == 0:
            raise InvalidParamsError("diagonal entries must form a nonempty vector")
        frac, _ = np.frexp(e)
        if not np.isfinite(e).all() or not (np.abs(frac) == 0.5).all():
            raise NonPowerOfTwoScaleError("diagonal entries must be nonzero signed powers of two")
        e = e.copy()
        e.setflags(write=False)
        object.__setattr__(self, "entries", e)


@dataclass(frozen=True)
class Permutation:
    """Gather permutation: output position i takes input index indices[i]
    (matgen.py:198-216)."""

    indices: np.ndarray

    def __post_init__(self):
        idx = np.atleast_1d(np.asarray(self.indices))
        if idx.ndim != 1 or idx.size == 0 or not np.issubdtype(idx.dtype, np.integer):
            raise InvalidPermutationError("indices must form a nonempty integer vector")
        seen = np.zeros(idx.size, dtype=bool)
        ok = bool(((idx >= 0) & (idx < idx.size)).all())
        if ok:
            seen[idx] = True
            ok = bool(seen.all())
        if not ok:
            raise InvalidPermutationError("indices are not a permutation of 0..n-1")
        idx = idx.copy()
        idx.setflags(write=False)
        object.__setattr__(self, "indices", idx)


def _apply_side(out: np.ndarray, op, axis: int, side: str) -> np.ndarray:
    size = out.shape[axis]
    what = "row" if axis == 0 else "column"
    if isinstance(op, DiagonalScale):
        if op.entries.size != size:
            raise ShapeMismatchError(f"{side} diagonal length must match {what} count")
        return out * (op.entries[:, None] if axis == 0 else op.entries[None, :])
    if isinstance(op, Permutation):
        if op.indices.size != size:
            raise ShapeMismatchError(f"{side} permutation length must match {what} count")
        return np.take(out, op.indices, axis=axis)
    raise InvalidParamsError(f"{side} must be DiagonalScale or Permutation")


def apply_scaling(a, left=None, right=None) -> np.ndarray:
    """Exact power-of-two scalings / permutations of rows (left) and columns
    (right) (matgen.py:219-251); returns a new array."""
    out = np.array(a, dtype=np.float64, copy=True)
    if out.ndim != 2:
        raise ShapeMismatchError("expected a 2-D matrix")
    if left is not None:
        out = _apply_side(out, left, 0, "left")
    if right is not None:
        out = _apply_side(out, right, 1, "right")
    return out
