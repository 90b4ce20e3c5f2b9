"""CPU oracle for the Ozaki-INT8 HPL hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (arXiv 2509.23565 reference
package `ozemu`, /root/reference/pkg/src/ozemu), written independently and
used only as the checker: by tests/, by __graft_entry__.smoke() and by
bench.py's cpu_baseline / --impl reference leg.  The product path
(paper_2509_23565_b200) never imports this module.

Pinned against the reference itself: tests/golden/*.npz were produced by
oracle/make_golden.py, which imports the reference from /root/reference in
the build container; tests/test_oracle_golden.py checks this restatement
against those fixtures bit-for-bit (integer/byte work, the emulated GEMM and
the unblocked LU) and to tolerance where the reference calls LAPACK/BLAS.

Each function cites the reference lines it restates.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

EPS = 2.0**-52  # solve.py:38
THRESHOLD = 16.0  # solve.py:36

ROW, COL = "row", "col"
PER_VECTOR, GLOBAL = "pervector", "global"


# ----------------------------------------------------------------- splitting
def split(a, k: int, q: int = 7, orient: str = ROW, mode: str = PER_VECTOR):
    """split.py:109-160.  Returns (slices [k, rows, cols] int8/int16, exps int64)."""
    a = np.asarray(a, dtype=np.float64)
    mag = np.abs(a)
    if mode == GLOBAL:                                           # split.py:131-134
        e = np.frexp(mag.max())[1]
        exps = np.full(a.shape[0] if orient == ROW else a.shape[1], e, dtype=np.int64)
    else:                                                        # split.py:135-138
        exps = np.frexp(mag.max(axis=1 if orient == ROW else 0))[1].astype(np.int64)
    scale = exps[:, None] if orient == ROW else exps[None, :]
    x = np.ldexp(a, -scale)                                      # split.py:142
    out = np.empty((k,) + a.shape, dtype=np.int8 if q <= 7 else np.int16)
    r = float(2**q)
    for s in range(k):                                           # split.py:147-151
        y = x * r
        t = np.trunc(y)
        out[s] = t
        x = y - t
    return out, exps


def reconstruct(slices, exps, q: int, orient: str = ROW):
    """split.py:163-172."""
    scale = exps[:, None] if orient == ROW else exps[None, :]
    out = np.zeros(slices.shape[1:])
    for s in range(slices.shape[0]):
        out += np.ldexp(slices[s].astype(np.float64), scale - (s + 1) * q)
    return out


# ---------------------------------------------------------------- emulated GEMM
def pairs(k: int, limit: int | None = None):
    """gemm.py:157-178: (i, j) 1-based with i+j <= limit, sorted by (i+j, i).
    limit None = Full (2k); default Band is k+1 (gemm.py:107-108)."""
    lim = 2 * k if limit is None else limit
    out = [(i, j) for i in range(1, k + 1) for j in range(1, k + 1) if i + j <= lim]
    return sorted(out, key=lambda ij: (ij[0] + ij[1], ij[0]))


def emulated_product(a, b, k: int, q: int = 7, limit: int | None = None,
                     mode: str = PER_VECTOR):
    """gemm.py:190-229 (without the host-exactness guards)."""
    sa, ea = split(a, k, q, ROW, mode)
    sb, eb = split(b, k, q, COL, mode)
    base = ea[:, None] + eb[None, :]
    out = np.zeros((a.shape[0], b.shape[1]))
    for i, j in pairs(k, limit):
        ai, bj = sa[i - 1], sb[j - 1]
        if not (ai.any() and bj.any()):                          # gemm.py:219-220
            continue
        prod = ai.astype(np.float64) @ bj.astype(np.float64)     # exact integers
        out += np.ldexp(prod, base - (i + j) * q)                # gemm.py:222
    return out


def pair_product(a, b, k: int, i: int, j: int, q: int = 7, mode: str = PER_VECTOR):
    """Raw integer product of slice pair (i, j), 1-based (test_gemm.py:218-240)."""
    sa, _ = split(a, k, q, ROW, mode)
    sb, _ = split(b, k, q, COL, mode)
    return sa[i - 1].astype(np.int64) @ sb[j - 1].astype(np.int64)


def gemm(alpha, a, b, beta, c=None, k: int | None = None, q: int = 7,
         limit: int | None = -1, mode: str = PER_VECTOR):
    """gemm.py:232-271.  k=None -> native FP64; limit=-1 -> default Band(k+1)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if k is None:
        ab = a @ b
    else:
        lim = k + 1 if limit == -1 else limit
        ab = emulated_product(a, b, k, q, lim, mode)
    out = ab
    if alpha != 1.0:
        out = alpha * ab
    if c is not None and beta != 0.0:
        out = out + beta * np.asarray(c, dtype=np.float64)
    return out


# ------------------------------------------------------------------------ LU
def lu_factor(a, nb: int = 64, k: int | None = None, q: int = 7,
              limit: int | None = -1, mode: str = PER_VECTOR):
    """solve.py:66-140.  Returns (lu F-order, perm, growth)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    lu = np.array(a, order="F", copy=True)
    perm = np.arange(n)
    top = float(np.abs(a).max())
    seen = 0.0
    for j in range(0, n, nb):
        jb = min(nb, n - j)
        for t in range(j, j + jb):                               # solve.py:75-90
            p = t + int(np.argmax(np.abs(lu[t:, t])))
            if lu[p, t] == 0.0:
                raise ZeroDivisionError(f"exact zero pivot column at index {t}")
            if p != t:
                lu[[t, p], :] = lu[[p, t], :]
                perm[[t, p]] = perm[[p, t]]
            if t + 1 < n:
                lu[t + 1:, t] /= lu[t, t]
                if t + 1 < j + jb:
                    lu[t + 1:, t + 1:j + jb] -= np.outer(lu[t + 1:, t], lu[t, t + 1:j + jb])
                    seen = max(seen, float(np.abs(lu[t + 1:, t + 1:j + jb]).max()))
        if j + jb < n:                                           # solve.py:121-137
            lu[j:j + jb, j + jb:] = solve_triangular(
                lu[j:j + jb, j:j + jb], lu[j:j + jb, j + jb:], lower=True,
                unit_diagonal=True, check_finite=False)
            lu[j + jb:, j + jb:] = gemm(-1.0, lu[j + jb:, j:j + jb], lu[j:j + jb, j + jb:],
                                        1.0, lu[j + jb:, j + jb:], k=k, q=q, limit=limit,
                                        mode=mode)
            seen = max(seen, float(np.abs(lu[j + jb:, j + jb:]).max()))
        seen = max(seen, float(np.abs(np.triu(lu[j:j + jb, j:])).max()))
    growth = seen / top if top > 0 else 1.0
    return lu, perm, growth


def lu_solve(lu, perm, b):
    """solve.py:143-156."""
    x = np.asarray(b, dtype=np.float64)[perm]
    x = solve_triangular(lu, x, lower=True, unit_diagonal=True, check_finite=False)
    return solve_triangular(lu, x, lower=False, check_finite=False)


def residual(a, x, b):
    """solve.py:181-214 -> (scaled, raw, ||A||, ||x||, ||b||)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    raw = float(np.abs(a @ x - b).max())
    na = float(np.abs(a).sum(axis=1).max())
    nx = float(np.abs(x).max())
    nbv = float(np.abs(b).max())
    den = (na * nx + nbv) * n * EPS
    scaled = 0.0 if raw == 0.0 else (float("inf") if den == 0.0 else raw / den)
    return scaled, raw, na, nx, nbv


def solve(a, nb: int = 64, k: int | None = None):
    """harness.py:124-128 + solve.py:217-239: b = A@1, factor, solve, residual."""
    a = np.asarray(a, dtype=np.float64)
    b = a @ np.ones(a.shape[0])
    lu, perm, growth = lu_factor(a, nb, k)
    x = lu_solve(lu, perm, b)
    return residual(a, x, b)[0], growth


# ---------------------------------------------------------------- generators
def parawilk(n: int, d: int, blk: int, alpha: float = 1.0):
    """matgen.py:133-146 (d capped at n-1, matgen.py:65-66)."""
    d = min(d, n - 1)
    i, j = np.indices((n, n))
    a = np.where((i - j >= 1) & (i - j <= d), -1.0, 0.0)
    a[np.arange(n), np.arange(n)] = 1.0
    for c in range(blk, n, blk):
        a[:c, c] = alpha
    return a


def parawilk_randomized(n, d, blk, alpha, seed):
    """matgen.py:149-161."""
    base = parawilk(n, d, blk, alpha)
    u = np.random.default_rng(seed).random((n, n))
    return np.where(base != 0.0, base, 2.0 * u * u)


def hpl_uniform(n, seed):
    """matgen.py:164-171."""
    return np.random.default_rng(seed).random((n, n)) - 0.5


# PCG64 restatement (numpy's default_rng bit generator).
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1


def pcg64_seed_state(seed: int):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def pcg64_advance(state: int, inc: int, delta: int) -> int:
    acc_m, acc_p, cm, cp = 1, 0, PCG_MULT, inc
    while delta > 0:
        if delta & 1:
            acc_m = (acc_m * cm) & M128
            acc_p = (acc_p * cm + cp) & M128
        cp = ((cm + 1) * cp) & M128
        cm = (cm * cm) & M128
        delta >>= 1
    return (acc_m * state + acc_p) & M128


def pcg64_uniform_at(seed: int, index: int) -> float:
    """random() value at stream position `index` (row-major i*n+j)."""
    state, inc = pcg64_seed_state(seed)
    s = pcg64_advance(state, inc, index + 1)
    hi, lo = s >> 64, s & ((1 << 64) - 1)
    x = hi ^ lo
    rot = hi >> 58
    x = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
    return (x >> 11) * 2.0**-53
