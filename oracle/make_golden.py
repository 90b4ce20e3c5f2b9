"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

The fixtures pin both the CPU oracle (oracle/ozaki_oracle.py) and the GPU
path.  Every fixture is produced by calling the reference's public API
(ozemu.split_matrix, ozemu.gemm, ozemu.lu_factor, ozemu.sweep_splits, ...);
Schur-update operands are captured by spying on the reference LU's gemm call
(SURVEY A.6).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    sys.path.insert(0, REF)
    import ozemu
    from ozemu import (FULL, Band, GemmBackend, MatrixSpec, Orientation, ParaWilkParams,
                       ScalingMode, gemm, hpl_uniform, lu_factor, parawilk, parawilk_randomized,
                       solve_system, split_matrix, sweep_splits)

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20240901)

    # ---- split fixtures (split.py:109-160)
    split_cases = {}
    wide = (rng.random((9, 13)) - 0.5) * np.ldexp(1.0, rng.integers(-60, 61, size=(9, 1)))
    zero_rows = rng.random((6, 5)) - 0.5
    zero_rows[[1, 4]] = 0.0
    inputs = {
        "uniform": rng.random((7, 19)) - 0.5,
        "wide": wide,
        "range2x2": np.array([[2.0**53, 2.0**53], [2.0**-53, 2.0**-53]]),
        "zero_rows": zero_rows,
        "big": (rng.random((37, 70)) * 100 - 50),
        "subnormal": np.array([[5e-324, -1e-310, 3e-320], [1.0, 2.0**-1074, -0.0]]),
        "huge": np.array([[1.7e308, -1e300, 1e-300], [2.0**1023, 1.0, -3.0]]),
    }
    idx = 0
    for name, a in inputs.items():
        for k in (1, 3, 7, 9):
            for orient in (Orientation.ROW_SCALED, Orientation.COL_SCALED):
                for mode in (ScalingMode.PER_VECTOR, ScalingMode.GLOBAL):
                    st = split_matrix(a, k, 7, orient, mode)
                    key = f"s{idx}"
                    split_cases[key + "_a"] = a
                    split_cases[key + "_meta"] = np.array(
                        [k, 7, 0 if orient is Orientation.ROW_SCALED else 1,
                         0 if mode is ScalingMode.PER_VECTOR else 1])
                    split_cases[key + "_slices"] = np.stack(st.slices)
                    split_cases[key + "_exps"] = st.exponents
                    idx += 1
    split_cases["count"] = np.array([idx])
    np.savez_compressed(os.path.join(OUT, "split.npz"), **split_cases)

    # ---- emulated gemm fixtures (gemm.py:190-271)
    g = {}
    idx = 0

    def add(a, b, k, trunc, alpha=1.0, beta=0.0, c=None, scaling=ScalingMode.PER_VECTOR):
        nonlocal idx
        bk = GemmBackend.int8(k, 7, truncation=trunc, scaling=scaling)
        out = gemm(bk, alpha, a, b, beta, c)
        limit = 2 * k if trunc is FULL else trunc.limit
        key = f"g{idx}"
        g[key + "_a"], g[key + "_b"] = a, b
        g[key + "_c"] = c if c is not None else np.zeros((0, 0))
        g[key + "_meta"] = np.array([k, limit, 0 if scaling is ScalingMode.PER_VECTOR else 1],
                                    dtype=np.int64)
        g[key + "_ab"] = np.array([alpha, beta])
        g[key + "_out"] = out
        idx += 1

    a = rng.random((33, 45)) - 0.5
    b = rng.random((45, 29)) - 0.5
    for k in range(1, 10):
        add(a, b, k, Band(k + 1))
    add(a, b, 9, FULL)
    add(a, b, 4, Band(6))
    aw = (rng.random((40, 150)) - 0.5) * np.ldexp(1.0, rng.integers(-60, 61, size=(40, 1)))
    bw = (rng.random((150, 36)) - 0.5) * np.ldexp(1.0, rng.integers(-60, 61, size=(1, 36)))
    for k in (3, 7, 9):
        add(aw, bw, k, Band(k + 1))
    c = rng.random((33, 29)) - 0.5
    add(a, b, 4, Band(5), alpha=-2.0, beta=0.5, c=c)
    add(a, b, 7, Band(8), alpha=-1.0, beta=1.0, c=c)
    add(np.array([[2.0**40, 0.0], [0.0, 2.0**-40]]), np.eye(2), 4, Band(5),
        scaling=ScalingMode.GLOBAL)
    a3 = rng.random((200, 300)) - 0.5
    b3 = rng.random((300, 170)) - 0.5
    add(a3, b3, 7, Band(8))
    g["count"] = np.array([idx])
    np.savez_compressed(os.path.join(OUT, "gemm.npz"), **g)

    # ---- Schur-update captures from the reference LU
    sol = sys.modules["ozemu.solve"]
    real = sol.gemm
    cap = {}
    calls = []

    def spy(backend, alpha, A, B, beta, C=None, counter=None):
        out = real(backend, alpha, A, B, beta, C, counter)
        calls.append((backend.splits, np.array(A), np.array(B), np.array(C), out))
        return out

    p = ParaWilkParams(256, 4, 15, 0.5, randomize=True, seed=42)
    apw = parawilk_randomized(p)
    sol.gemm = spy
    try:
        for k in (3, 7, 9):
            lu_factor(apw, 64, GemmBackend.int8(k))
    finally:
        sol.gemm = real
    for i, (k, A, B, Cm, out) in enumerate(calls):
        cap[f"c{i}_k"] = np.array([k])
        cap[f"c{i}_a"], cap[f"c{i}_b"], cap[f"c{i}_c"], cap[f"c{i}_out"] = A, B, Cm, out
    cap["count"] = np.array([len(calls)])
    np.savez_compressed(os.path.join(OUT, "schur.npz"), **cap)

    # ---- LU fixtures (solve.py)
    lu = {}
    a24 = rng.random((24, 24)) - 0.5
    f = lu_factor(a24, 24)
    lu["unblocked_a"], lu["unblocked_lu"], lu["unblocked_perm"] = a24, f.lu, f.pivots
    lu["unblocked_growth"] = np.array([f.growth])
    a64 = np.random.default_rng(11).random((64, 64)) - 0.5
    f16 = lu_factor(a64, 16)
    lu["blocked_a"], lu["blocked_lu"], lu["blocked_perm"] = a64, f16.lu, f16.pivots
    for n in range(5, 21):
        lu[f"wilkinson_{n}_growth"] = np.array([lu_factor(ozemu.wilkinson(n), min(4, n)).growth])
    np.savez_compressed(os.path.join(OUT, "lu.npz"), **lu)

    # ---- residual tables (test_acceptance.py:118-154)
    res = {}
    spec = MatrixSpec("parawilk", 256, depth=4, block=15, alpha=0.5, randomize=True, seed=42)
    rows = sweep_splits(spec, range(3, 10), lu_block=64)
    res["parawilk256_splits"] = np.array([r.splits if r.splits is not None else 0 for r in rows])
    res["parawilk256_resid"] = np.array([r.scaled_residual for r in rows])
    for n in (256, 512, 1024):
        u = hpl_uniform(n, 99)
        rhs = u @ np.ones(n)
        vals = []
        for bk in (GemmBackend.native(), GemmBackend.int8(6), GemmBackend.int8(7)):
            vals.append(solve_system(u, rhs, 64, bk)[1].scaled_residual)
        res[f"uniform{n}_resid"] = np.array(vals)  # fp64, k=6, k=7
    np.savez_compressed(os.path.join(OUT, "residual.npz"), **res)

    # ---- generators (matgen.py:133-171)
    gen = {}
    gen["pw40"] = parawilk_randomized(ParaWilkParams(40, 3, 7, 0.5, randomize=True, seed=9))
    gen["pw5_det"] = parawilk(ParaWilkParams(5, 4, 2, 1.0))
    gen["uni64"] = hpl_uniform(64, 99)
    big = hpl_uniform(2048, 7)
    pos = np.random.default_rng(5).integers(0, 2048 * 2048, size=500)
    gen["uni2048_seed7_pos"] = pos
    gen["uni2048_seed7_val"] = big.ravel()[pos]
    gen["pw256_seed42"] = parawilk_randomized(p)
    np.savez_compressed(os.path.join(OUT, "matgen.npz"), **gen)

    print("golden fixtures written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main()
