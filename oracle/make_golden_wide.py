"""Generate tests/golden/wide.npz from the REFERENCE itself (build container
only; needs /root/reference): int16 slices, slice_bits 8..10 — split.py:144
and the emulated GEMM / LU with them.  Test infrastructure, like
make_golden.py."""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from ozemu import Band, GemmBackend, Orientation, gemm, lu_factor, split_matrix

    rng = np.random.default_rng(99)
    g = {}
    # split (split.py:109-160, int16 slices for q > 7)
    a = (rng.random((11, 23)) - 0.5) * np.ldexp(1.0, rng.integers(-40, 41, size=(11, 1)))
    i = 0
    for q in (8, 9, 10):
        for k in (2, 4):
            for orient in (Orientation.ROW_SCALED, Orientation.COL_SCALED):
                st = split_matrix(a, k, q, orient)
                g[f"s{i}_meta"] = np.array([k, q, 0 if orient is Orientation.ROW_SCALED else 1])
                g[f"s{i}_slices"] = np.stack(st.slices)
                g[f"s{i}_exps"] = st.exponents
                i += 1
    g["split_a"] = a
    g["split_count"] = np.array([i])
    # emulated GEMM (gemm.py:190-271)
    A = rng.random((37, 130)) - 0.5
    B = rng.random((130, 29)) - 0.5
    C = rng.random((37, 29)) - 0.5
    i = 0
    for q, k in ((8, 2), (9, 3), (10, 3), (10, 5)):
        bk = GemmBackend.int8(k, q, truncation=Band(k + 1))
        g[f"g{i}_meta"] = np.array([k, q])
        g[f"g{i}_out"] = gemm(bk, -1.0, A, B, 1.0, C)
        i += 1
    g["gemm_a"], g["gemm_b"], g["gemm_c"] = A, B, C
    g["gemm_count"] = np.array([i])
    # LU with int16-slice Schur updates (solve.py:94-140)
    L = rng.random((96, 96)) - 0.5
    f = lu_factor(L, 16, GemmBackend.int8(3, 10))
    g["lu_a"], g["lu_lu"], g["lu_perm"] = L, f.lu, f.pivots
    g["lu_growth"] = np.array([f.growth])
    np.savez_compressed(os.path.join(OUT, "wide.npz"), **g)
    print("wrote", os.path.join(OUT, "wide.npz"))


if __name__ == "__main__":
    main()
