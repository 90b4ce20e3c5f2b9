"""Host utilities re-exported for drop-in completeness (no GPU needed):
the exact big-integer product behind gemm_error_profile (exact.py, the
reference's ozemu.oracle) and the test-matrix helpers of matgen.py:98-251."""

from fractions import Fraction

import numpy as np
import pytest

import paper_2509_23565_b200 as oz
from paper_2509_23565_b200 import exact


def test_exact_product_matches_fractions(rng):
    a = rng.random((4, 3)) - 0.5
    b = rng.random((3, 5)) - 0.5
    got = exact.exact_gemm_fractions(a, b)
    for i in range(4):
        for j in range(5):
            assert got[i][j] == sum(Fraction(float(a[i, t])) * Fraction(float(b[t, j]))
                                    for t in range(3))
    ints, s = exact.exact_gemm_scaled(a, b)
    assert Fraction(ints[1][2]) * Fraction(2) ** s == got[1][2]


def test_exact_product_edge_cases(rng):
    ai = rng.integers(-8, 9, size=(6, 6)).astype(float)
    bi = rng.integers(-8, 9, size=(6, 6)).astype(float)
    assert np.array_equal(exact.exact_gemm_float(ai, bi), ai @ bi)
    assert exact.rel_error_vs_exact(ai @ bi, ai, bi).max() == 0.0
    wide = np.array([[2.0**300, 2.0**-300], [1.0, 5e-324]])
    assert exact.abs_error_vs_exact(wide, wide, np.eye(2)).max() == 0.0
    z = np.zeros((2, 2))
    assert exact.rel_error_vs_exact(z, z, z).max() == 0.0
    assert np.isinf(exact.rel_error_vs_exact(np.array([[1e-20]]), np.array([[1.0, -1.0]]),
                                             np.array([[1.0], [1.0]]))[0, 0])
    with pytest.raises(oz.ShapeMismatchError):
        exact.exact_gemm_scaled(np.ones((2, 3)), np.ones((2, 3)))
    with pytest.raises(oz.ShapeMismatchError):
        exact.abs_error_vs_exact(np.ones((3, 3)), np.ones((2, 2)), np.ones((2, 2)))


def test_exact_vs_oracle_restatement(rng):
    """The package's exact product agrees with the test oracle's FP64 product
    wherever FP64 is exact (small integers), and is the correctly rounded value
    otherwise (never further from the exact value than numpy's)."""
    a = rng.random((5, 7)) - 0.5
    b = rng.random((7, 4)) - 0.5
    fl = exact.exact_gemm_float(a, b)
    err_np = exact.abs_error_vs_exact(a @ b, a, b)
    err_fl = exact.abs_error_vs_exact(fl, a, b)
    assert (err_fl <= err_np).all()


def test_generalized_fibonacci_and_turing_inverse():
    assert oz.generalized_fibonacci(2, 8) == [1, 1, 2, 3, 5, 8, 13, 21]
    assert oz.generalized_fibonacci(1, 4) == [1, 1, 1, 1]
    for d in range(1, 6):
        assert oz.generalized_fibonacci(d, d + 1)[:d] == [1] + [2**i for i in range(d - 1)]
    with pytest.raises(oz.InvalidParamsError):
        oz.generalized_fibonacci(0, 3)
    n, d = 8, 3
    inv = oz.turing_inverse(n, d)
    # exact: turing(n, d) @ inv == I with Python integers
    t = np.zeros((n, n), dtype=object)
    for i in range(n):
        t[i, i] = 1
        for j in range(max(0, i - d), i):
            t[i, j] = -1
    assert (t.dot(inv) == np.eye(n, dtype=int)).all()
    assert list(inv[:, 0]) == oz.generalized_fibonacci(d, n)
    with pytest.raises(oz.InvalidDimError):
        oz.turing_inverse(4, 4)


def test_scaling_and_permutations():
    a = np.arange(12.0).reshape(3, 4)
    assert np.array_equal(oz.apply_scaling(a), a)
    out = oz.apply_scaling(a, left=oz.DiagonalScale(np.array([2.0, -0.5, 2.0**-60])),
                           right=oz.Permutation(np.array([3, 2, 1, 0])))
    assert np.array_equal(out, (a * np.array([2.0, -0.5, 2.0**-60])[:, None])[:, ::-1])
    p = oz.Permutation(np.array([2, 0, 1]))
    assert np.array_equal(oz.apply_scaling(np.eye(3), left=p, right=p), np.eye(3))
    assert oz.nnz_pattern(np.array([[0.0, 1.0], [2.0, 0.0]])).tolist() == [[0, 1], [1, 0]]
    for bad in ([3.0], [0.0], [np.inf]):
        with pytest.raises(oz.NonPowerOfTwoScaleError):
            oz.DiagonalScale(np.array(bad))
    for bad in ([0, 0, 1], [0.5, 1.0], [1, 2]):
        with pytest.raises(oz.InvalidPermutationError):
            oz.Permutation(np.array(bad))
    with pytest.raises(oz.ShapeMismatchError):
        oz.apply_scaling(np.ones((2, 3)), left=oz.DiagonalScale(np.ones(3)))
    with pytest.raises(oz.ShapeMismatchError):
        oz.apply_scaling(np.ones((2, 3)), right=oz.Permutation(np.array([1, 0])))
    with pytest.raises(oz.InvalidParamsError):
        oz.apply_scaling(np.ones((2, 2)), left="x")
