"""Does cuBLAS DGEMM reproduce numpy/OpenBLAS bits on tiny products?
(reference test_gemm.py:91-94 asserts gemm(native, -1, a, b, 1, c) == c - a @ b
exactly.)  Prints the number of differing elements for a few shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2509_23565_b200 as oz  # noqa: E402

rng = np.random.default_rng(20240901)
for shape in ((4, 4, 4), (8, 8, 8), (16, 16, 16), (64, 64, 64), (100, 37, 61)):
    m, k, n = shape
    a, b, c = (rng.random((m, k)) - 0.5, rng.random((k, n)) - 0.5, rng.random((m, n)) - 0.5)
    ab = oz.gemm(oz.GemmBackend.native(), 1.0, a, b, 0.0)
    full = oz.gemm(oz.GemmBackend.native(), -1.0, a, b, 1.0, c)
    print(shape, "ab diff", int((ab != a @ b).sum()), "c-ab diff", int((full != c - a @ b).sum()),
          "max", float(np.abs(ab - a @ b).max()))
