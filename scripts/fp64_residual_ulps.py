"""Why the configs[0] FP64 row differs from the reference by 14/9 (CPU only).

At FP64 accuracy the HPL residual's numerator ||Ax - b||_inf is a handful of
ulps of ||b||, so any valid change of summation order moves it by whole ulps.
This script factors ParaWilk_256(4, 15, 1/2) seed 42 with the oracle (the
reference's algorithm) and solves with b = A @ 1 summed two ways:
  A@1 (BLAS order, the reference)  -> 9 ulp  (scaled residual 0.01161)
  column-sequential order           -> 10 ulp (0.01290)
The B200 path (device GEMV for b, cuBLAS/trsm orders) lands on 14 ulp
(0.01806), i.e. the 1.556 = 14/9 ratio of the bench table; k = 8 and k = 9
give 17/13 and 11/10 for the same reason."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ozaki_oracle as orc  # noqa: E402

a = orc.parawilk_randomized(256, 4, 15, 0.5, 42)
n = a.shape[0]
lu, perm, _ = orc.lu_factor(a, 64, None)
b_blas = a @ np.ones(n)
b_seq = np.zeros(n)
for j in range(n):
    b_seq += a[:, j]
for name, b in (("A@1 (BLAS order)", b_blas), ("column-sequential", b_seq)):
    x = orc.lu_solve(lu, perm, b)
    scaled, raw, *_ = orc.residual(a, x, b)
    print(f"{name:18s} scaled residual {scaled:.6g}  ||Ax-b||_inf = {raw / np.spacing(np.abs(b).max()):.2f} ulp(||b||_inf)")
