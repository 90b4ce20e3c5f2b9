"""Device time of oz_lu_solve (both triangles) at n, on the factors of
hpl_uniform(n, 99), and its agreement with x = 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_23565_b200 as oz  # noqa: E402
from paper_2509_23565_b200 import _dev, _lib  # noqa: E402
from paper_2509_23565_b200.matgen import generate_device  # noqa: E402
from paper_2509_23565_b200.solve import _solve_device, factor_device, ipiv_to_perm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a0 = generate_device(0, n, seed=99, layout="F")
b = torch.empty((n,), dtype=torch.float64, device="cuda")
_lib.call("oz_row_sums", a0.data_ptr(), n, 1, n, b.data_ptr(), _dev.stream())
work = a0.clone()
ipiv, _s, _i, _w = factor_device(work, 1024, oz.GemmBackend.int8(7))
perm = torch.from_numpy(ipiv_to_perm(ipiv.cpu().numpy())).cuda()
x, _ = _solve_device(work, perm, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    x, _ = _solve_device(work, perm, b)
e1.record()
torch.cuda.synchronize()
print(f"n={n}: solve {e0.elapsed_time(e1) / 5:.3f} ms, max|x-1| {float((x - 1).abs().max()):.3e}")
