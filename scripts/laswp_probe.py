"""oz_laswp timing at LU shapes: n x ncols column-major, the panel's pivots
among its rows (k1 .. n): the last step (pivots within the last 1024 rows,
every earlier column) and an early step (pivots anywhere below)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_23565_b200 import _dev, _lib  # noqa: E402

n, nb = 32768, 1024
a = torch.rand((n, n), dtype=torch.float64, device="cuda")   # column-major view: a[c] = column c
wsb = int(_lib.query("oz_lu_workspace_bytes", n, nb, 0, 7))
ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
_lib.call("oz_lu_ws_init", ws.data_ptr(), wsb, n, nb, 0, _dev.stream())
rng = np.random.default_rng(0)
for name, k1, cols in (("last step", n - nb, n - nb), ("step 0 L+rest", 0, n - nb)):
    t = np.arange(nb)
    piv = (k1 + t + (rng.random(nb) * (n - k1 - t)).astype(np.int64)).astype(np.int32)
    ip = torch.from_numpy(piv).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        e0.record()
        _lib.call("oz_laswp", a.data_ptr(), n, 0, cols, 0, 0, k1, ip.data_ptr(), nb,
                  ws.data_ptr(), wsb, n, nb, 0, _dev.stream())
        e1.record()
        torch.cuda.synchronize()
    print(f"{name}: {cols} columns, pivots in rows {k1}..{n}: {e0.elapsed_time(e1):.3f} ms", flush=True)
