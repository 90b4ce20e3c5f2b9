"""e2e solve_system on pinned host A (n = argv[1], nb = 1024, k = 7): wall time
per call, as bench.py's e2e leg.  Env knobs of the upload phase are read by
the library (OZ_UPLOAD_STEPS, OZ_UPLOAD_SMS, OZ_UPLOAD_BLOCK)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_23565_b200 as oz  # noqa: E402
from paper_2509_23565_b200.matgen import generate_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a0 = generate_device(0, n, seed=99)
a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
a_host.copy_(a0)
b_host = torch.empty((n,), dtype=torch.float64, pin_memory=True)
b_host.copy_(a0.sum(1))
del a0
torch.cuda.synchronize()
bk = oz.GemmBackend.int8(7)
oz.solve_system(a_host, b_host, 1024, bk)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = oz.solve_system(a_host, b_host, 1024, bk)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("OZ_"))
print(f"{env or 'default'}: e2e " + " ".join(f"{t:.1f}" for t in ts) + f" ms, residual {rep.scaled_residual:.3g}", flush=True)
