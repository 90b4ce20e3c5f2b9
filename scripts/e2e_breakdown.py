"""Time the pieces of solve_system on pinned host buffers (n = argv[1])."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_23565_b200 as oz
from paper_2509_23565_b200 import solve as S, _dev
from paper_2509_23565_b200.matgen import generate_device
n, nb = int(sys.argv[1]), 1024
a0 = generate_device(0, n, seed=99)
a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True); a_host.copy_(a0)
b_host = torch.empty((n,), dtype=torch.float64, pin_memory=True); b_host.copy_(a0.sum(1))
del a0; torch.cuda.synchronize()
bk = oz.GemmBackend.int8(7)
for rep in range(2):
    T = [time.perf_counter()]
    def mark(): torch.cuda.synchronize(); T.append(time.perf_counter())
    ad, host = S._as_square_device(a_host); mark()
    bd = S._vector_device(b_host, n, "rhs"); mark()
    ok = bool(torch.isfinite(ad).all().item()); mark()
    work = S._col_major_copy(ad); mark()
    ipiv, stats, info, _ws = S.factor_device(work, nb, bk); mark()
    perm, growth = S._finish_factor(ipiv, stats, info); mark()
    dperm = torch.from_numpy(perm).to("cuda", non_blocking=True)
    x, flag = S._solve_device(work, dperm, bd); int(flag[0].item()); mark()
    c = oz.FlopCounter(); S._count_flops(c, n, nb, bk); mark()
    raw = S._norms(ad, x, bd); mark()
    xh = x.cpu().numpy(); mark()
    names = ["upload", "rhs", "isfinite", "colmajor", "factor", "finish", "solve", "flops", "norms", "x D2H"]
    print(" ".join(f"{k}={1e3*(T[i+1]-T[i]):.1f}" for i, k in enumerate(names)), f"total={1e3*(T[-1]-T[0]):.1f} ms")
    del ad, work, x
