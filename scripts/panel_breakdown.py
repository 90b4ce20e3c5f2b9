"""Per-phase device time of one LU (oz_prof_*), to see where the panel chain goes.
usage: python scripts/panel_breakdown.py N NB K"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_23565_b200 as oz
from paper_2509_23565_b200 import _lib
from paper_2509_23565_b200.matgen import generate_device
from paper_2509_23565_b200.solve import factor_device
n, nb, k = (int(v) for v in sys.argv[1:4])
bk = oz.GemmBackend.int8(k) if k else oz.GemmBackend.native()
a0 = generate_device(0, n, seed=99, layout="F")
a = a0.clone(); factor_device(a, nb, bk); torch.cuda.synchronize()
a.copy_(a0)
_lib.call("oz_prof_enable", 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); factor_device(a, nb, bk); e1.record(); torch.cuda.synchronize()
prof = np.zeros(36); _lib.call("oz_prof_summary", prof.ctypes.data); _lib.call("oz_prof_enable", 0)
kinds = ["emu_gemm", "panel", "schur_dgemm", "split", "laswp", "trsm", "solve", "other",
         "swap_compose", "panel_dgemm", "trsm_dgemm", "-"]
print(f"n={n} nb={nb} k={k} factor {e0.elapsed_time(e1):.2f} ms")
for i, kd in enumerate(kinds):
    if prof[3*i+1] > 0:
        print(f"  {kd:13s} {prof[3*i]:8.2f} ms  {int(prof[3*i+1]):6d} launches  {prof[3*i]/prof[3*i+1]*1e3:8.1f} us/launch")
