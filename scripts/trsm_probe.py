"""Time oz_trsm_lunit (L11 1024 x 1024 unit lower, ncols right-hand sides).
usage: python scripts/trsm_probe.py NCOLS [JB]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_23565_b200 import _dev, _lib
nc = int(sys.argv[1]); jb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ld = 32768
torch.manual_seed(0)
L = torch.rand((jb, ld), dtype=torch.float64, device="cuda") - 0.5      # column-major jb cols, ld rows
B0 = torch.rand((nc, ld), dtype=torch.float64, device="cuda")
B = B0.clone()
def run():
    _lib.call("oz_trsm_lunit", L.data_ptr(), ld, jb, B.data_ptr(), ld, nc, _dev.stream())
for _ in range(3): B.copy_(B0); run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    B.copy_(B0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"trsm jb={jb} ncols={nc} {'legacy' if os.environ.get('OZ_TRSM_LEGACY') else 'fused'}: "
      f"{ts[len(ts)//2]*1e3:.1f} us  ({jb*jb*nc/ (ts[len(ts)//2]/1e3) / 1e12:.2f} TFLOP/s)")
