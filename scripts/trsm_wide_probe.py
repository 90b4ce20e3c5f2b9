"""Wide trsm (oz_trsm_lunit) at the LU's rest shape: L11 1024 x 1024 unit lower,
B 1024 x ncols (ncols = 30720, 16384).  Run under ncu for per-kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_23565_b200 import _dev, _lib  # noqa: E402

jb = 1024
for nc in (30720, 16384):
    g = torch.Generator(device="cuda").manual_seed(nc)
    L = torch.rand((jb, jb), dtype=torch.float64, device="cuda", generator=g) - 0.5
    L = torch.tril(L, -1) / jb + torch.eye(jb, dtype=torch.float64, device="cuda")
    L = L.t().contiguous().t()
    B0 = torch.rand((nc, jb), dtype=torch.float64, device="cuda", generator=g)
    B = B0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        B.copy_(B0)
        e0.record()
        _lib.call("oz_trsm_lunit", L.data_ptr(), jb, jb, B.data_ptr(), jb, nc, _dev.stream())
        e1.record()
        torch.cuda.synchronize()
        print(f"jb={jb} ncols={nc}: {e0.elapsed_time(e1) * 1e3:.1f} us", flush=True)
    X = B.t()
    print("residual", float((L @ X - B0.t()).abs().max()))
