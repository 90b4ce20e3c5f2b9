"""Narrow trsm (oz_trsm_lunit) timing at the LU's shapes: L11 jb x jb unit
lower, B jb x ncols; env selects the kernel (OZ_TRSM_NARROW_CUBLAS / LEGACY)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_23565_b200 import _dev, _lib  # noqa: E402

for jb, nc in ((1024, 1024), (512, 512), (256, 256), (128, 128), (64, 64), (512, 1536)):
    g = torch.Generator(device="cuda").manual_seed(jb)
    L = torch.rand((jb, jb), dtype=torch.float64, device="cuda", generator=g) - 0.5
    L = torch.tril(L, -1) / jb + torch.eye(jb, dtype=torch.float64, device="cuda")
    L = L.t().contiguous().t()  # column-major storage
    B0 = torch.rand((nc, jb), dtype=torch.float64, device="cuda", generator=g)  # col-major jb x nc
    B = B0.clone()

    def run():
        B.copy_(B0)
        _lib.call("oz_trsm_lunit", L.data_ptr(), jb, jb, B.data_ptr(), jb, nc, _dev.stream())
    run()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(10):
        B.copy_(B0)
    e1.record()
    for _ in range(10):
        run()
    e2.record()
    torch.cuda.synchronize()
    t = (e1.elapsed_time(e2) - e0.elapsed_time(e1)) / 10
    X = B.t()  # jb x nc row-major view of the col-major result
    res = float((L @ X - B0.t()).abs().max())
    print(f"jb={jb} ncols={nc}: {t * 1e3:.1f} us  residual {res:.2e}", flush=True)
