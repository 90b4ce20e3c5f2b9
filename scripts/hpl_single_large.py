"""One large HPL solve on one B200, in place (no second copy of A):
generate A on the device (hpl_uniform or randomized ParaWilk), b = A @ 1,
factor + solve (timed with CUDA events), regenerate A into the same buffer
and verify the scaled residual.  For configs[3]-sized matrices on a single
GPU (N = 131072: 137 GB of the 180 GB HBM).

usage: python scripts/hpl_single_large.py N NB K {uniform|parawilk}   (K = 0: native FP64)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2509_23565_b200 as oz
from paper_2509_23565_b200 import _dev, _lib
from paper_2509_23565_b200.matgen import generate_device
from paper_2509_23565_b200.solve import _report, _solve_device, factor_device, ipiv_to_perm


def main():
    n, nb, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    kind_name = sys.argv[4] if len(sys.argv) > 4 else "uniform"
    kind, seed = (0, 99) if kind_name == "uniform" else (2, 42)
    gen = dict(seed=seed, depth=4, block=15, alpha=0.5, layout="F")
    a = generate_device(kind, n, **gen)
    b = torch.empty((n,), dtype=torch.float64, device="cuda")
    _lib.call("oz_row_sums", a.data_ptr(), n, 1, n, b.data_ptr(), _dev.stream())
    bk = oz.GemmBackend.int8(k) if k else oz.GemmBackend.native()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ipiv, stats, info, _ws = factor_device(a, nb, bk)
    perm = ipiv_to_perm(ipiv.cpu().numpy())
    x, _ = _solve_device(a, torch.from_numpy(perm).cuda(), b)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    del _ws
    generate_device(kind, n, out=a, **{kk: v for kk, v in gen.items() if kk != "layout"})
    norms = torch.zeros((4,), dtype=torch.float64, device="cuda")
    _lib.call("oz_residual_norms", a.data_ptr(), n, 1, n, x.data_ptr(), b.data_ptr(),
              norms.data_ptr(), _dev.stream())
    raw, na, nx, nbv = (float(v) for v in norms.cpu().numpy())
    rep = _report(raw, na, nx, nbv, n)
    print(json.dumps({"n": n, "nb": nb, "k": k if k else "fp64", "matrix": kind_name,
                      "seconds": t, "tflops_fp64_equiv": 2.0 * n**3 / 3.0 / t / 1e12,
                      "scaled_residual": rep.scaled_residual, "passed": rep.passed,
                      "info": int(info.item())}), flush=True)


if __name__ == "__main__":
    main()
