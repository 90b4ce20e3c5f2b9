"""Developer probe: time the emulated GEMM / LU on device-resident inputs."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_23565_b200 as oz
from paper_2509_23565_b200 import _lib, _dev
from paper_2509_23565_b200.gemm import emulated_into
from paper_2509_23565_b200.matgen import generate_device
from paper_2509_23565_b200.solve import factor_device, _col_major_copy


def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def gemm_probe(n, ks):
    a = generate_device(0, n, seed=2)
    b = generate_device(0, n, seed=3)
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    fl = 2.0 * n**3
    t = timeit(lambda: _lib.call("oz_dgemm", 0, 0, n, n, n, 1.0, b.data_ptr(), n, a.data_ptr(), n,
                                 0.0, out.data_ptr(), n, _dev.stream()))
    print(f"gemm n={n} native cuBLAS DGEMM: {t*1e3:.2f} ms  {fl/t/1e12:.2f} TFLOP/s", flush=True)
    for k in ks:
        bk = oz.GemmBackend.int8(k)
        np_ = k * (k + 1) // 2
        t = timeit(lambda: emulated_into(bk, a, b, 1.0, 0.0, out, False))
        print(f"gemm n={n} k={k} pairs={np_}: {t*1e3:.2f} ms  {fl/t/1e12:.2f} TFLOP/s-eq  "
              f"int8 {np_*fl/t/1e15:.3f} POPS", flush=True)


def lu_probe(n, nb, backends):
    for name, bk in backends:
        a = generate_device(0, n, seed=99, layout="F")
        work = a.clone()
        def run():
            work.copy_(a)
            return factor_device(work, nb, bk)
        run(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = run(); e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 1e3
        print(f"lu n={n} nb={nb} {name}: {t*1e3:.1f} ms  {2*n**3/3/t/1e12:.2f} TFLOP/s-eq "
              f"info={int(r[2].item())}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what in ("gemm1", "lu1", "kern", "e2e", "starts"):
        pass
    elif what == "gemm":
        gemm_probe(int(sys.argv[2]), [int(k) for k in sys.argv[3].split(",")])
    else:
        n, nb = int(sys.argv[2]), int(sys.argv[3])
        lu_probe(n, nb, [("fp64", oz.GemmBackend.native()), ("k7", oz.GemmBackend.int8(7)),
                         ("k6", oz.GemmBackend.int8(6))])


def gemm_once(m, n, K, k, reps=2):
    """One emulated GEMM call (column-major C) for ncu capture."""
    a = torch.rand((m, K), dtype=torch.float64, device="cuda") - 0.5
    b = torch.rand((K, n), dtype=torch.float64, device="cuda") - 0.5
    out = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    bk = oz.GemmBackend.int8(k)
    for _ in range(reps):
        emulated_into(bk, a, b, -1.0, 1.0, out, True)
    torch.cuda.synchronize()


if __name__ == "__main__" and sys.argv[1] == "gemm1":
    gemm_once(*[int(v) for v in sys.argv[2:6]])


if __name__ == "__main__" and sys.argv[1] == "lu1":
    n, nb, k = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    bk = oz.GemmBackend.int8(k) if k > 0 else oz.GemmBackend.native()
    for _ in range(int(os.environ.get("OZ_PROBE_REPS", "1"))):  # >1: trace a warm run
        a = generate_device(0, n, seed=99, layout="F")
        r = factor_device(a, nb, bk)
        torch.cuda.synchronize()
        del a
    print("lu1 done info", int(r[2].item()))


if __name__ == "__main__" and sys.argv[1] == "kern":
    # kern m n K k[,k2..] : device-resident emulated GEMM, per-phase event times
    m, n, K = (int(v) for v in sys.argv[2:5])
    ks = [int(v) for v in sys.argv[5].split(",")]
    a = torch.rand((m, K), dtype=torch.float64, device="cuda") - 0.5
    b = torch.rand((K, n), dtype=torch.float64, device="cuda") - 0.5
    out = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    for k in ks:
        bk = oz.GemmBackend.int8(k)
        npairs = k * (k + 1) // 2
        for _ in range(2):
            emulated_into(bk, a, b, -1.0, 1.0, out, True)
        torch.cuda.synchronize()
        reps = 5
        _lib.call("oz_prof_enable", 1)
        for _ in range(reps):
            emulated_into(bk, a, b, -1.0, 1.0, out, True)
        torch.cuda.synchronize()
        prof = np.zeros(36)
        _lib.call("oz_prof_summary", prof.ctypes.data)
        _lib.call("oz_prof_enable", 0)
        g_ms, s_ms = prof[0] / reps, prof[9] / reps
        ops = 2.0 * npairs * m * n * K
        print(f"kern m={m} n={n} K={K} k={k}: gemm {g_ms:.3f} ms {ops/g_ms/1e9:.1f} TOPS int8 "
              f"({2.0*m*n*K/g_ms/1e9:.1f} TFLOP/s-eq), split {s_ms:.3f} ms", flush=True)


if __name__ == "__main__" and sys.argv[1] == "e2e":
    # e2e n nb: solve_system on pinned host buffers, with the H2D copy timed alone
    n, nb = int(sys.argv[2]), int(sys.argv[3])
    a0 = generate_device(0, n, seed=99)
    a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    a_host.copy_(a0)
    b_host = torch.empty((n,), dtype=torch.float64, pin_memory=True)
    b_host.copy_(a0.sum(1))
    del a0
    torch.cuda.synchronize()
    for rep in range(3):
        t0 = time.perf_counter()
        d = a_host.to("cuda", non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        del d
        xh, r = oz.solve_system(a_host, b_host, nb, oz.GemmBackend.int8(7))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"e2e n={n}: H2D alone {1e3*(t1-t0):.1f} ms ({8*n*n/(t1-t0)/1e9:.1f} GB/s), "
              f"solve_system {1e3*(t2-t1):.1f} ms (factor+solve {1e3*r.seconds:.1f} ms), "
              f"resid {r.scaled_residual:.3g}", flush=True)


if __name__ == "__main__" and sys.argv[1] == "starts":
    # OZ_GEMM_STARTS=1: CTA start/end spread of each emulated-GEMM launch in one LU
    n, nb, k = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    a = generate_device(0, n, seed=99, layout="F")
    r = factor_device(a, nb, oz.GemmBackend.int8(k))
    torch.cuda.synchronize()
    from paper_2509_23565_b200 import _lib
    _lib.call("oz_gemm_starts_dump")
