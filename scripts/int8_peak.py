"""Measured dense INT8 tensor-core peak on this B200.

Three figures, each burst (best single launch of 10) and sustained (back to
back for ~4 s, total ops / total event time), with nvidia-smi clocks sampled
during the sustained runs:
  * cublaslt_int8: torch._int_mm (cuBLASLt s8 x s8 -> s32) at 8192^3 and 16384^3;
  * ours_mma_only: the emulated-GEMM kernel on the D3 shape (16384^3, k = 7,
    28 slice pairs) with OZ_GEMM_EXPERIMENT=2 (TMA + tcgen05.mma only, the FP64
    recombine and the C write skipped) - the kernel's own tensor ceiling;
  * ours_full: the same launch with the fused FP64 epilogue (split excluded).
Writes profiles/<tag>_int8_peak.json (tag = argv[1], default r02).
"""
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + "/scripts")

import numpy as np  # noqa: E402
import torch  # noqa: E402


class Clocks:
    def __enter__(self):
        self.lines = []
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,"
                                   "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits",
                                   "-lms", "200", "-i", "0"], stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=lambda: [self.lines.append(x) for x in self.p.stdout],
                                  daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()

    def summary(self):
        sm = sorted(float(x.split(",")[0]) for x in self.lines if x.strip())
        pw = [float(x.split(",")[1]) for x in self.lines if x.strip()]
        return {"sm_mhz_median": sm[len(sm) // 2] if sm else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm)}


def measure(fn, ops, seconds=4.0):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    with Clocks() as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        it = 0
        while time.perf_counter() - t0 < seconds:
            for _ in range(4):
                fn()
            it += 4
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / 1e3 / it
    return {"burst_tops": ops / best / 1e12, "sustained_tops": ops / sus / 1e12,
            "burst_ms": best * 1e3, "sustained_ms": sus * 1e3, "iters": it,
            "clocks_sustained": clk.summary()}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    torch.cuda.set_device(0)
    res = {"gpu": torch.cuda.get_device_name(0), "how": __doc__.strip().splitlines()[0]}
    for n in (8192, 16384):
        a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
        try:
            res[f"cublaslt_int8_{n}"] = measure(lambda: torch._int_mm(a, b), 2.0 * n**3)
        except RuntimeError as e:  # pragma: no cover
            res[f"cublaslt_int8_{n}"] = {"error": str(e)[:200]}
        print(n, res[f"cublaslt_int8_{n}"], flush=True)
        del a, b
        torch.cuda.empty_cache()

    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200 import _dev, _lib
    from paper_2509_23565_b200.gemm import pair_table
    from paper_2509_23565_b200.matgen import generate_device
    n, k = 16384, 7
    a = generate_device(0, n, seed=2, layout="F")
    b = generate_device(0, n, seed=3, layout="F")
    sa = _dev.split_device(a, k, 7, 0, 0)
    sb = _dev.split_device(b, k, 7, 1, 0)
    del a, b
    bk = oz.GemmBackend.int8(k)
    pa, pb, sh = pair_table(bk)
    out = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    ops = 2.0 * len(pa) * n**3

    def launch():
        _lib.call("oz_gemm_emu", n, n, n, sa.slices.data_ptr(), sa.ld, sa.nvec * sa.ld, k,
                  sa.exps.data_ptr(), sb.slices.data_ptr(), sb.ld, sb.nvec * sb.ld, k,
                  sb.exps.data_ptr(), len(pa), pa.ctypes.data, pb.ctypes.data, sh.ctypes.data,
                  7, 1.0, 0.0, out.data_ptr(), n, 0, None, _dev.stream())
    os.environ["OZ_GEMM_EXPERIMENT"] = "2"
    res["ours_mma_only_d3_k7"] = measure(launch, ops)
    print("mma only", res["ours_mma_only_d3_k7"], flush=True)
    os.environ["OZ_GEMM_EXPERIMENT"] = "0"
    res["ours_full_d3_k7"] = measure(launch, ops)
    print("full", res["ours_full_d3_k7"], flush=True)
    best = max(v.get("sustained_tops", 0) for key, v in res.items()
               if isinstance(v, dict) and key != "ours_full_d3_k7")
    best_b = max(v.get("burst_tops", 0) for key, v in res.items()
                 if isinstance(v, dict) and key != "ours_full_d3_k7")
    res["int8_tops_sustained"] = best
    res["int8_tops_burst"] = best_b
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for d in ("profiles", "gpurun_out"):
        with open(os.path.join(ROOT, d, f"{tag}_int8_peak.json"), "w") as f:
            json.dump(res, f, indent=1)
    print(json.dumps({"int8_tops_sustained": best, "int8_tops_burst": best_b}))


if __name__ == "__main__":
    main()
