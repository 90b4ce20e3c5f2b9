"""configs[4] (D5) per-rank work on ONE B200: rank 0 of a
1 x 8 block-cyclic grid at N = 262144, nb = 1024, k = 7 holds 262144 x 32768
(68.7 GB).  Times, with CUDA events on the launching stream:
  * the tall panel oz_lu_panel (m x 1024) at S = 16..148 CTAs, for m = 262144
    (step 0) and smaller m (later steps);
  * the rank's laswp of 1024 interchanges over its trailing columns;
  * trsm + split of U12 (1024 x nt) and L21;
  * the Schur update m x nt x 1024 through the fused emulated GEMM.
Usage: python scripts/d5_rank_probe.py [n] [Q] [out.jsonl]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2509_23565_b200 as oz  # noqa: E402
from paper_2509_23565_b200 import hpl  # noqa: E402
from paper_2509_23565_b200.matgen import GEN_UNIFORM  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/d5_rank_probe.jsonl"
nb, k = 1024, 7
torch.cuda.set_device(0)
ops = hpl.DeviceOps(n, nb, Q, 0, oz.GemmBackend.int8(k))
ops.generate(GEN_UNIFORM, 99)
ops.begin()
ncl = ops.ncl
fh = open(out, "w")


def emit(d):
    print(json.dumps(d), flush=True)
    fh.write(json.dumps(d) + "\n")


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


emit({"n": n, "Q": Q, "nb": nb, "k": k, "local_cols": ncl,
      "slab_gb": ops.slab.numel() * 8 / 1e9})
# panel timing at several heights: the panel occupies local columns [0, nb)
# with its diagonal at global row j (rows j..n of the slab)
backup = ops.slab[:nb].clone()
for j in (0, n // 2, n - 8 * nb):
    m = n - j
    for S in (16, 22, 32, 48, 74, 0):
        def run():
            ops.slab[:nb].copy_(backup)
            ops.panel(0, j, nb, 0, S)
        t_copy = timed(lambda: ops.slab[:nb].copy_(backup))
        t = timed(run) - t_copy
        emit({"what": "panel", "m": m, "jb": nb, "S": S if S else ops.sms, "ms": t,
              "ms_per_64_cols": t * 64 / nb, "info": int(ops.info.item())})
ops.slab[:nb].copy_(backup)
ops.info.zero_()
# one full step of this rank at j = 0 (rank 0 owns panel 0 at local columns 0..nb)
j, jb = 0, nb
ops.panel(0, j, jb, 0, 0)
torch.cuda.synchronize()
lstart, nt = nb, ncl - nb
emit({"what": "laswp", "cols": nt, "rows": n,
      "ms": timed(lambda: ops.laswp(((nb, ncl), (ncl, ncl)), j, jb, 0))})
emit({"what": "trsm+split", "cols": nt, "m": n - jb,
      "ms": timed(lambda: ops.trsm_split(j, jb, lstart, nt, 0))})
ops.slab[:nb].copy_(backup)          # (values only matter for timing from here on)
t = timed(lambda: ops.schur_cols(j, jb, lstart, nt, 0, nt, 0))
ops_int8 = 2.0 * 28 * (n - jb) * nt * jb
emit({"what": "schur_emulated", "m": n - jb, "n": nt, "K": jb, "ms": t,
      "int8_tops": ops_int8 / t / 1e9, "tflops_fp64_equiv": 2.0 * (n - jb) * nt * jb / t / 1e9})
t = timed(lambda: ops.schur_cols(j, jb, lstart, nt, 0, nt, 0, 22))
emit({"what": "schur_emulated_126sms", "m": n - jb, "n": nt, "K": jb, "ms": t,
      "int8_tops": ops_int8 / t / 1e9})
fh.close()
