"""Standalone panel timing (oz_lu_panel) over heights m and SM caps S, with the
per-kind device time inside the panel (oz_prof_*): leaf window kernels, row
swaps inside the panel, trsm, in-panel DGEMM.  Tuning tool.
usage: python scripts/panel_probe.py [m,m,...] [S,S,...] [jb] [out.jsonl]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_23565_b200 import _dev, _lib  # noqa: E402

ms = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048,4096,8192,16384,30720").split(",")]
Ss = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "16,32,74,148").split(",")]
jb = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
out = sys.argv[4] if len(sys.argv) > 4 else None
KINDS = ["emu_gemm", "window", "schur_dgemm", "split", "swap", "trsm", "solve", "other",
         "compose", "panel_dgemm", "trsm_dgemm"]
torch.cuda.set_device(0)
fh = open(out, "a") if out else None
for m in ms:
    g = torch.Generator(device="cuda").manual_seed(m)
    src = (torch.rand((jb, m), dtype=torch.float64, device="cuda", generator=g) - 0.5)
    a = torch.empty_like(src)
    wsb = int(_lib.query("oz_lu_workspace_bytes", m, jb, 0, 7))
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    _lib.call("oz_lu_ws_init", ws.data_ptr(), wsb, m, jb, 0, _dev.stream())
    ipiv = torch.zeros((jb,), dtype=torch.int32, device="cuda")
    info = torch.zeros((1,), dtype=torch.int32, device="cuda")
    bits = torch.zeros((2,), dtype=torch.int64, device="cuda")
    ref_piv = None
    for S in Ss:
        def run():
            a.copy_(src)
            _lib.call("oz_lu_panel", a.data_ptr(), m, m, jb, 0, ipiv.data_ptr(), info.data_ptr(),
                      bits.data_ptr(), ws.data_ptr(), wsb, m, jb, 0, S, _dev.stream())
        run()
        torch.cuda.synchronize()
        if ref_piv is None:
            ref_piv = ipiv.clone()
        same = bool(torch.equal(ref_piv, ipiv))
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        reps = 3
        e0.record()
        for _ in range(reps):
            a.copy_(src)
        e1.record()
        _lib.call("oz_prof_enable", 1)
        for _ in range(reps):
            run()
        e2.record()
        torch.cuda.synchronize()
        prof = np.zeros(36)
        _lib.call("oz_prof_summary", prof.ctypes.data)
        _lib.call("oz_prof_enable", 0)
        t = (e1.elapsed_time(e2) - e0.elapsed_time(e1)) / reps
        kinds = {KINDS[i]: {"ms": round(prof[3 * i] / reps, 3),
                            "launches": int(prof[3 * i + 1] / reps)}
                 for i in range(len(KINDS)) if prof[3 * i + 1] > 0}
        dbg = np.zeros(8, dtype=np.uint64)
        _lib.call("oz_panel_debug_counters", dbg.ctypes.data)
        phases = None
        if dbg[7] > 0:  # OZ_PANEL_TIMING=1 with the register leaf: cycles per column step
            names = ["argmax", "reduce", "push", "deferred", "wait", "tail", "owner_push"]
            phases = {nm: round(float(dbg[i]) / float(dbg[7]), 1) for i, nm in enumerate(names)}
        elif dbg[:6].sum() > 0:  # shared-memory leaf: cycles summed over CTAs and columns
            names = ["publish", "wait", "reduce", "urow", "deferred", "update"]
            phases = {nm + "_Mcyc_all_ctas": round(float(dbg[i]) / reps / 1e6, 2)
                      for i, nm in enumerate(names)}
        rec = {"m": m, "jb": jb, "S": S, "ms": round(t, 3), "us_per_col": round(t * 1e3 / jb, 2),
               "leaf_cycles_per_step": phases,
               "pivots_same_as_first_S": same, "info": int(info.item()), "kinds": kinds}
        print(json.dumps(rec), flush=True)
        if fh:
            fh.write(json.dumps(rec) + "\n")
    del src, a, ws
    torch.cuda.empty_cache()
