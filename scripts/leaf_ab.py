"""A/B check of the panel leaf variants: factor the same m x jb panel with
oz_lu_panel in two processes (OZ_PANEL_LEAF=1 register leaf, =0 shared-memory
leaf) and compare factors and pivots bit for bit.  Same leaf widths -> same
recursion -> identical bits expected.
usage: python scripts/leaf_ab.py m jb [S]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 4 and sys.argv[4] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2509_23565_b200 import _dev, _lib
    m, jb, S, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[5]
    g = torch.Generator(device="cuda").manual_seed(1234 + m)
    a = (torch.rand((jb, m), dtype=torch.float64, device="cuda", generator=g) - 0.5)
    wsb = int(_lib.query("oz_lu_workspace_bytes", m, jb, 0, 7))
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    _lib.call("oz_lu_ws_init", ws.data_ptr(), wsb, m, jb, 0, _dev.stream())
    ipiv = torch.zeros((jb,), dtype=torch.int32, device="cuda")
    info = torch.zeros((1,), dtype=torch.int32, device="cuda")
    bits = torch.zeros((2,), dtype=torch.int64, device="cuda")
    _lib.call("oz_lu_panel", a.data_ptr(), m, m, jb, 0, ipiv.data_ptr(), info.data_ptr(),
              bits.data_ptr(), ws.data_ptr(), wsb, m, jb, 0, S, _dev.stream())
    torch.cuda.synchronize()
    np.savez(out, a=a.cpu().numpy(), ipiv=ipiv.cpu().numpy(), info=info.cpu().numpy(),
             bits=bits.cpu().numpy())
    sys.exit(0)

m, jb = int(sys.argv[1]), int(sys.argv[2])
S = int(sys.argv[3]) if len(sys.argv) > 3 else 0
res = {}
for v in ("1", "0"):
    out = f"/tmp/leaf_ab_{v}.npz"
    env = dict(os.environ, OZ_PANEL_LEAF=v)
    subprocess.run([sys.executable, __file__, str(m), str(jb), str(S), "child", out], env=env,
                   check=True)
    import numpy as np
    res[v] = np.load(out)
import numpy as np
a1, a0 = res["1"]["a"], res["0"]["a"]
same_piv = np.array_equal(res["1"]["ipiv"], res["0"]["ipiv"])
nd = int(np.sum(a1.view(np.int64) != a0.view(np.int64)))
print(f"leaf A/B m={m} jb={jb}: pivots identical {same_piv}, differing factor entries {nd}, "
      f"max |diff| {np.max(np.abs(a1 - a0)):.3g}, growth bits equal "
      f"{np.array_equal(res['1']['bits'], res['0']['bits'])}, info {res['1']['info']} {res['0']['info']}",
      flush=True)
