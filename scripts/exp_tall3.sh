#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
OZ_PANEL_LEAF_TALL=3 timeout 900 python -m pytest tests/test_gpu_lu.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
OZ_PANEL_LEAF_TALL=3 timeout 300 python -c "
import numpy as np, sys
sys.path.insert(0,'tests')
from test_gpu_panel_leaf import _reference_panel, _device_panel
for m, jb, ctas in ((12000, 16, 8), (30000, 16, 20), (5000, 16, 4)):
    rng = np.random.default_rng(m)
    a = rng.integers(-4, 5, size=(m, jb)).astype(np.float64)
    want, piv, zero = _reference_panel(a)
    got, ipiv, info = _device_panel(a, ctas)
    print(m, jb, ctas, np.array_equal(ipiv, piv), np.array_equal(got, want), info == zero)
" >> $O/${T}_tests.log 2>&1
for e in OZ_PANEL_LEAF_TALL=1 OZ_PANEL_LEAF_TALL=3; do env $e timeout 300 python scripts/panel_probe.py 30720,24576 20,24,32 1024 >> $O/${T}_probe.log 2>&1; done
bash scripts/exp_ab32k.sh $T OZ_PANEL_LEAF_TALL=1 OZ_PANEL_LEAF_TALL=3
