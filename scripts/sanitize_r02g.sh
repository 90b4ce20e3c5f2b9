#!/bin/bash
# compute-sanitizer over this session's kernels: the LL-record grid leaves
# (incl. the tall 1024-row variant), the narrow trsm (cp.async diagonal
# blocks), the wide-trsm leaf (cp.async tiles).
TAG=${1:-r02g}; O=gpurun_out; mkdir -p $O

LU="tests/test_gpu_lu.py::test_unblocked_lu_bit_exact tests/test_gpu_lu.py::test_blocked_lu_close"
run() { local name=$1; shift; timeout 1500 "$@" > $O/${TAG}_${name}.log 2>&1; echo "rc=$?" >> $O/${TAG}_${name}.log; }
run memcheck_grid compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_panel_leaf.py -q -p no:cacheprovider -k "tall or 12000 or 40000"
OZ_PANEL_LEAF=0 run memcheck_lu_trsm compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $LU -q -p no:cacheprovider
run racecheck_leaf compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_panel_leaf.py -q -p no:cacheprovider
run racecheck_lu compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest $LU -q -p no:cacheprovider
run synccheck compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_panel_leaf.py $LU -q -p no:cacheprovider
OZ_PANEL_LEAF=0 run initcheck_lu compute-sanitizer --tool initcheck --print-limit 20 python -m pytest $LU -q -p no:cacheprovider
