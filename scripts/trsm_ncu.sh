#!/bin/bash
# ncu --set full of the narrow trsm kernel at jb = ncols = 512 (panel recursion shape)
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_fused -s 12 -c 1 \
  -o $O/${T}_trsm512 python scripts/trsm_probe2.py > $O/${T}_trsm_ncu.log 2>&1
