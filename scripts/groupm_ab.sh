#!/bin/bash
# A/B of the GEMM raster band (OZ_GEMM_GROUPM) at D3 16384^3 k=7, interleaved
# so clock/thermal drift hits both arms alike.
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
  for g in 2 4 6 8; do
    echo "GROUP_M=$g rep=$rep $(OZ_GEMM_GROUPM=$g timeout 200 python scripts/probe.py kern 16384 16384 16384 7 2>&1 | tail -1)" >> $O/r02ag_groupm.log
  done
done
