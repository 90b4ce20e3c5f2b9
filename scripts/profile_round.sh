#!/bin/bash
# Profiling evidence for profiles/ (run under gpurun, one GPU):
#  1. launch list of one LU bench step (cold-cache, serialised: compare shares)
#  2. ncu --set full of one emulated-GEMM launch inside the LU (K = nb = 1024)
#  3. ncu --set full of the standalone D3 GEMM (8192^3, k=7) for the tensor-pipe figure
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $OUT/launches.csv python bench.py --n 16384 --nb 1024 --steps 1 --warmup 1 \
  --e2e-steps 0 --skip-native --sweep-k "" > $OUT/launches_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emu_gemm_pair -s 3 -c 1 \
  -o $OUT/emu_gemm_lu python scripts/probe.py lu1 16384 1024 7 > $OUT/ncu_lu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:emu_gemm_pair -s 1 -c 1 \
  -o $OUT/emu_gemm_d3 python scripts/probe.py gemm1 8192 8192 8192 7 > $OUT/ncu_d3.log 2>&1
ls -la $OUT
