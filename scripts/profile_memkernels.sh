#!/bin/bash
# HBM-bound kernels of the path (split, laswp, compose, trsm, panel): per-launch
# duration and DRAM bytes under ncu, for profiles/ (one GPU, under gpurun).
OUT=${1:-gpurun_out}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none -k regex:"exps_|slices_" -c 4 --csv \
  --log-file $OUT/split_d3.csv python scripts/probe.py gemm1 16384 16384 16384 3 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"laswp_list|compose_ipiv|trsm_unit|panel_window|exps_|slices_" \
  -c 60 --csv --log-file $OUT/lu_mem.csv python scripts/probe.py lu1 16384 1024 7 > /dev/null 2>&1
ls -la $OUT
