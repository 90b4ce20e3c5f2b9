#!/bin/bash
# Round-2 ncu evidence (one GPU): per-launch duration + DRAM bytes of the
# HBM-bound kernels inside an n = 16384 LU (split, row swaps, leaves, flat
# passes) and of the D3 split; one --set full capture of the register grid leaf.
O=gpurun_out; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none -k regex:"laswp|compose_ipiv|panel_leaf|panel_window|exps_|slices_|max_abs|copy_flat|trsm_fused" \
  -c 400 --csv --log-file $O/r02ax_lu_mem.csv python scripts/probe.py lu1 16384 1024 7 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"exps_|slices_" -c 4 --csv \
  --log-file $O/r02ax_split_d3.csv python scripts/probe.py gemm1 16384 16384 16384 7 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"panel_leaf_kernel<64, 1, 256, 1>|panel_leaf_kernel<64,1,256,1>" -s 3 -c 1 \
  -o $O/r02ax_leaf_grid python scripts/panel_probe.py 16384 74 1024 > /dev/null 2>&1
ls -la $O | grep r02ax
