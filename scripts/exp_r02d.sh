#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 600 python scripts/panel_probe.py 2048,4096,8192,16384,30720 16,32,74,148 1024 $O/r02d_panel_probe.jsonl > $O/r02d_panel_probe.log 2>&1
for g in 2 4 6 8 12; do
  echo "GROUP_M=$g" >> $O/r02d_groupm.log
  OZ_GEMM_GROUPM=$g timeout 200 python scripts/probe.py kern 16384 16384 16384 7 >> $O/r02d_groupm.log 2>&1
  OZ_GEMM_GROUPM=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:emu_gemm_pair -s 1 -c 1 --csv python scripts/probe.py gemm1 16384 16384 16384 7 2>&1 | grep emu_gemm >> $O/r02d_groupm.log
done
