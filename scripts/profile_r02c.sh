#!/bin/bash
# Round-2 evidence pass (one GPU): full GPU tests, per-step LU trace at the
# headline and k-sweep sizes, per-phase breakdown, D3 16384^3 ncu capture.
TAG=${1:-r02c}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/ref_suite > $O/${TAG}_gputest.log 2>&1; echo rc=$? >> $O/${TAG}_gputest.log
for cfg in "32768 1024 7" "16384 1024 7" "16384 1024 3"; do
  OZ_LU_TRACE=1 OZ_PROBE_REPS=2 timeout 300 python scripts/probe.py lu1 $cfg >> $O/${TAG}_lu_trace.log 2>&1
  echo "=== $cfg" >> $O/${TAG}_lu_trace.log
  timeout 300 python scripts/panel_breakdown.py $cfg >> $O/${TAG}_breakdown.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:emu_gemm_pair -s 1 -c 1 \
  -o $O/${TAG}_emu_gemm_d3 python scripts/probe.py gemm1 16384 16384 16384 7 > $O/${TAG}_ncu_d3.log 2>&1
ncu -i $O/${TAG}_emu_gemm_d3.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active > $O/${TAG}_ncu_d3_metrics.csv 2>&1
