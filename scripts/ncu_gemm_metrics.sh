set -x
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__d_sectors.sum"
for cfg in "16384 16384 16384 7" "16384 16384 16384 3" "14336 14336 512 7"; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:emu_gemm -s 1 -c 1 python scripts/probe.py gemm1 $cfg 2>&1 | grep -v "^==PROF==" | tail -25
done
