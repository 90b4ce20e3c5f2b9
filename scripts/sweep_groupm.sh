nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 500 > gpurun_out/clk_gm.csv &
SMI=$!
for g in 16 8 4 2; do echo "GROUP_M=$g"; OZ_GEMM_GROUPM=$g timeout 120 python scripts/probe.py kern 16384 16384 16384 7; OZ_GEMM_GROUPM=$g timeout 120 python scripts/probe.py kern 14336 14336 512 7; done
kill $SMI
