#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_split_gemm.py tests/test_gpu_lu.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"onepass|exps_|slices_" -c 24 --log-file $O/${T}_split.csv python scripts/panel_breakdown.py 16384 1024 7 > /dev/null 2>&1
OZ_SPLIT_ONEPASS=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"onepass|exps_|slices_" -c 24 --log-file $O/${T}_split0.csv python scripts/panel_breakdown.py 16384 1024 7 > /dev/null 2>&1
bash scripts/exp_ab32k.sh $T OZ_SPLIT_ONEPASS=0 OZ_SPLIT_ONEPASS=1
