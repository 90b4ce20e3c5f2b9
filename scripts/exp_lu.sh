#!/bin/bash
# GPU tests + LU timings at the bench sizes (tuning loop)
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --ignore=tests/ref_suite > $O/${T}_gputest.log 2>&1; echo rc=$? >> $O/${T}_gputest.log
for n in 8192 16384 32768; do timeout 300 python scripts/panel_breakdown.py $n 1024 7 >> $O/${T}_breakdown.log 2>&1; done
timeout 300 python scripts/panel_breakdown.py 16384 1024 3 >> $O/${T}_breakdown.log 2>&1
