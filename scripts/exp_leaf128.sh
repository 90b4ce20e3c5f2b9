#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
for e in OZ_TRSM_LEAF128=0 OZ_TRSM_LEAF128=1; do echo "== $e" >> $O/${T}_trsm_wide.log; env $e timeout 300 python scripts/trsm_wide_probe.py >> $O/${T}_trsm_wide.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_baseline_configs.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
bash scripts/exp_ab32k.sh $T OZ_TRSM_LEAF128=0 OZ_TRSM_LEAF128=1
