#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lu.py -q -x -p no:cacheprovider -k "upload or host or overlapped" > $O/${T}_tests.log 2>&1
bash scripts/exp_ab32k.sh $T OZ_LA_TALL_MAX=0 OZ_LA_TALL_MAX=32
for e in OZ_LA_TALL_MAX=0 OZ_LA_TALL_MAX=32 "OZ_LA_TALL_MAX=32 OZ_UPLOAD_STEPS=4" "OZ_LA_TALL_MAX=32 OZ_UPLOAD_STEPS=5"; do env $e timeout 300 python scripts/e2e_probe.py 32768 3 >> $O/${T}_e2e.log 2>&1; done
