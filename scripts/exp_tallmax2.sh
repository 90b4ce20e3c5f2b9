#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
bash scripts/exp_ab32k.sh $T OZ_LA_TALL_MAX=32 OZ_LA_TALL_MAX=40 OZ_LA_TALL_MAX=48
for e in OZ_LA_TALL_MAX=32 OZ_LA_TALL_MAX=40 OZ_LA_TALL_MAX=48 "OZ_LA_TALL_MAX=40 OZ_UPLOAD_STEPS=5" "OZ_UPLOAD_BLOCK=1024" "OZ_UPLOAD_BLOCK=4096"; do env $e timeout 300 python scripts/e2e_probe.py 32768 3 >> $O/${T}_e2e.log 2>&1; done
