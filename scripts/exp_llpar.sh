#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_panel_leaf.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
for rep in 1 2; do for e in OZ_LEAF_LL_PAR=0 OZ_LEAF_LL_PAR=1; do
  echo "== $e" >> $O/${T}_probe.log
  env $e timeout 300 python scripts/panel_probe.py 12288,16384,20480 20,32,100 1024 >> $O/${T}_probe.log 2>&1
done; done
bash scripts/exp_ab32k.sh $T OZ_LEAF_LL_PAR=0 OZ_LEAF_LL_PAR=1
