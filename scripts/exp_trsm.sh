#!/bin/bash
# narrow trsm kernel durations (ncu launch list), standalone panels, LU A/B
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:trsm_fused \
  --log-file $O/${T}_trsm_launches.csv python scripts/trsm_probe2.py > $O/${T}_trsm_probe.log 2>&1
for e in "$@"; do
  env $e timeout 300 python scripts/panel_probe.py 2048,8192,12288 100 1024 >> $O/${T}_probe.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_panel_leaf.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
bash scripts/exp_ab32k.sh $T "$@"
for e in "$@"; do
  echo "== $e $(env $e timeout 300 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
done
