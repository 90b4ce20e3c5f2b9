#!/bin/bash
# memcheck / racecheck on the register panel leaves only (tuning of sanitizer evidence)
TAG=${1:-r02d}
SEL="tests/test_gpu_panel_leaf.py"
for tool in memcheck racecheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 \
      python -m pytest $SEL -q -p no:cacheprovider > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
OZ_PANEL_LEAF=0 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $SEL -q -p no:cacheprovider > gpurun_out/${TAG}_sanitize_memcheck_smemleaf.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_sanitize_memcheck_smemleaf.log
