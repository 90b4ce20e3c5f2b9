#!/bin/bash
# compute-sanitizer over the round-2 kernels: register panel leaves (cluster
# push exchange through cp.async.bulk + mbarrier; grid exchange through tagged
# global records), the tag-polling shared-memory grid leaf, the flat HBM passes.
TAG=${1:-r02c}
SEL="tests/test_gpu_panel_leaf.py tests/test_gpu_lu.py::test_unblocked_lu_bit_exact tests/test_gpu_lu.py::test_blocked_lu_close tests/test_gpu_lu.py::test_parawilk256_residual_table"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      python -m pytest $SEL -q -p no:cacheprovider -x > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
