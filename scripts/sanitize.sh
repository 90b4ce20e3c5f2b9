#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the GPU
# tests that exercise the spin-waiting kernels (grid-barrier and cluster-DSMEM
# panel leaves, sync-free trsv), the split kernels, the tcgen05 GEMM and the
# distributed step entries.  Run on a B200 box:
#   scripts/sanitize.sh [tag]  -> gpurun_out/<tag>_sanitize_<tool>.log
set -u
TAG=${1:-r02}
SEL=${SEL:-"tests/test_gpu_lu.py::test_unblocked_lu_bit_exact tests/test_gpu_lu.py::test_blocked_lu_close tests/test_gpu_lu.py::test_wilkinson_growth tests/test_gpu_lu.py::test_solve_small_and_norms tests/test_gpu_lu.py::test_parawilk256_residual_table tests/test_gpu_split_gemm.py::test_split_matches_reference_golden tests/test_gpu_split_gemm.py::test_gemm_matches_reference_golden tests/test_gpu_split_gemm.py::test_schur_calls_match_reference_golden tests/test_gpu_hpl.py::test_one_rank_matches_single_gpu_lu tests/test_gpu_hpl2d.py::test_pxq_native_passes"}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 900 compute-sanitizer --tool $tool $extra --target-processes all \
      --print-limit 200 --error-exitcode 99 \
      python -m pytest $SEL -q -p no:cacheprovider -x \
      > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
  tail -3 gpurun_out/${TAG}_sanitize_${tool}.log
done
