TAG=${1:-r02b}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --ignore=tests/ref_suite > gpurun_out/${TAG}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_gputest.log
timeout 600 python -m pytest tests/ref_suite -m gpu -q -p no:cacheprovider -rs > gpurun_out/${TAG}_ref_suite.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_ref_suite.log
timeout 900 python scripts/d5_rank_probe.py 262144 8 gpurun_out/${TAG}_d5_rank_probe.jsonl > gpurun_out/${TAG}_d5.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_d5.log
timeout 2400 bash scripts/sanitize.sh ${TAG} > gpurun_out/${TAG}_sanitize_summary.log 2>&1
