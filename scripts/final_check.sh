#!/bin/bash
# full GPU test suite + reference suite + round bench
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --ignore=tests/ref_suite > $O/${T}_gputest.log 2>&1; echo rc=$? >> $O/${T}_gputest.log
timeout 600 python -m pytest tests/ref_suite -m gpu -q -p no:cacheprovider -rs > $O/${T}_ref_suite.log 2>&1; echo rc=$? >> $O/${T}_ref_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1
bash scripts/bench_round.sh $T
