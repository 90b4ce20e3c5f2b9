#!/bin/bash
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lu.py -q -x -p no:cacheprovider -k "upload or host or overlapped" > $O/${T}_tests.log 2>&1
for e in "$@"; do env $e timeout 300 python scripts/e2e_probe.py 32768 3 >> $O/${T}_e2e.log 2>&1; done
