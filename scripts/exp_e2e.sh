#!/bin/bash
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
for e in "$@"; do env $e timeout 300 python scripts/e2e_probe.py 32768 3 >> $O/${T}_e2e.log 2>&1; done
