"""Time the parameter search (harness.search_params, harness.py:256-310) on the
B200 with sequential cells vs batches of concurrent solves, next to the
reference's measured CPU time (n=256, k=7 scan of 620 cells in
156 s on 8 cores).  Usage: python scripts/search_bench.py [n] [k] [batch...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_23565_b200 import harness  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 7
batches = [int(v) for v in sys.argv[3:]] or [1, 4, 8, 16]
harness.search_params(n, k, 1.0, 42, depth_max=1, block_max=3)      # warm
out = []
for bsz in batches:
    os.environ["OZEMU_THREADS"] = str(bsz)
    t0 = time.perf_counter()
    r = harness.search_params(n, k, 1.0, 42)
    dt = time.perf_counter() - t0
    out.append({"n": n, "splits": k, "batch": bsz, "seconds": dt, "cells": r.cells_scanned,
                "cells_per_s": r.cells_scanned / dt, "exhausted": r.exhausted,
                "d": r.depth, "b": r.block, "residual": r.scaled_residual})
    print(json.dumps(out[-1]), flush=True)
