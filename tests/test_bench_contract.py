"""bench.py's JSON-line contract: the reference arm on CPU, our arm on a B200
(small sizes; the driver runs the defaults)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-n", "256",
              "--cpu-nb", "64"], 600)
    assert BASE_KEYS <= set(d)
    # the sample runs emulated Schur updates (nb < n), at the config the GPU
    # line's same_config row reports
    assert d["config"]["nb"] < d["config"]["n"] and d["config"]["k"] == 7
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--n", "4096", "--nb", "512", "--steps", "3", "--warmup", "3", "--sweep-k", "",
              "--skip-native", "--e2e-steps", "1", "--cpu-n", "256", "--cpu-nb", "64",
              "--size-sweep", "1024,2048"], 900)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["gpu_launches"] > 0 and d["passed"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] >= 8 * 4096 * 4096
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["parawilk256_table"]["all_verdicts_match"]
    same = d["same_config"]
    ref = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-n", "256",
                "--cpu-nb", "64"], 600)
    assert same["config"] == ref["config"]
    assert same["gpu"]["value"] > 0 and same["e2e"]["value"] > 0
    runs = d["lu_size_sweep"]["runs"]
    assert {(r["n"], r["k"]) for r in runs} == {(n, k) for n in (1024, 2048)
                                                 for k in (6, 7, "fp64")}
    for r in runs:                      # k = 6 fails, k = 7 and FP64 pass
        assert r["passed"] == (r["k"] != 6), r


@pytest.mark.gpu
def test_distributed_arm_line_gloo():
    """run_distributed (configs[3] shape, randomized ParaWilk) with 2 ranks
    sharing the one GPU over gloo: one JSON line, residual table k = 6, 7 and
    native with the configs' verdicts."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "1", "--dist-n", "2048", "--nb", "256",
                        "--sweep-k", "6,7", "--e2e-steps", "1", "--cpu-n", "256",
                        "--cpu-nb", "64"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["matrix"] == "parawilk"
    assert d["config"]["workload"].startswith("configs[3]")
    assert d["passed"]
    verdicts = {row["k"]: row["passed"] for row in d["residual_table"]["runs"]}
    assert verdicts == {6: False, 7: True, "fp64": True}, verdicts
