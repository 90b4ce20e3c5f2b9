"""GPU: the experiment drivers and CLI on the B200 path reproduce the
reference's tables — sweep-splits on ParaWilk_256(4,15,1/2) seed 42 nb=64
(the paper's table, golden fixture from the reference itself): identical
verdicts, every residual within 2x; search-params finds a failing cell at
k=3; bench rows carry the reference's cost model."""

import io

import numpy as np
import pytest

from testutil import load_golden

pytestmark = pytest.mark.gpu


def test_sweep_splits_reproduces_reference_table():
    from paper_2509_23565_b200 import harness
    g = load_golden("residual")
    spec = harness.MatrixSpec("parawilk", 256, 4, 15, 0.5, randomize=True, seed=42)
    rows = harness.sweep_splits(spec, range(3, 10), lu_block=64)
    assert [r.splits for r in rows] == [3, 4, 5, 6, 7, 8, 9, None]
    for r, ref in zip(rows, g["parawilk256_resid"]):
        assert r.error == ""
        assert r.passed == (ref < 16.0)
        assert 0.5 <= r.scaled_residual / ref <= 2.0
    k7 = rows[4]
    assert k7.slice_pairs == 3 * 28                     # 3 Schur updates x P(7)


def test_cli_sweep_splits_csv():
    from paper_2509_23565_b200 import cli
    import contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.run_cli(["sweep-splits", "--n", "256", "--matrix", "parawilk", "--d", "4",
                          "--b", "15", "--alpha", "0.5", "--randomize", "--seed", "42",
                          "--splits", "6:7", "--lu-block", "64", "--strict"])
    lines = buf.getvalue().splitlines()
    assert rc == 1                                         # k=6 fails under --strict
    assert lines[0].startswith("# ozemu csv v1 experiment=sweep-splits matrix=parawilk[n=256")
    assert [ln.split(",")[2] for ln in lines[2:]] == ["false", "true", "true"]


def test_search_params_and_bench():
    from paper_2509_23565_b200 import GemmBackend, harness
    r = harness.search_params(128, 3, 0.5, 42, depth_max=2, block_max=6, lu_block=32)
    assert not r.exhausted and r.depth == 1 and r.scaled_residual >= 16.0
    rows = harness.bench([512], [128, 100], GemmBackend.int8(7), seed=99)
    assert rows[0].skipped == "" and rows[0].model_ops == 28 * 512 ** 3
    assert rows[0].scaled_residual < 16.0 and rows[0].model_gops > 0
    assert rows[1].skipped.startswith("lu_block 100 does not divide")


def test_cli_gen_matrix_market_roundtrip(tmp_path):
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200 import cli
    from paper_2509_23565_b200.mmio import read_matrix_market
    out = tmp_path / "a.mtx"
    assert cli.run_cli(["gen", "--n", "40", "--matrix", "uniform", "--seed", "5",
                        "--out", str(out)]) == 0
    assert np.array_equal(read_matrix_market(str(out)), orc.hpl_uniform(40, 5))


def test_gemm_error_profile_on_device_output():
    """gemm_error_profile (gemm.py:289-339) profiles the DEVICE product
    against the exact host product: integer inputs are exact on both
    backends, more splits strictly better, deterministic trials, and the
    `gemm` CLI (cli.py:142-175) prints the same numbers."""
    import contextlib
    import io as _io

    from paper_2509_23565_b200 import FULL, GemmBackend, cli, gemm_error_profile
    rng = np.random.default_rng(4)
    ai = rng.integers(-8, 9, size=(8, 8)).astype(float)
    bi = rng.integers(-8, 9, size=(8, 8)).astype(float)
    for bk in (GemmBackend.native(), GemmBackend.int8(3)):
        p = gemm_error_profile(bk, ai, bi)
        assert p.max_rel_error == 0.0 and p.max_abs_error == 0.0, bk.describe()
    a, b = rng.random((16, 16)) - 0.5, rng.random((16, 16)) - 0.5
    p3 = gemm_error_profile(GemmBackend.int8(3), a, b)
    p9 = gemm_error_profile(GemmBackend.int8(9), a, b)
    assert p9.max_rel_error < p3.max_rel_error
    full = gemm_error_profile(GemmBackend.int8(4, truncation=FULL), a, b)
    assert full.backend.startswith("int8[splits=4") and "full" in full.backend
    assert gemm_error_profile(GemmBackend.int8(3), a, b, trials=3, rng_seed=5) == \
        gemm_error_profile(GemmBackend.int8(3), a, b, trials=3, rng_seed=5)
    # k = 7 on U(-1/2,1/2): the element-scaled error stays at the FP64 level
    # (2.9e-15 at n = 512); here 64^3
    a, b = rng.random((64, 64)) - 0.5, rng.random((64, 64)) - 0.5
    assert gemm_error_profile(GemmBackend.int8(7), a, b).max_scaled_error < 1e-14
    buf = _io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.run_cli(["gemm", "--n", "24", "--matrix", "uniform", "--seed", "3",
                          "--backend", "int8", "--splits", "5", "--format", "csv"])
    assert rc == 0
    lines = buf.getvalue().splitlines()
    assert lines[0] == "# ozemu csv v1 experiment=gemm"
    # the reference writes the backend tag (which contains commas) unquoted
    # (cli.py:164-170), so the row is parsed from both ends
    head, row = lines[1].split(","), lines[2].split(",")
    assert head[:3] == ["m", "n", "p"] and row[:3] == ["24", "24", "24"]
    fields = dict(zip(head[-4:], row[-4:]))
    assert ",".join(row[3:-5]) == GemmBackend.int8(5).describe() and row[-5] == "1"
    prof = gemm_error_profile(GemmBackend.int8(5), oz_uniform(24, 3), oz_uniform(24, 4),
                              rng_seed=3)
    assert float(fields["max_rel_error"]) == float(f"{prof.max_rel_error:.10g}")


def oz_uniform(n, seed):
    from paper_2509_23565_b200 import hpl_uniform
    return hpl_uniform(n, seed)


def test_concurrent_cells_match_sequential(monkeypatch):
    """Sweeps and the parameter search run independent cells concurrently on
    per-thread streams; the rows equal the sequential ones bit for bit."""
    from paper_2509_23565_b200 import harness
    spec = harness.MatrixSpec("parawilk", 256, 4, 15, 0.5, randomize=True, seed=42)
    monkeypatch.setenv("OZEMU_THREADS", "1")
    seq = harness.sweep_splits(spec, range(3, 10))
    monkeypatch.setenv("OZEMU_THREADS", "8")
    par = harness.sweep_splits(spec, range(3, 10))
    assert [r.scaled_residual for r in seq] == [r.scaled_residual for r in par]
    monkeypatch.setenv("OZEMU_THREADS", "1")
    s1 = harness.search_params(256, 6, 1.0, 42)
    monkeypatch.delenv("OZEMU_THREADS")
    monkeypatch.setenv("OZEMU_THREADS", "8")
    s8 = harness.search_params(256, 6, 1.0, 42)
    assert (s1.depth, s1.block, s1.scaled_residual, s1.cells_scanned) == \
        (s8.depth, s8.block, s8.scaled_residual, s8.cells_scanned)
