"""CPU: the harness/CLI drop-in's host logic (harness.py, cli.py) —
range parsing, the CSV v1 / table formats of the reference
(harness.py:400-435, cli.py:35-51) and the usage-error exit codes, which
must trigger before any device work."""

import io

import pytest

from paper_2509_23565_b200 import cli, harness
from paper_2509_23565_b200.errors import InvalidParamsError


def test_parse_int_list():
    assert cli.parse_int_list("3:9", "x") == [3, 4, 5, 6, 7, 8, 9]
    assert cli.parse_int_list("256:1024:256", "x") == [256, 512, 768, 1024]
    assert cli.parse_int_list("3,5,7", "x") == [3, 5, 7]
    for bad in ("9:3", "1:2:0", "a,b", "1:2:3:4"):
        with pytest.raises(InvalidParamsError):
            cli.parse_int_list(bad, "--splits")


def test_default_blocks_and_bounds():
    assert harness.default_lu_block(256) == 64 and harness.default_lu_block(100) == 25
    assert harness.default_lu_block(2) == 1
    assert harness.default_search_bounds(256) == (20, 32)
    assert harness.default_search_bounds(64) == (8, 16)


def _rows():
    return [harness.SolveRow(3, 147971467.1234, False, 18 * 10, 99, 18, 0.01234567, "int8[k=3]"),
            harness.SolveRow(None, 0.011611101234, True, 0, 123, 0, 1.5, "fp64")]


def test_csv_v1_format():
    buf = io.StringIO()
    harness.write_csv(_rows(), buf, "sweep-splits", "matrix=x lu_block=64")
    lines = buf.getvalue().splitlines()
    assert lines[0] == "# ozemu csv v1 experiment=sweep-splits matrix=x lu_block=64"
    assert lines[1] == ("splits,scaled_residual,passed,int_macs,f64_macs,slice_pairs,seconds,"
                        "backend,error")
    assert lines[2] == "3,147971467.1,false,180,99,18,0.012346,int8[k=3],"
    assert lines[3] == "fp64,0.01161110123,true,0,123,0,1.500000,fp64,"
    buf = io.StringIO()
    harness.write_csv([], buf, "bench")
    assert buf.getvalue() == "# ozemu csv v1 experiment=bench\n"


def test_table_format_aligns_columns():
    t = harness.format_table(_rows()).splitlines()
    assert t[0].startswith("splits  scaled_residual  passed")
    assert len({len(line.rstrip()) > 0 for line in t}) == 1
    assert harness.format_table([]) == "(no rows)\n"


def test_search_and_bench_rows_csv():
    r = harness.SearchResult(256, 6, 1, 2, 143.1, 1, False, "int8[k=6]")
    assert r.to_csv_dict() == {"n": "256", "splits": "6", "d": "1", "b": "2",
                               "scaled_residual": "143.1", "cells_scanned": "1",
                               "exhausted": "false", "backend": "int8[k=6]"}
    e = harness.SearchResult(256, 7, None, None, None, 620, True, "int8[k=7]")
    assert e.to_csv_dict()["d"] == "" and e.to_csv_dict()["exhausted"] == "true"
    b = harness.BenchRow(1024, 128, "fp64", 0.5, 1, 2, 3, 715827882, 1.4316, 0.01)
    assert b.to_csv_dict()["model_gops"] == "1.432" and b.to_csv_dict()["seconds"] == "0.500000"


@pytest.mark.parametrize("argv", [
    ["sweep-splits", "--n", "64", "--splits", "3:9"],                 # --seed missing
    ["solve", "--n", "64", "--matrix", "uniform"],                    # seed needed for uniform
    ["solve", "--n", "64", "--matrix", "uniform", "--seed", "1", "--backend", "int8"],
    ["solve", "--n", "64", "--seed", "1", "--backend", "int8", "--splits", "7",
     "--truncation", "bogus"],
    ["sweep-splits", "--n", "64", "--seed", "1", "--splits", "9:3"],
    ["gemm", "--n", "8", "--matrix", "uniform"],                      # seed needed for uniform
    ["gemm", "--n", "8", "--matrix", "uniform", "--seed", "1", "--backend", "int8"],
    ["nonsense"],
])
def test_cli_usage_errors_exit_2(argv):
    assert cli.run_cli(argv) == 2
