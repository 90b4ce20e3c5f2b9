"""CPU: the C-ABI library loads and exports every symbol include/ozb200.h
declares; host-only entry points and the drop-in's host logic (pair tables,
backend validation, grouping plan, flop counting, generator parameters)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from testutil import ROOT

HEADER = os.path.join(ROOT, "include", "ozb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(oz_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_2509_23565_b200 import _lib
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(_lib.exported_symbols())


def test_host_entry_points():
    from paper_2509_23565_b200 import _lib
    lib = _lib.load()
    assert lib.oz_version() >= 100
    assert _lib.query("oz_split_aux_bytes") == 16
    assert _lib.query("oz_lu_workspace_bytes", 4096, 512, 7, 7) > 2 * 7 * 4096 * 512
    # slice_bits > 7: two int8 planes per slice
    assert (_lib.query("oz_lu_workspace_bytes", 4096, 512, 7, 10)
            > _lib.query("oz_lu_workspace_bytes", 4096, 512, 14, 7) - 4096)
    ipiv = np.array([2, 2, 3, 3], dtype=np.int32)
    perm = np.empty(4, dtype=np.int64)
    _lib.call("oz_ipiv_to_perm", ipiv.ctypes.data, 4, perm.ctypes.data)
    assert perm.tolist() == [2, 0, 3, 1]
    bad = np.array([5, 0], dtype=np.int32)
    from paper_2509_23565_b200.errors import InvalidParamsError
    with pytest.raises(InvalidParamsError):
        _lib.call("oz_ipiv_to_perm", bad.ctypes.data, 2, perm.ctypes.data)


def _plan(k, inner, q=7):
    from paper_2509_23565_b200 import _lib
    from paper_2509_23565_b200.gemm import GemmBackend, pair_table
    _, _, sh = pair_table(GemmBackend.int8(k, q))
    gs = np.zeros(len(sh) + 1, dtype=np.int32)
    gsh = np.zeros(len(sh), dtype=np.int32)
    ng = _lib.query("oz_plan_groups", len(sh), sh.ctypes.data, inner, q, gs.ctypes.data,
                    gsh.ctypes.data)
    return ng, gs[:ng + 1], gsh[:ng], sh


def test_grouping_plan_is_exact_and_ordered():
    for k in range(1, 10):
        for inner in (7, 64, 512, 16384, 130000):
            ng, gs, gsh, sh = _plan(k, inner)
            assert gs[0] == 0 and gs[-1] == len(sh)
            assert (np.diff(gs) >= 1).all()
            # groups are contiguous runs of one level
            for g in range(ng):
                assert (sh[gs[g]:gs[g + 1]] == gsh[g]).all()
            # once a level is split, no later group has more than one pair
            sizes = np.diff(gs)
            first_single = next((g for g in range(ng) if sizes[g] == 1 and
                                 (g + 1 < ng and gsh[g + 1] == gsh[g])), None)
            if first_single is not None:
                assert (sizes[first_single:] == 1).all()
            # exactness bound of the grouped prefix (INT32 and 53-bit)
            bound = 0.0
            for g in range(ng):
                if sizes[g] > 1 or (g + 1 < ng and gsh[g + 1] != gsh[g]):
                    lvl = inner * 127.0 * 127.0 * sizes[g]
                    if lvl >= 2**31:
                        break
                    bound += lvl * 2.0 ** -gsh[g]
                    if sizes[g] > 1:
                        assert bound * 2.0 ** gsh[g] < 2**53
    ng7, _, _, _ = _plan(7, 512)
    assert ng7 == 18          # levels 2..6 grouped, levels 7 and 8 per pair
    ng3, _, _, _ = _plan(3, 16384)
    assert ng3 == 3
    # int16 slices (q = 10): the 53-bit bound uses |slice| <= 1023
    for k in (3, 5):
        ng, gs, gsh, sh = _plan(k, 256, q=10)
        bound = 0.0
        for g in range(ng):
            if gs[g + 1] - gs[g] > 1:
                bound += 256 * 1023.0**2 * (gs[g + 1] - gs[g]) * 2.0 ** -gsh[g]
                assert bound * 2.0 ** gsh[g] < 2**53


def test_pair_tables_match_enumeration():
    import paper_2509_23565_b200 as oz
    for k in range(1, 10):
        for t in range(2, 2 * k + 1):
            prs = oz.retained_pairs(k, oz.Band(t))
            brute = sorted(((i, j) for i in range(1, k + 1) for j in range(1, k + 1)
                            if i + j <= t), key=lambda p: (p[0] + p[1], p[0]))
            assert list(prs) == brute
        assert len(oz.retained_pairs(k, oz.FULL)) == k * k
    with pytest.raises(oz.InvalidParamsError):
        oz.retained_pairs(2, oz.Band(1))
    with pytest.raises(oz.InvalidParamsError):
        oz.retained_pairs(2, oz.Band(5))


def test_backend_config_and_describe():
    import paper_2509_23565_b200 as oz
    assert oz.GemmBackend.native().describe() == "fp64"
    bk = oz.GemmBackend.int8(5)
    assert bk.truncation == oz.Band(6) and "band:6" in bk.describe()
    assert oz.GemmBackend.int8(7).describe() == "int8[splits=7,q=7,trunc=band:8,scale=pervector]"
    for bad in (lambda: oz.GemmBackend.int8(0), lambda: oz.GemmBackend.int8(3, slice_bits=11),
                lambda: oz.GemmBackend.int8(3, truncation=oz.Band(7))):
        with pytest.raises(oz.InvalidParamsError):
            bad()
    assert oz.GemmBackend(kind=oz.BackendKind.NATIVE_F64, splits=0).describe() == "fp64"


def test_flop_counts_match_reference_formulae():
    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200.solve import _count_flops
    c = oz.FlopCounter()
    _count_flops(c, 16, 4, oz.GemmBackend.int8(2))
    # recompute with the reference loop structure (solve.py:88-90,128-129; gemm.py:224-228)
    f64 = emu = pairs = 0
    n, nb, k, npairs = 16, 4, 2, 3
    for j in range(0, n, nb):
        jb = min(nb, n - j)
        for t in range(j, j + jb):
            rows = n - t - 1
            f64 += rows + rows * max(j + jb - t - 1, 0)
        rest = n - j - jb
        if rest > 0:
            f64 += jb * (jb - 1) // 2 * rest
            emu += npairs * rest * jb * rest
            pairs += npairs
            f64 += npairs * rest * rest + 2 * k * (rest * jb + jb * rest)
    assert (c.f64_ops, c.emulated_int_ops, c.slice_products_computed) == (f64, emu, pairs)


def test_parawilk_params_validation():
    import paper_2509_23565_b200 as oz
    assert oz.ParaWilkParams(5, 99, 2, 1.0).depth == 4
    assert "randomized,seed=4" in oz.ParaWilkParams(8, 2, 3, 0.5, True, 4).describe()
    for args in ((5, 0, 2, 1.0), (5, 2, 0, 1.0), (5, 2, 2, 0.0), (5, 2, 2, float("inf"))):
        with pytest.raises(oz.InvalidParamsError):
            oz.ParaWilkParams(*args)
    with pytest.raises(oz.InvalidDimError):
        oz.ParaWilkParams(1, 1, 1, 1.0)


def test_error_hierarchy_and_status_mapping():
    from paper_2509_23565_b200 import errors as E
    assert issubclass(E.NonSquareError, E.ShapeMismatchError)
    assert issubclass(E.InvalidDimError, E.InvalidParamsError)
    assert issubclass(E.SingularPivotError, ArithmeticError)
    assert E.STATUS_TO_ERROR[5] is E.SingularPivotError
    assert E.STATUS_TO_ERROR[4] is E.AccumulatorOverflowError


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_2509_23565_b200 as oz
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(oz.DeviceError):
        oz.gemm(oz.GemmBackend.int8(3), 1.0, np.eye(2), np.eye(2), 0.0)
    with pytest.raises(oz.DeviceError):
        oz.hpl_uniform(4, 1)
