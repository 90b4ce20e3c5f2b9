"""GPU parity: split kernel and tcgen05 emulated GEMM vs the reference.

Golden fixtures come from the reference itself (oracle/make_golden.py); the
larger cases are checked against the CPU oracle restatement on the same seeded
inputs.  The bar is bit-exactness (np.array_equal) for slices, exponents,
per-pair INT32 products and the emulated GEMM output.
"""

import numpy as np
import pytest

from testutil import load_golden
from oracle import ozaki_oracle as orc

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2509_23565_b200 as oz
    return oz


def test_split_matches_reference_golden():
    oz = _pkg()
    g = load_golden("split")
    for i in range(int(g["count"][0])):
        k, q, orient, mode = (int(v) for v in g[f"s{i}_meta"])
        st = oz.split_matrix(g[f"s{i}_a"], k, q,
                             oz.Orientation.COL_SCALED if orient else oz.Orientation.ROW_SCALED,
                             oz.ScalingMode.GLOBAL if mode else oz.ScalingMode.PER_VECTOR)
        assert np.array_equal(np.stack(st.slices), g[f"s{i}_slices"]), i
        assert np.array_equal(st.exponents, g[f"s{i}_exps"]), i


@pytest.mark.parametrize("shape", [(1, 1), (7, 300), (300, 7), (129, 1000), (2048, 96)])
@pytest.mark.parametrize("orient", ["row", "col"])
def test_split_matches_oracle_random(shape, orient):
    oz = _pkg()
    rng = np.random.default_rng(hash((shape, orient)) % 2**32)
    a = (rng.random(shape) - 0.5) * np.ldexp(1.0, rng.integers(-70, 71, size=(shape[0], 1)))
    for k in (1, 7, 12):
        st = oz.split_matrix(a, k, 7, oz.Orientation.ROW_SCALED if orient == "row"
                             else oz.Orientation.COL_SCALED)
        ref_s, ref_e = orc.split(a, k, 7, orient)
        assert np.array_equal(np.stack(st.slices), ref_s)
        assert np.array_equal(st.exponents, ref_e)


@pytest.mark.parametrize("shape", [(1, 1), (17, 1024), (3000, 1000), (40, 1023)])
def test_split_vector_contiguous_onepass(shape):
    """Row-scaled split of a column-major source (the LU's A21 layout: one
    pass through shared memory for K <= 1024) and column-scaled split of a
    row-major one: bit-exact against the oracle, zero rows included."""
    oz = _pkg()
    rng = np.random.default_rng(shape[0] * 31 + shape[1])
    a = (rng.random(shape) - 0.5) * np.ldexp(1.0, rng.integers(-70, 71, size=(shape[0], 1)))
    a[::7] = 0.0
    for k in (1, 7):
        st = oz.split_matrix(np.asfortranarray(a), k, 7, oz.Orientation.ROW_SCALED)
        ref_s, ref_e = orc.split(a, k, 7, "row")
        assert np.array_equal(np.stack(st.slices), ref_s)
        assert np.array_equal(st.exponents, ref_e)
        st = oz.split_matrix(np.ascontiguousarray(a.T), k, 7, oz.Orientation.COL_SCALED)
        ref_s, ref_e = orc.split(a.T, k, 7, "col")
        assert np.array_equal(np.stack(st.slices), ref_s)
        assert np.array_equal(st.exponents, ref_e)


def test_split_nonfinite_raises():
    oz = _pkg()
    with pytest.raises(oz.NonFiniteEntryError):
        oz.split_matrix(np.array([[np.nan, 1.0]]), 2)
    with pytest.raises(oz.NonFiniteEntryError):
        oz.split_matrix(np.array([[np.inf], [1.0]]), 2, orientation=oz.Orientation.COL_SCALED)


@pytest.mark.parametrize("m,n,kk", [(1, 1, 1), (128, 128, 128), (129, 257, 300), (300, 100, 1000),
                                    (64, 512, 4096), (1000, 700, 33)])
def test_pair_product_int32_exact(m, n, kk):
    """Per-slice-pair INT32 products are exact (test_gemm.py:218-240 pattern)."""
    import torch
    from paper_2509_23565_b200 import _lib
    rng = np.random.default_rng(m * 7 + n * 13 + kk)
    a = rng.integers(-127, 128, size=(m, kk), dtype=np.int8)
    b = rng.integers(-127, 128, size=(n, kk), dtype=np.int8)
    ld = -(-kk // 16) * 16
    da = torch.zeros((m, ld), dtype=torch.int8, device="cuda")
    db = torch.zeros((n, ld), dtype=torch.int8, device="cuda")
    da[:, :kk] = torch.from_numpy(a).cuda()
    db[:, :kk] = torch.from_numpy(b).cuda()
    out = torch.zeros((n, m), dtype=torch.int32, device="cuda")  # column-major m x n
    _lib.call("oz_gemm_pair_i32", m, n, kk, da.data_ptr(), ld, db.data_ptr(), ld,
              out.data_ptr(), m, torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy().T
    want = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(got.astype(np.int64), want)


def test_gemm_matches_reference_golden():
    oz = _pkg()
    g = load_golden("gemm")
    for i in range(int(g["count"][0])):
        k, limit, mode = (int(v) for v in g[f"g{i}_meta"])
        alpha, beta = (float(v) for v in g[f"g{i}_ab"])
        trunc = oz.FULL if limit == 2 * k else oz.Band(limit)
        bk = oz.GemmBackend.int8(k, 7, truncation=trunc,
                                 scaling=oz.ScalingMode.GLOBAL if mode else
                                 oz.ScalingMode.PER_VECTOR)
        c = g[f"g{i}_c"]
        out = oz.gemm(bk, alpha, g[f"g{i}_a"], g[f"g{i}_b"], beta, c if c.size else None)
        assert np.array_equal(out, g[f"g{i}_out"]), (i, k, limit)


def test_schur_calls_match_reference_golden():
    """The 9 Schur updates of the reference LU on ParaWilk_256 (k=3,7,9), bit-exact."""
    oz = _pkg()
    g = load_golden("schur")
    for i in range(int(g["count"][0])):
        k = int(g[f"c{i}_k"][0])
        out = oz.gemm(oz.GemmBackend.int8(k), -1.0, g[f"c{i}_a"], g[f"c{i}_b"], 1.0,
                      g[f"c{i}_c"])
        assert np.array_equal(out, g[f"c{i}_out"]), (i, k)


@pytest.mark.parametrize("k", [3, 6, 7, 9])
def test_gemm_matches_oracle_larger(k):
    oz = _pkg()
    rng = np.random.default_rng(k)
    a = rng.random((700, 1200)) - 0.5
    b = rng.random((1200, 530)) - 0.5
    out = oz.gemm(oz.GemmBackend.int8(k), 1.0, a, b, 0.0)
    assert np.array_equal(out, orc.gemm(1.0, a, b, 0.0, k=k))


def test_gemm_device_tensors_and_layouts():
    import torch
    oz = _pkg()
    rng = np.random.default_rng(3)
    a = rng.random((300, 257)) - 0.5
    b = rng.random((257, 190)) - 0.5
    c = rng.random((300, 190)) - 0.5
    want = orc.gemm(-1.0, a, b, 1.0, c, k=7)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda().t().contiguous().t()   # column-major view
    dc = torch.from_numpy(c).cuda()
    out = oz.gemm(oz.GemmBackend.int8(7), -1.0, da, db, 1.0, dc)
    assert out.is_cuda
    assert np.array_equal(out.cpu().numpy(), want)
    assert np.array_equal(dc.cpu().numpy(), c)   # inputs never mutated


def test_gemm_native_close():
    oz = _pkg()
    rng = np.random.default_rng(4)
    a, b, c = rng.random((64, 80)) - 0.5, rng.random((80, 50)) - 0.5, rng.random((64, 50)) - 0.5
    out = oz.gemm(oz.GemmBackend.native(), -1.0, a, b, 1.0, c)
    scale = np.abs(a) @ np.abs(b) + np.abs(c)
    assert (np.abs(out - (c - a @ b)) <= 4 * 2.0**-52 * scale).all()


def test_int16_slices_bit_exact():
    """slice_bits 8..10: the device split (int16 slices as hi/lo int8 planes)
    and the wide GEMM (exact recombination of the four plane products) are
    bit-identical to the reference (wide.npz) and to the oracle."""
    import paper_2509_23565_b200 as oz
    from oracle import ozaki_oracle as orc
    g = load_golden("wide")
    for i in range(int(g["split_count"][0])):
        k, q, orient = (int(v) for v in g[f"s{i}_meta"])
        st = oz.split_matrix(g["split_a"], k, q,
                             oz.Orientation.COL_SCALED if orient else oz.Orientation.ROW_SCALED)
        assert np.array_equal(np.stack(st.slices), g[f"s{i}_slices"]), i
        assert np.array_equal(st.exponents, g[f"s{i}_exps"]), i
    for i in range(int(g["gemm_count"][0])):
        k, q = (int(v) for v in g[f"g{i}_meta"])
        out = oz.gemm(oz.GemmBackend.int8(k, q), -1.0, g["gemm_a"], g["gemm_b"], 1.0, g["gemm_c"])
        assert np.array_equal(out, g[f"g{i}_out"]), (k, q)
    rng = np.random.default_rng(5)
    a = rng.random((300, 700)) - 0.5
    b = rng.random((700, 260)) - 0.5
    for q, k in ((8, 4), (10, 3), (10, 6)):
        got = oz.gemm(oz.GemmBackend.int8(k, q), 1.0, a, b, 0.0)
        assert np.array_equal(got, orc.gemm(1.0, a, b, 0.0, k=k, q=q)), (k, q)


def test_int16_slice_lu():
    import paper_2509_23565_b200 as oz
    g = load_golden("wide")
    f = oz.lu_factor(g["lu_a"], 16, oz.GemmBackend.int8(3, 10))
    assert np.array_equal(f.pivots, g["lu_perm"])
    assert np.abs(f.lu - g["lu_lu"]).max() <= 2.0**-40
    from oracle import ozaki_oracle as orc
    m = oz.hpl_uniform(512, 99)
    for k in (4, 6):      # 40 vs 60 mantissa bits: same verdict as the reference algorithm
        _, rep = oz.solve_system(m, m @ np.ones(512), 128, oz.GemmBackend.int8(k, 10))
        lu, perm, _ = orc.lu_factor(m, 128, k, q=10)
        ref = orc.residual(m, orc.lu_solve(lu, perm, m @ np.ones(512)), m @ np.ones(512))[0]
        assert rep.passed == (ref < 16.0) and 0.5 <= rep.scaled_residual / ref <= 2.0, (k, ref)
