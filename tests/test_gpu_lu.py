"""GPU parity: generators, LU factor/solve and the HPL scaled residual.

Bars:
  * generators: bit-exact with numpy's PCG64 stream (golden fixtures);
  * unblocked LU (lu_block = n <= 64): bit-exact factors, pivots and growth;
  * blocked LU: identical pivots, factors within 2^-40 (test_solve.py:61-66);
  * residual table on ParaWilk_256(4,15,1/2): identical verdicts, each entry
    within 2x of the reference oracle on the same matrix.
"""

import numpy as np
import pytest

from testutil import load_golden

pytestmark = pytest.mark.gpu


def _oz():
    import paper_2509_23565_b200 as oz
    return oz


def test_generators_bit_exact():
    oz = _oz()
    g = load_golden("matgen")
    assert np.array_equal(
        oz.parawilk_randomized(oz.ParaWilkParams(40, 3, 7, 0.5, randomize=True, seed=9)), g["pw40"])
    assert np.array_equal(oz.parawilk(oz.ParaWilkParams(5, 4, 2, 1.0)), g["pw5_det"])
    assert np.array_equal(oz.hpl_uniform(64, 99), g["uni64"])
    big = oz.hpl_uniform(2048, 7)
    assert np.array_equal(big.ravel()[g["uni2048_seed7_pos"]], g["uni2048_seed7_val"])
    assert np.array_equal(
        oz.parawilk_randomized(oz.ParaWilkParams(256, 4, 15, 0.5, randomize=True, seed=42)),
        g["pw256_seed42"])


def test_generator_layouts_agree():
    import torch
    from paper_2509_23565_b200.matgen import generate_device
    for kind in (0, 2):
        c = generate_device(kind, 333, seed=5, depth=3, block=7, alpha=0.25, layout="C")
        f = generate_device(kind, 333, seed=5, depth=3, block=7, alpha=0.25, layout="F")
        assert f.stride() == (1, 333)
        assert torch.equal(c, f)


def test_generator_sampled_at_scale():
    """Sampled stream positions of a large U(-1/2,1/2) draw match the PCG64 restatement."""
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200.matgen import generate_device
    n = 20000
    a = generate_device(0, n, seed=99)
    rng = np.random.default_rng(1)
    for idx in list(rng.integers(0, n * n, size=20)) + [0, n * n - 1]:
        i, j = divmod(int(idx), n)
        assert float(a[i, j]) == orc.pcg64_uniform_at(99, int(idx)) - 0.5


def test_unblocked_lu_bit_exact():
    oz = _oz()
    g = load_golden("lu")
    f = oz.lu_factor(g["unblocked_a"], 24)
    assert np.array_equal(f.pivots, g["unblocked_perm"])
    assert np.array_equal(f.lu, g["unblocked_lu"])
    assert f.growth == float(g["unblocked_growth"][0])


def test_blocked_lu_close():
    oz = _oz()
    g = load_golden("lu")
    f = oz.lu_factor(g["blocked_a"], 16)
    assert np.array_equal(f.pivots, g["blocked_perm"])
    assert np.abs(f.lu - g["blocked_lu"]).max() <= 2.0**-40


def test_wilkinson_growth():
    oz = _oz()
    g = load_golden("lu")
    for n in range(5, 21):
        f = oz.lu_factor(oz.wilkinson(n), min(4, n))
        assert f.growth == 2.0 ** (n - 1) == float(g[f"wilkinson_{n}_growth"][0])


@pytest.mark.parametrize("n,nb", [(40, 8), (100, 7), (257, 64), (700, 128), (1500, 300)])
def test_factorization_reconstructs(n, nb):
    oz = _oz()
    a = np.random.default_rng(n).random((n, n)) - 0.5
    f = oz.lu_factor(a, nb)
    l = np.tril(f.lu, -1) + np.eye(n)
    u = np.triu(f.lu)
    assert np.allclose(l @ u, a[f.pivots], atol=1e-12 * n)
    assert np.abs(np.tril(f.lu, -1)).max() <= 1.0
    # same pivots as the unblocked CPU oracle on a generic matrix
    from oracle import ozaki_oracle as orc
    _, perm, _ = orc.lu_factor(a, nb)
    assert np.array_equal(f.pivots, perm)


def test_singular_and_validation():
    oz = _oz()
    a = np.ones((3, 3))
    a[:, 0] = 0.0
    with pytest.raises(oz.SingularPivotError):
        oz.lu_factor(a, 1)
    with pytest.raises(oz.NonSquareError):
        oz.lu_factor(np.ones((2, 3)), 1)
    for nb in (0, -1, 5):
        with pytest.raises(oz.InvalidParamsError):
            oz.lu_factor(np.eye(4), nb)
    f = oz.lu_factor(np.random.default_rng(0).random((4, 4)), 2)
    with pytest.raises(ValueError):
        f.lu[0, 0] = 0.0


def test_solve_small_and_norms():
    oz = _oz()
    b = np.random.default_rng(1).random(5)
    f = oz.lu_factor(np.eye(5), 2)
    assert np.array_equal(oz.lu_solve(f, b), b)
    f = oz.lu_factor(np.array([[2.0, 0.0], [0.0, 4.0]]), 1)
    assert np.array_equal(oz.lu_solve(f, np.array([2.0, 8.0])), np.array([1.0, 2.0]))
    rep = oz.scaled_residual(np.array([[1.0, -2.0], [3.0, 4.0]]), np.array([1.0, -5.0]),
                             np.array([0.5, 2.0]))
    assert (rep.norm_a_inf, rep.norm_x_inf, rep.norm_b_inf) == (7.0, 5.0, 2.0)
    for backend in (oz.GemmBackend.native(), oz.GemmBackend.int8(3)):
        x, rep = oz.solve_system(np.eye(8), np.ones(8), 2, backend)
        assert rep.scaled_residual == 0.0 and rep.passed
        assert np.array_equal(x, np.ones(8))


def test_parawilk256_residual_table():
    """Paper table: fail k<=6, pass k>=7, each within 2x of the oracle."""
    oz = _oz()
    g = load_golden("residual")
    ks = list(g["parawilk256_splits"])
    ref = list(g["parawilk256_resid"])
    a = oz.parawilk_randomized(oz.ParaWilkParams(256, 4, 15, 0.5, randomize=True, seed=42))
    b = a @ np.ones(256)
    for k, r in zip(ks, ref):
        bk = oz.GemmBackend.native() if k == 0 else oz.GemmBackend.int8(int(k))
        _, rep = oz.solve_system(a, b, 64, bk)
        assert rep.passed == (r < 16.0), (k, rep.scaled_residual, r)
        assert 0.5 <= rep.scaled_residual / r <= 2.0, (k, rep.scaled_residual, r)


@pytest.mark.parametrize("n", [256, 512, 1024])
def test_uniform_residuals_vs_oracle(n):
    oz = _oz()
    g = load_golden("residual")
    ref = g[f"uniform{n}_resid"]
    a = oz.hpl_uniform(n, 99)
    b = a @ np.ones(n)
    for bk, r in zip((oz.GemmBackend.native(), oz.GemmBackend.int8(6), oz.GemmBackend.int8(7)),
                     ref):
        _, rep = oz.solve_system(a, b, 64, bk)
        assert rep.passed == (r < 16.0), (bk.describe(), rep.scaled_residual, r)
        assert 0.5 <= rep.scaled_residual / r <= 2.0, (bk.describe(), rep.scaled_residual, r)


def test_uniform_2048_nb256_verdicts():
    """n=2048, nb=256 -> fp64 0.0101, k=6 65.1 (fail), k=7 0.597."""
    oz = _oz()
    a = oz.hpl_uniform(2048, 99)
    b = a @ np.ones(2048)
    res = {}
    for name, bk in (("fp64", oz.GemmBackend.native()), ("k6", oz.GemmBackend.int8(6)),
                     ("k7", oz.GemmBackend.int8(7))):
        res[name] = oz.solve_system(a, b, 256, bk)[1].scaled_residual
    assert res["fp64"] < 1.0 and res["k7"] < 16.0 and res["k6"] >= 16.0, res
    assert 0.5 <= res["k6"] / 65.12 <= 2.0 and 0.5 <= res["k7"] / 0.5967 <= 2.0, res


@pytest.mark.parametrize("k", [5, 7])
def test_emulated_lu_global_scaling_matches_oracle(k):
    """Schur updates with ScalingMode.GLOBAL (one exponent per operand,
    split.py:131-134): identical pivots and factors close to the oracle LU
    run with mode=GLOBAL (the emulated products are bit-exact; the FP64
    panel/trsm parts are pinned to tolerance, test_solve.py:61-66)."""
    oz = _oz()
    from oracle import ozaki_oracle as orc
    from paper_2509_23565_b200.split import ScalingMode
    a = np.random.default_rng(3).random((300, 300)) - 0.5
    bk = oz.GemmBackend.int8(k, scaling=ScalingMode.GLOBAL)
    f = oz.lu_factor(a, 64, bk)
    lu_ref, perm_ref, _ = orc.lu_factor(a, 64, k, mode=orc.GLOBAL)
    assert np.array_equal(f.pivots, perm_ref)
    assert np.abs(f.lu - lu_ref).max() <= 2.0**-30
    # and it differs from per-vector scaling (the mode really reaches the kernel)
    g = oz.lu_factor(a, 64, oz.GemmBackend.int8(k))
    assert not np.array_equal(f.lu, g.lu)


_VARIANT_SCRIPT = r"""
import sys
import numpy as np
import paper_2509_23565_b200 as oz
from paper_2509_23565_b200.matgen import generate_device
from paper_2509_23565_b200.solve import factor_device
n, nb, k, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
a = generate_device(0, n, seed=7, layout="F")
ipiv, stats, info, _ = factor_device(a, nb, oz.GemmBackend.int8(k) if k else oz.GemmBackend.native())
np.savez(out, lu=a.cpu().numpy(), ipiv=ipiv.cpu().numpy(), info=int(info.item()),
         growth=float(stats[0].item()))
"""


@pytest.mark.parametrize("n,nb,k", [(3000, 512, 7), (2304, 1024, 0)])
def test_panel_exchange_variants(n, nb, k, tmp_path):
    """The panel leaf's three variants (shared-memory slab with grid-wide
    records + counter, shared-memory slab with cluster DSMEM + cluster
    barrier, register-resident rows with the cluster push exchange) compute
    the same arithmetic: factors, pivots and growth are bit-identical.
    Without look-ahead the trsm of the next panel's columns runs in the
    wide-trsm kernel (different FP64 summation order): same pivots, factors
    equal to rounding."""
    import os
    import subprocess
    import sys
    script = tmp_path / "variant.py"
    script.write_text(_VARIANT_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for i, env_extra in enumerate(({"OZ_PANEL_LEAF": "0", "OZ_PANEL_CLUSTER": "0"},
                                   {"OZ_PANEL_LEAF": "0", "OZ_PANEL_CLUSTER": "16"},
                                   {"OZ_LOOKAHEAD_SMS": "0"}, {})):
        env = dict(os.environ, PYTHONPATH=root, **env_extra)
        out = tmp_path / f"r{i}.npz"
        r = subprocess.run([sys.executable, str(script), str(n), str(nb), str(k), str(out)],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(out))
    grid, cluster, nola, reg = res
    for other in (cluster, reg):
        assert np.array_equal(grid["lu"], other["lu"])
        assert np.array_equal(grid["ipiv"], other["ipiv"])
        assert float(grid["growth"]) == float(other["growth"])
    assert np.array_equal(grid["ipiv"], nola["ipiv"])
    np.testing.assert_allclose(nola["lu"], grid["lu"], rtol=0,
                               atol=1e-9 * np.abs(grid["lu"]).max())


@pytest.mark.parametrize("n,nb", [(1500, 256), (3000, 1024), (2100, 64)])
def test_solve_system_host_overlapped_upload_matches_device(n, nb):
    """Host (row-major) inputs take the overlapped upload (column blocks over
    PCIe while the first panels factor): same x bit for bit as a device input,
    and non-finite entries still raise NonFiniteEntryError."""
    import torch

    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200.errors import NonFiniteEntryError
    from paper_2509_23565_b200.matgen import generate_device
    a = generate_device(0, n, seed=5)
    b = a.sum(1)
    bk = oz.GemmBackend.int8(7)
    x_dev, rep_dev = oz.solve_system(a, b, nb, bk)
    a_np, b_np = a.cpu().numpy(), b.cpu().numpy()
    x_np, rep_np = oz.solve_system(a_np, b_np, nb, bk)
    pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(a.cpu())
    x_pin, rep_pin = oz.solve_system(pinned, b_np, nb, bk)
    assert np.array_equal(x_dev.cpu().numpy(), x_np)
    assert np.array_equal(x_np, x_pin)
    assert rep_np.scaled_residual == rep_dev.scaled_residual < 16.0
    bad = a_np.copy()
    bad[n - 3, n - 2] = np.nan                  # in the last upload block
    with pytest.raises(NonFiniteEntryError):
        oz.solve_system(bad, b_np, nb, bk)


def test_solve_system_upload_phase_multi_block():
    """n = 6000, nb = 512: three 2048-column upload blocks, the first three
    steps left-looking over them; same pivots and residual verdict as the
    device-input path, x equal to rounding (different trsm kernels)."""
    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200.matgen import generate_device
    n, nb = 6000, 512
    a = generate_device(0, n, seed=9)
    b = a.sum(1)
    bk = oz.GemmBackend.int8(7)
    x_dev, rep_dev = oz.solve_system(a, b, nb, bk)
    x_np, rep_np = oz.solve_system(a.cpu().numpy(), b.cpu().numpy(), nb, bk)
    # the two paths differ only in trsm summation order; the k = 7 Schur
    # update carries that rounding into x at the level of x's own error
    xd = x_dev.cpu().numpy()
    err = max(np.max(np.abs(xd - 1.0)), np.max(np.abs(x_np - 1.0)))
    assert np.max(np.abs(x_np - xd)) <= max(1e-9, 2.0 * err), (np.max(np.abs(x_np - xd)), err)
    assert rep_np.passed and rep_dev.passed
    assert rep_np.scaled_residual < 2 * rep_dev.scaled_residual + 0.1


def test_solve_system_upload_phase_native_backend():
    """The upload phase with the native FP64 Schur update (solve_system's
    default backend): the deferred L-column interchanges keep every step's
    A21 rows in the order its pending block updates need.
    n = 6000, nb = 512 -> three 2048-column upload blocks."""
    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200.matgen import generate_device
    n, nb = 6000, 512
    a = generate_device(0, n, seed=11)
    b = a.sum(1)
    bk = oz.GemmBackend.native()
    x_dev, rep_dev = oz.solve_system(a, b, nb, bk)
    x_np, rep_np = oz.solve_system(a.cpu().numpy(), b.cpu().numpy(), nb)
    assert rep_dev.passed and rep_np.passed, (rep_dev.scaled_residual, rep_np.scaled_residual)
    assert rep_np.scaled_residual < 2 * rep_dev.scaled_residual + 0.1
    np.testing.assert_allclose(x_np, x_dev.cpu().numpy(), rtol=1e-9, atol=1e-9)
    # and the factors themselves: host-input LU == device-input LU to rounding
    f_dev = oz.lu_factor(a, nb)
    f_np = oz.lu_factor(a.cpu().numpy(), nb)
    assert np.array_equal(np.asarray(f_np.pivots), f_dev.pivots.cpu().numpy())


@pytest.mark.parametrize("k", [0, 7])
def test_lu_block_above_1024(k):
    """lu_block may be anything in 1..n (solve.py:109-110): nb = 1100 > 1024
    interchanges per panel compose chunk by chunk; pivots equal the oracle's."""
    oz = _oz()
    from oracle import ozaki_oracle as orc
    n, nb = 1200, 1100
    a = np.random.default_rng(5).random((n, n)) - 0.5
    bk = oz.GemmBackend.int8(k) if k else oz.GemmBackend.native()
    f = oz.lu_factor(a, nb, bk)
    lu_ref, perm_ref, _ = orc.lu_factor(a, nb, k if k else None)
    assert np.array_equal(f.pivots, perm_ref)
    assert np.abs(f.lu - lu_ref).max() <= 2.0**-30
    x, rep = oz.solve_system(a, a @ np.ones(n), nb, bk)
    assert rep.passed
    x2, rep2 = oz.solve_system(a, a @ np.ones(n), n, bk)      # lu_block = n: one panel
    assert rep2.passed


def test_solve_system_error_order():
    """lu_factor's checks come before lu_solve's rhs check (solve.py:227-228):
    NaN matrix + bad rhs -> NonFiniteEntryError, singular matrix + bad rhs ->
    SingularPivotError, bad lu_block + NaN -> NonFiniteEntryError; host and
    device inputs alike."""
    import torch
    oz = _oz()
    n = 300
    nan = np.random.default_rng(2).random((n, n))
    nan[5, 7] = np.nan
    sing = np.random.default_rng(2).random((n, n))
    sing[:, 3] = 0.0
    bad_rhs = np.ones(n + 1)
    for conv in (lambda x: x, lambda x: torch.from_numpy(x).cuda()):
        with pytest.raises(oz.NonFiniteEntryError):
            oz.solve_system(conv(nan), bad_rhs, 64)
        with pytest.raises(oz.SingularPivotError):
            oz.solve_system(conv(sing), bad_rhs, 64)
        with pytest.raises(oz.NonFiniteEntryError):
            oz.solve_system(conv(nan), np.ones(n), 0)
        with pytest.raises(oz.InvalidParamsError):
            oz.solve_system(conv(sing), np.ones(n), n + 1)
        with pytest.raises(oz.ShapeMismatchError):
            oz.solve_system(conv(np.eye(n)), bad_rhs, 64)
    # the device stays usable after an exception in the overlapped path
    x, rep = oz.solve_system(np.eye(n) * 2.0, np.ones(n) * 2.0, 64)
    assert np.array_equal(x, np.ones(n))


_LARGE_SCRIPT = r"""
import hashlib, json, sys
import torch
import paper_2509_23565_b200 as oz
from paper_2509_23565_b200.matgen import generate_device
n, nb = int(sys.argv[1]), int(sys.argv[2])
a = generate_device(0, n, seed=99)
b = a.sum(1)
x, rep = oz.solve_system(a, b, nb, oz.GemmBackend.int8(7))
f = oz.lu_factor(a, nb, oz.GemmBackend.int8(7))
piv = f.pivots.cpu().numpy().tobytes()
print(json.dumps({"resid": rep.scaled_residual, "piv": hashlib.sha256(piv).hexdigest()}))
"""


def test_large_lu_leaf_variants_agree(tmp_path):
    """An LU large enough for every register-leaf variant and the planner's
    paths (grid leaves with tagged-word records, the tall 1024-row leaf on the
    look-ahead's capped grid, two-phase look-ahead, aux-stream interchanges):
    the same pivots and a passing residual as with the shared-memory leaf for
    the tallest panels (OZ_PANEL_LEAF_TALL=0) — the leaf choice only moves the
    in-panel blocking, so factors agree to rounding."""
    import json
    import os
    import subprocess
    import sys
    script = tmp_path / "large.py"
    script.write_text(_LARGE_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for env_extra in ({}, {"OZ_PANEL_LEAF_TALL": "0"}):
        env = dict(os.environ, PYTHONPATH=root, **env_extra)
        r = subprocess.run([sys.executable, str(script), "20480", "1024"], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert out[0]["piv"] == out[1]["piv"]
    assert 0.0 < out[0]["resid"] < 1.0 and 0.0 < out[1]["resid"] < 1.0
