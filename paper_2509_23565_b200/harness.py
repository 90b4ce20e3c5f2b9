"""Experiment drivers on the B200 path: residual-vs-splits sweeps, the
first-failing ParaWilk parameter search and the blocking-factor benchmark,
with the reference's CSV v1 / table output (drop-in for
/root/reference/pkg/src/ozemu/harness.py:41-435).

Differences from the reference that do not change any row value:

* matrices are generated directly in HBM (bit-identical to numpy's draw,
  matgen.py:133-171) and stay there for every cell of a sweep;
* b = A @ ones is formed on the device (harness.py:126) — the same FP64
  values up to summation order, which the residual verdicts do not see;
* with ``OZEMU_THREADS`` > 1, independent cells run concurrently, each on
  its own CUDA stream from a worker thread (harness.py:56-72 uses a thread
  pool the same way); the parameter search scans its cells in batches of
  that many concurrent solves.  Rows and the first-failing cell are taken in
  scan order, so the results do not depend on the concurrency (the solver is
  deterministic and reentrant).  Default 1: a 256-order cell takes ~1.6 ms
  on the B200 and concurrent Python workers measured slower
  (profiles/r02_search_bench.log).
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .errors import InvalidParamsError, OzemuError
from .gemm import BackendKind, GemmBackend, retained_pairs
from .matgen import (GEN_PARAWILK, GEN_PARAWILK_RANDOMIZED, GEN_UNIFORM, ParaWilkParams,
                     generate_device)
from .solve import SolveReport, solve_system
from .split import ScalingMode

__all__ = ["CSV_SCHEMA_VERSION", "MatrixSpec", "SolveRow", "SearchResult", "BenchRow",
           "default_lu_block", "default_search_bounds", "sweep_splits", "search_params",
           "bench", "write_csv", "format_table"]

CSV_SCHEMA_VERSION = "ozemu csv v1"


def default_lu_block(n: int) -> int:
    """The reference's default panel width, max(1, min(64, n // 4))
    (harness.py:41-47); performance runs pass a wider one explicitly."""
    return max(1, min(64, n // 4))


def default_search_bounds(n: int) -> tuple[int, int]:
    """(depth_max, block_max) scanned by search_params (harness.py:256-258)."""
    return min(20, n // 8), min(32, n // 4)


def _clamp_block(lu_block, n):
    return default_lu_block(n) if lu_block is None else max(1, min(int(lu_block), n))


# ------------------------------------------------------------------ matrices
@dataclass(frozen=True)
class MatrixSpec:
    """A named test matrix (harness.py:75-121), generated on the device."""

    kind: str
    n: int
    depth: int | None = None
    block: int | None = None
    alpha: float | None = None
    randomize: bool = False
    seed: int | None = None

    def needs_seed(self) -> bool:
        return self.kind == "uniform" or (self.kind == "parawilk" and self.randomize)

    def build_device(self):
        """The matrix as a CUDA float64 tensor (row-major)."""
        n = self.n
        if self.kind == "parawilk":
            if None in (self.depth, self.block, self.alpha):
                raise InvalidParamsError("parawilk requires depth, block and alpha")
            p = ParaWilkParams(n, self.depth, self.block, self.alpha, randomize=self.randomize,
                               seed=self.seed)
            if p.randomize and p.seed is None:
                raise InvalidParamsError("a seed is required for randomized generation")
            kind = GEN_PARAWILK_RANDOMIZED if p.randomize else GEN_PARAWILK
            return generate_device(kind, n, p.seed, p.depth, p.block, p.alpha)
        if self.kind == "uniform":
            if self.seed is None:
                raise InvalidParamsError("uniform matrices require a seed")
            if n < 1:
                raise InvalidParamsError("n must be >= 1")
            return generate_device(GEN_UNIFORM, n, self.seed)
        if self.kind == "wilkinson":
            if n < 2:
                raise InvalidParamsError("n must be >= 2")
            return generate_device(GEN_PARAWILK, n, None, n - 1, n - 1, 1.0)
        if self.kind == "turing":
            if self.depth is None:
                raise InvalidParamsError("turing requires depth")
            if n < 2 or not 1 <= self.depth <= n - 1:
                raise InvalidParamsError(f"turing depth must be in 1..{n - 1}")
            return generate_device(GEN_PARAWILK, n, None, self.depth, n, 1.0)
        if self.kind == "identity":
            t = _dev.torch()
            return t.eye(n, dtype=t.float64, device="cuda")
        raise InvalidParamsError(f"unknown matrix kind {self.kind!r}")

    def build(self) -> np.ndarray:
        return self.build_device().cpu().numpy()

    def describe(self) -> str:
        if self.kind == "parawilk":
            tag = f"parawilk[n={self.n},d={self.depth},b={self.block},alpha={self.alpha!r}"
            return tag + (f",randomized,seed={self.seed}]" if self.randomize else "]")
        if self.kind == "uniform":
            return f"uniform[n={self.n},seed={self.seed}]"
        if self.kind == "turing":
            return f"turing[n={self.n},d={self.depth}]"
        return f"{self.kind}[n={self.n}]"


def _rhs_ones(a_dev):
    """b = A @ ones(n) on the device (harness.py:126)."""
    t = _dev.torch()
    n = int(a_dev.shape[0])
    b = t.empty((n,), dtype=t.float64, device="cuda")
    rs, cs = _dev.strides2d(a_dev)
    _lib.call("oz_row_sums", a_dev.data_ptr(), n, rs, cs, b.data_ptr(), _dev.stream())
    return b


def _solve_once(a_dev, backend: GemmBackend, lu_block: int) -> SolveReport:
    """Solve A x = A @ ones and report (harness.py:124-128); the module-level
    hook the drivers call (and the reference's tests monkeypatch)."""
    _, report = solve_system(a_dev, _rhs_ones(a_dev), lu_block=lu_block, backend=backend)
    return report


def _worker_count(default: int = 1) -> int:
    """OZEMU_THREADS (harness.py:56-61); unset -> default."""
    try:
        return max(1, int(os.environ["OZEMU_THREADS"]))
    except (KeyError, ValueError):
        return default


_tls = threading.local()


def _own_stream():
    """This worker thread's CUDA stream (created once per thread)."""
    s = getattr(_tls, "stream", None)
    if s is None:
        s = _tls.stream = _dev.torch().cuda.Stream()
    return s


def _map_in_order(fn, items, workers: int):
    """fn over items, results in item order; with workers > 1 each call runs
    on its worker thread's own stream, after the caller's stream (which
    produced the inputs), so independent solves overlap on the GPU."""
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    t = _dev.torch()
    origin = t.cuda.current_stream()
    dev = t.cuda.current_device()

    def run(x):
        t.cuda.set_device(dev)
        s = _own_stream()
        s.wait_stream(origin)
        with t.cuda.stream(s):
            return fn(x)

    with ThreadPoolExecutor(max_workers=min(workers, len(items))) as pool:
        return list(pool.map(run, items))


# ------------------------------------------------------------------ rows
def _fmt_res(x: float) -> str:
    return f"{x:.10g}"


def _fmt_sec(x: float) -> str:
    return f"{x:.6f}"


def _fmt_bool(x: bool) -> str:
    return "true" if x else "false"


@dataclass
class SolveRow:
    """One sweep row (harness.py:130-167); splits None = the FP64 baseline."""

    splits: int | None
    scaled_residual: float
    passed: bool
    int_macs: int
    f64_macs: int
    slice_pairs: int
    seconds: float
    backend: str
    error: str = ""

    CSV_FIELDS = ("splits", "scaled_residual", "passed", "int_macs", "f64_macs",
                  "slice_pairs", "seconds", "backend", "error")

    def to_csv_dict(self) -> dict:
        return {"splits": "fp64" if self.splits is None else str(self.splits),
                "scaled_residual": _fmt_res(self.scaled_residual),
                "passed": _fmt_bool(self.passed), "int_macs": str(self.int_macs),
                "f64_macs": str(self.f64_macs), "slice_pairs": str(self.slice_pairs),
                "seconds": _fmt_sec(self.seconds), "backend": self.backend,
                "error": self.error}

    @classmethod
    def from_report(cls, splits, rep: SolveReport) -> "SolveRow":
        fl = rep.flops
        return cls(splits=splits, scaled_residual=rep.scaled_residual, passed=rep.passed,
                   int_macs=fl.emulated_int_ops if fl else 0, f64_macs=fl.f64_ops if fl else 0,
                   slice_pairs=fl.slice_products_computed if fl else 0,
                   seconds=rep.seconds or 0.0, backend=rep.backend)


@dataclass
class SearchResult:
    """First failing (depth, block) cell in scan order (harness.py:213-247)."""

    n: int
    splits: int
    depth: int | None
    block: int | None
    scaled_residual: float | None
    cells_scanned: int
    exhausted: bool
    backend: str

    CSV_FIELDS = ("n", "splits", "d", "b", "scaled_residual", "cells_scanned", "exhausted",
                  "backend")

    def to_csv_dict(self) -> dict:
        return {"n": str(self.n), "splits": str(self.splits),
                "d": "" if self.depth is None else str(self.depth),
                "b": "" if self.block is None else str(self.block),
                "scaled_residual": ("" if self.scaled_residual is None
                                    else _fmt_res(self.scaled_residual)),
                "cells_scanned": str(self.cells_scanned), "exhausted": _fmt_bool(self.exhausted),
                "backend": self.backend}


@dataclass
class BenchRow:
    """Timing and analytic cost of one (n, lu_block, backend) cell
    (harness.py:313-352): model_ops = retained pairs x n^3 integer MACs
    (emulated) or 2 n^3 / 3 (native), model_gops = model_ops / seconds."""

    n: int
    lu_block: int
    backend: str
    seconds: float
    f64_macs: int
    int_macs: int
    slice_pairs: int
    model_ops: int
    model_gops: float
    scaled_residual: float
    skipped: str = ""

    CSV_FIELDS = ("n", "lu_block", "backend", "seconds", "f64_macs", "int_macs", "slice_pairs",
                  "model_ops", "model_gops", "scaled_residual", "skipped")

    def to_csv_dict(self) -> dict:
        return {"n": str(self.n), "lu_block": str(self.lu_block), "backend": self.backend,
                "seconds": _fmt_sec(self.seconds), "f64_macs": str(self.f64_macs),
                "int_macs": str(self.int_macs), "slice_pairs": str(self.slice_pairs),
                "model_ops": str(self.model_ops), "model_gops": f"{self.model_gops:.3f}",
                "scaled_residual": _fmt_res(self.scaled_residual), "skipped": self.skipped}


# ------------------------------------------------------------------ drivers
def sweep_splits(spec: MatrixSpec, splits_list, *, lu_block: int | None = None,
                 slice_bits: int = 7, scaling: ScalingMode = ScalingMode.PER_VECTOR,
                 include_baseline: bool = True) -> list[SolveRow]:
    """One solve per split count on one device-resident matrix, then the
    native FP64 baseline (harness.py:176-212).  Solver errors become the row's
    ``error`` instead of aborting the sweep."""
    ks = list(splits_list)
    if not ks:
        raise InvalidParamsError("splits range is empty")
    a = spec.build_device()
    nb = _clamp_block(lu_block, spec.n)

    def run(k):
        bk = GemmBackend.native() if k is None else GemmBackend.int8(k, slice_bits,
                                                                     scaling=scaling)
        try:
            return SolveRow.from_report(k, _solve_once(a, bk, nb))
        except OzemuError as exc:
            return SolveRow(splits=k, scaled_residual=float("nan"), passed=False,
                            int_macs=0, f64_macs=0, slice_pairs=0, seconds=0.0,
                            backend=bk.describe(), error=f"{type(exc).__name__}: {exc}")

    return _map_in_order(run, ks + ([None] if include_baseline else []), _worker_count())


def search_params(n: int, splits: int, alpha: float, seed: int, *,
                  depth_max: int | None = None, block_max: int | None = None,
                  lu_block: int | None = None, slice_bits: int = 7,
                  scaling: ScalingMode = ScalingMode.PER_VECTOR) -> SearchResult:
    """Scan depth, then block (ascending) until a randomized ParaWilk instance
    fails the scaled-residual check (harness.py:256-310).  A solver error
    (e.g. an exactly zero pivot) counts as a failure."""
    d0, b0 = default_search_bounds(n)
    depth_max = d0 if depth_max is None else depth_max
    block_max = b0 if block_max is None else block_max
    if depth_max < 1 or block_max < 2:
        raise InvalidParamsError("search bounds too small")
    bk = GemmBackend.int8(splits, slice_bits, scaling=scaling)
    nb = _clamp_block(lu_block, n)
    cells = [(d, b) for d in range(1, depth_max + 1) for b in range(2, block_max + 1)]

    def run(cell):
        d, b = cell
        spec = MatrixSpec("parawilk", n, d, b, alpha, randomize=True, seed=seed)
        try:
            rep = _solve_once(spec.build_device(), bk, nb)
        except OzemuError:
            return True, float("inf")
        return not rep.passed, rep.scaled_residual

    # batches of concurrent solves, consumed in scan order
    batch = _worker_count()
    scanned = 0
    for start in range(0, len(cells), batch):
        chunk = cells[start:start + batch]
        for (d, b), (failed, resid) in zip(chunk, _map_in_order(run, chunk, batch)):
            scanned += 1
            if failed:
                return SearchResult(n=n, splits=splits, depth=d, block=b,
                                    scaled_residual=resid, cells_scanned=scanned,
                                    exhausted=False, backend=bk.describe())
    return SearchResult(n=n, splits=splits, depth=None, block=None, scaled_residual=None,
                        cells_scanned=scanned, exhausted=True, backend=bk.describe())


def bench(n_values, lu_blocks, backend: GemmBackend, seed: int) -> list[BenchRow]:
    """Time U(-1/2,1/2) solves over sizes x panel widths (harness.py:355-395);
    widths that do not divide n are reported as skipped."""
    rows = []
    for n in n_values:
        a = MatrixSpec("uniform", n, seed=seed).build_device()
        for nb in lu_blocks:
            if nb > n or n % nb:
                rows.append(BenchRow(n=n, lu_block=nb, backend=backend.describe(), seconds=0.0,
                                     f64_macs=0, int_macs=0, slice_pairs=0, model_ops=0,
                                     model_gops=0.0, scaled_residual=float("nan"),
                                     skipped=f"lu_block {nb} does not divide n {n}"))
                continue
            rep = _solve_once(a, backend, nb)
            if backend.kind is BackendKind.EMULATED_INT8:
                model = len(retained_pairs(backend.splits, backend.truncation)) * n ** 3
            else:
                model = 2 * n ** 3 // 3
            fl, sec = rep.flops, rep.seconds or 0.0
            rows.append(BenchRow(n=n, lu_block=nb, backend=backend.describe(), seconds=sec,
                                 f64_macs=fl.f64_ops, int_macs=fl.emulated_int_ops,
                                 slice_pairs=fl.slice_products_computed, model_ops=model,
                                 model_gops=model / sec / 1e9 if sec > 0 else 0.0,
                                 scaled_residual=rep.scaled_residual))
    return rows


# ------------------------------------------------------------------ output
def write_csv(rows, stream, experiment: str, config_desc: str = "") -> None:
    """CSV with the schema line first (harness.py:410-422)."""
    head = f"# {CSV_SCHEMA_VERSION} experiment={experiment}"
    stream.write(head + (f" {config_desc}" if config_desc else "") + "\n")
    if not rows:
        return
    cols = type(rows[0]).CSV_FIELDS
    stream.write(",".join(cols) + "\n")
    for r in rows:
        d = r.to_csv_dict()
        stream.write(",".join(d[c] for c in cols) + "\n")


def format_table(rows) -> str:
    """Aligned plain-text table of the CSV values (harness.py:425-435)."""
    if not rows:
        return "(no rows)\n"
    cols = type(rows[0]).CSV_FIELDS
    ds = [r.to_csv_dict() for r in rows]
    w = {c: max([len(c)] + [len(d[c]) for d in ds]) for c in cols}
    out = ["  ".join(c.ljust(w[c]) for c in cols)]
    out += ["  ".join(d[c].ljust(w[c]) for c in cols) for d in ds]
    return "\n".join(out) + "\n"


del field
