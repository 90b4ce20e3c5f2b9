"""Import alias `ozemu` -> paper_2509_23565_b200, so the reference's own test
suite (/root/reference/pkg/tests, staged by scripts/run_ref_suite.sh) runs
unmodified against the B200 drop-in (implication 1).

Every submodule the suite imports is the drop-in's own module object (one
copy, so enum/class identities and monkeypatches are shared); `ozemu.oracle`
is the drop-in's exact host product (exact.py).  `ozemu.cli` is left to the
import system: `python -m ozemu.cli` then runs the drop-in's cli.py as
__main__ through the aliased package path.
"""

import importlib
import sys

_pkg = importlib.import_module("paper_2509_23565_b200")
sys.modules["ozemu"] = _pkg
# module objects via import_module: the package attribute `gemm` is the
# function (as in the reference, whose __init__ also re-exports gemm.gemm)
for _name, _real in (("errors", "errors"), ("gemm", "gemm"), ("harness", "harness"),
                     ("matgen", "matgen"), ("mmio", "mmio"), ("solve", "solve"),
                     ("split", "split"), ("oracle", "exact")):
    sys.modules["ozemu." + _name] = importlib.import_module("paper_2509_23565_b200." + _real)
