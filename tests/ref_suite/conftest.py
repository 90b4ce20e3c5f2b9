"""Runs the reference's own pytest suite against the drop-in (VERDICT r1,
next 1).  scripts/run_ref_suite.sh copies /root/reference/pkg/tests into
tests/ref_suite/_staged/ (git-ignored, deleted after the run: reference
sources are never committed) and runs it on the B200 box, where
/root/reference does not exist.  Without a staged copy nothing is collected.

Every staged test is marked `gpu`: the drop-in computes on the device.
Deselections are listed in DESELECT, each with its reason.
"""

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SHIM = os.path.join(HERE, "ozemu_shim")
STAGED = os.path.join(HERE, "_staged")
ROOT = os.path.dirname(os.path.dirname(HERE))

if os.path.isdir(STAGED):
    for p in (ROOT, SHIM, STAGED):
        if p not in sys.path:
            sys.path.insert(0, p)
    # subprocess CLI tests (python -m ozemu.cli) resolve the alias too
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [ROOT, SHIM] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])
    import ozemu  # noqa: F401,E402  (installs the alias before the suite imports it)

# test node id suffix -> reason.  Empty: nothing is deselected unless a
# reference test exercises something outside SURVEY §8 (listed here if so).
DESELECT: dict[str, str] = {}


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(STAGED):
            item.add_marker(pytest.mark.gpu)
            for suffix, why in DESELECT.items():
                if item.nodeid.endswith(suffix):
                    item.add_marker(pytest.mark.skip(reason=why))
