"""Run the reference's OWN unit tests (pkg/tests/*.py) against this package.

build() packs /root/reference/pkg/tests/test_*.py, unmodified, into the
git-ignored archive reference_tests.tar.gz (reference sources stay out of
this repository's history; the archive travels to the GPU box with the
snapshot like the built .so files).  tests/conftest.py extracts them into
_vendored/ for the length of a pytest session only.  This conftest makes `import lanevec`
resolve to paper_1109_1264_b200 — the drop-in claim of SURVEY.md §8(b) —
before those modules are imported:

    lanevec              -> paper_1109_1264_b200
    lanevec.vectors      -> .vectors        lanevec.expressions -> .expressions
    lanevec.lanes        -> .lanes          lanevec.engine      -> .engine
    lanevec.ops          -> .ops            lanevec.bench       -> .benchmark
    lanevec.oracle       -> .checks (CountingVector + the scalar loops)

Every collected test is marked `gpu` (the package evaluates on the GPU
only), except test_lanes.py, which never evaluates a tree and also runs in
the CPU suite.  XFAIL lists the tests
whose reference contract this package deliberately does not keep, each with
its reason.
"""

import sys
from pathlib import Path

import pytest

import paper_1109_1264_b200 as _pkg
from paper_1109_1264_b200 import benchmark, checks, engine, expressions, lanes, ops, vectors

VENDORED = Path(__file__).resolve().parent / "_vendored"

ALIASES = {
    "lanevec": _pkg,
    "lanevec.vectors": vectors,
    "lanevec.expressions": expressions,
    "lanevec.lanes": lanes,
    "lanevec.engine": engine,
    "lanevec.ops": ops,
    "lanevec.bench": benchmark,
    "lanevec.oracle": checks,
}
for _name, _mod in ALIASES.items():
    sys.modules[_name] = _mod

CPU_FILES = {"test_lanes.py"}

# test node id (file::name, parametrisation stripped) -> reason
XFAIL = {
    "test_acceptance.py::test_criterion_7_performance_smoke": (
        "CPU-specific criterion: 'unroll 8 at least 1.1x faster than unroll 1' measures the "
        "reference's host lane loop.  Here engine-U1..U8 validate the plan and run the SAME fused "
        "GPU kernel (the unroll is a per-tree-shape kernel constant, SURVEY.md §8(a) a9), so the "
        "ratio is ~1.0 by design; the other half of the criterion (engine >= 2x naive) is asserted "
        "first and passes"),
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        path = Path(str(item.fspath))
        if VENDORED not in path.parents:
            continue
        if path.name not in CPU_FILES:
            item.add_marker(pytest.mark.gpu)
        key = f"{path.name}::{item.originalname if hasattr(item, 'originalname') else item.name}"
        if key in XFAIL:
            item.add_marker(pytest.mark.xfail(reason=XFAIL[key], strict=False))
