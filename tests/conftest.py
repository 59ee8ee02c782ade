"""Shared test setup.

Markers: `gpu` tests need a CUDA device (run on the B200 box with
`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`).
Golden fixtures in tests/golden/ were produced by the reference itself
(tests/golden/make_golden.py).
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
NP = {"f32": np.float32, "f64": np.float64}

# The reference's own unit tests (tests/reference_suite/): __graft_entry__.build()
# packs them into a git-ignored archive; they are extracted here for the
# length of the session (collected from tests/reference_suite/_vendored/)
# and removed again in pytest_sessionfinish.
REF_SUITE = ROOT / "tests" / "reference_suite"
REF_ARCHIVE = REF_SUITE / "reference_tests.tar.gz"
REF_DIR = REF_SUITE / "_vendored"


def _extract_reference_suite():
    import tarfile

    if not REF_ARCHIVE.exists():
        return
    REF_DIR.mkdir(exist_ok=True)
    with tarfile.open(REF_ARCHIVE) as tar:
        for m in tar.getmembers():
            if m.isfile() and m.name.startswith("test_") and m.name.endswith(".py") and "/" not in m.name:
                tar.extract(m, REF_DIR, filter="data")


_extract_reference_suite()


def pytest_sessionfinish(session, exitstatus):
    import shutil

    if REF_ARCHIVE.exists():
        shutil.rmtree(REF_DIR, ignore_errors=True)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configuration")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this process")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_cache = {}


def golden(name):
    """(meta list, npz mapping) of tests/golden/<name>.npz."""
    if name not in _cache:
        z = np.load(GOLDEN / f"{name}.npz")
        _cache[name] = (json.loads(str(z["meta"])), z)
    return _cache[name]


def same_bits(a, b) -> bool:
    """Bitwise equality, except that NaNs only need to be NaN in the same
    positions (NaN payloads are not specified)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return a[~na].tobytes() == b[~nb].tobytes()
