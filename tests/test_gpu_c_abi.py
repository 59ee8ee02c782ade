"""The C ABI used from plain C (examples/c_abi_demo.c): no Python in the
process — cudaMalloc'd vectors, salt_assign / salt_reduce /
salt_assign_reduce / salt_assign_host / salt_assign_batch, results checked
in C (bit-exact elementwise, 1e-12 for reductions)."""

import subprocess
from pathlib import Path

import pytest

DEMO = Path(__file__).resolve().parents[1] / "examples" / "c_abi_demo"


def test_demo_is_built():
    assert DEMO.exists(), "run __graft_entry__.build() (make -C paper_1109_1264_b200/csrc)"


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1000, (1 << 22) + 3])
def test_c_abi_demo(n):
    r = subprocess.run([str(DEMO), str(n)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
