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


@pytest.mark.gpu
def test_result_slot_receives_the_reduction_without_a_copy():
    """salt_result_slot: this thread's pinned slot, mapped on the device at
    the same address; a reduction given it as out_dev stores its result
    straight into host memory (what lv.dot's fast path does)."""
    import ctypes

    import numpy as np
    import torch

    import paper_1109_1264_b200 as lv
    from paper_1109_1264_b200 import _native

    h = _native.lib()
    slot = ctypes.c_void_p()
    assert h.salt_result_slot(ctypes.byref(slot)) == 0 and slot.value
    again = ctypes.c_void_p()
    assert h.salt_result_slot(ctypes.byref(again)) == 0 and again.value == slot.value  # per thread
    for dt, code, ct in (("f64", 1, ctypes.c_double), ("f32", 0, ctypes.c_float)):
        for n in (1000, (1 << 20) + 7):
            g = np.random.default_rng(n)
            x, y = g.standard_normal(n), g.standard_normal(n)
            X, Y = (lv.DenseVector.from_values(v, dt, device="cuda") for v in (x, y))
            want = lv.dot(X, Y)
            ws = torch.zeros(h.salt_reduce_workspace_bytes(), dtype=torch.uint8, device="cuda")
            leaves, keep = _native.ptr_array([X.address, Y.address])
            sc, keep2 = _native.double_array([])
            ct.from_address(slot.value).value = -1.0
            stream = torch.cuda.current_stream().cuda_stream
            rc = h.salt_reduce(code, b"L0 L1 *", leaves, 2, sc, 0, n, 0, ws.data_ptr(), ws.numel(),
                               slot.value, None, stream)
            assert rc == 0, h.salt_last_error()
            assert h.salt_stream_synchronize(stream) == 0
            got = ct.from_address(slot.value).value
            assert np.asarray(got, dtype=want.dtype).tobytes() == np.asarray(want).tobytes(), (dt, n, got, want)
