"""Host side of scalar programs (runtime._scalar_program, no GPU needed):
lazy DeviceScalar arithmetic records operations, and lowering turns the
tree's device scalars into the postfix program salt_fused_prog runs."""

import numpy as np
import pytest
import torch

from paper_1109_1264_b200.runtime import _scalar_program
from paper_1109_1264_b200.vectors import DeviceScalar


def ds(v, dt="f64"):
    return DeviceScalar(torch.tensor([v], dtype=torch.float64 if dt == "f64" else torch.float32), dt)


def test_lazy_ops_record_and_materialise_with_ieee_ops():
    a, b = ds(1.5), ds(3.0)
    s = (a - 2.0) * b / (a + 0.25)
    assert s.lazy and s.program_size() == 9
    assert s.item() == np.float64((1.5 - 2.0) * 3.0 / (1.5 + 0.25))
    assert not s.lazy
    n = -a
    assert n.lazy and n.item() == -1.5
    f32 = ds(1.0, "f32") / 3.0
    assert f32.item().tobytes() == (np.float32(1.0) / np.float32(3.0)).tobytes()


def test_no_lazy_operand_means_no_program():
    a, b = ds(1.0), ds(2.0)
    raw, host, prog = _scalar_program([a, b], [0.5])
    assert raw == [a, b] and host == [0.5] and prog is None


def test_program_text_dedupes_raw_scalars_and_appends_constants():
    a, b = ds(1.0), ds(2.0)
    alpha = a / b
    raw, host, prog = _scalar_program([alpha, alpha, b], [7.0])
    assert raw == [a, b]
    assert prog == "p0 p1 / =0 p0 p1 / =1 p1 =2"
    assert host == [7.0]
    beta = (a - 2.0) * 3.0
    raw, host, prog = _scalar_program([beta], [])
    assert prog == "p0 S0 - S1 * =0" and host == [2.0, 3.0] and raw == [a]
    raw, host, prog = _scalar_program([-a], [])
    assert prog == "p0 neg =0"


def test_oversized_program_falls_back_to_raw_scalars():
    a, b = ds(1.0), ds(2.0)
    s = a
    for _ in range(20):
        s = s * 1.5 + b
    assert s.program_size() > DeviceScalar.MAX_PROGRAM_OPS
    raw, host, prog = _scalar_program([s], [])
    assert prog is None and raw == [s]   # materialised when the kernel reads its address
    mid = a
    for _ in range(10):
        mid = mid + 1.0                 # 21 ops: fits one, not two
    raw, host, prog = _scalar_program([mid, mid * 2.0], [])
    assert prog is None                 # > 32 ops together: everything raw


def test_modified_operand_is_refused():
    a, b = ds(1.0), ds(2.0)
    s = a / b
    b.copy_(4.0)
    with pytest.raises(RuntimeError, match="modified in place"):
        _scalar_program([s], [])
    with pytest.raises(RuntimeError, match="modified in place"):
        s.item()
