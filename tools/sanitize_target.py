#!/usr/bin/env python
"""Small run of every kernel kind for compute-sanitizer (one tool per run):
aligned and misaligned assignments (V = 4/8 and V = 1), reductions (single
CTA, one group, two levels), fused assign+reduce, the exchange emulation,
the host-streaming pipeline and a JIT tree.

    compute-sanitizer --tool memcheck python tools/sanitize_target.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import _native  # noqa: E402
from paper_1109_1264_b200.engine import execute_reduce  # noqa: E402
from paper_1109_1264_b200.expressions import SumNode, as_node  # noqa: E402


def main():
    g = np.random.default_rng(0)
    for dt in ("f32", "f64"):
        for n in (0, 1, 7, 1000, 4099, 300_001, 3_000_017):
            base = [torch.from_numpy(g.uniform(-1, 1, n + 3)).to(torch.float32 if dt == "f32" else torch.float64).cuda()
                    for _ in range(4)]
            for off in (0, 1):
                a, b, c, d = (lv.DenseVector.from_tensor(t[off:off + n]) for t in base)
                d.assign(1.5 * a + -0.5 * (b - c))
                d.assign(a * b * c - 2.0 * a)  # JIT tree
                lv.dot(a, b)
                lv.norm2(a)
                lv.axpy_dot(0.25, a, b, c)
                execute_reduce(SumNode(as_node(a) - as_node(b)))
        h = [lv.DenseVector.from_values(g.uniform(-1, 1, 100_003), dt, device="cpu") for _ in range(3)]
        h[2].assign(h[0] + 3.0 * h[1])
        lv.dot(h[0], h[1])
    lib = _native.lib()
    w, rounds = 4, 8
    tot = torch.randn(rounds * w * 2, dtype=torch.float64, device="cuda")
    res = torch.zeros_like(tot)
    scratch = torch.zeros(w * _native.XCHG_BUFFER_BYTES, dtype=torch.uint8, device="cuda")
    _native.check(lib.salt_exchange_emulate(w, rounds, 1, tot.data_ptr(), res.data_ptr(), scratch.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    print("sanitize target OK")


if __name__ == "__main__":
    main()
