#!/usr/bin/env python
"""Conjugate gradient on the 1-D Poisson matrix, written only with the
expression-tree API — the "iterative solver" that BASELINE config 5's
axpy -> dot step is the building block of.

    A = tridiag(-1, 2, -1) (n x n),  solve A u = b

* the matrix-vector product q = A p is ONE fused elementwise tree over
  shifted views of p (interior points; the two boundary rows are two tiny
  trees): 2*p[i] - p[i-1] - p[i+1];
* the step  u += a p ; r -= a q ; rr = r.r  is ONE fused kernel (lv.fused);
* p.q and the new direction p = r + beta p are fused trees too;
* reductions stay on the device (lazy=True) until the convergence check.

    python examples/cg_poisson1d.py --n 1048576 --iters 200
"""

import os
import argparse
import sys
import time
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1109_1264_b200 as lv  # noqa: E402


def views(v: lv.DenseVector):
    """(whole, interior, left neighbours, right neighbours) as DenseVectors
    sharing v's storage."""
    t = v.tensor
    n = t.shape[0]
    return (v, lv.DenseVector.from_tensor(t[1:n - 1]), lv.DenseVector.from_tensor(t[0:n - 2]),
            lv.DenseVector.from_tensor(t[2:n]))


def matvec(q, p):
    """q = A p for A = tridiag(-1, 2, -1)."""
    qt, pt = q.tensor, p.tensor
    n = pt.shape[0]
    _, qi, _, _ = views(q)
    _, pi, pl, pr = views(p)
    qi.assign(2.0 * pi - pl - pr)
    q0 = lv.DenseVector.from_tensor(qt[0:1])
    qn = lv.DenseVector.from_tensor(qt[n - 1:n])
    p0, p1 = lv.DenseVector.from_tensor(pt[0:1]), lv.DenseVector.from_tensor(pt[1:2])
    pn, pm = lv.DenseVector.from_tensor(pt[n - 1:n]), lv.DenseVector.from_tensor(pt[n - 2:n - 1])
    q0.assign(2.0 * p0 - p1)
    qn.assign(2.0 * pn - pm)


def cg(b: lv.DenseVector, iters: int, tol: float = 1e-10):
    n = len(b)
    u = lv.DenseVector.zeros(n, "f64")
    r = lv.DenseVector.zeros(n, "f64")
    r.assign(b)                         # r = b - A*0
    p = lv.DenseVector.zeros(n, "f64")
    p.assign(r)
    q = lv.DenseVector.zeros(n, "f64")
    rr = float(lv.dot(r, r))
    rr0 = rr
    k = 0
    for k in range(1, iters + 1):
        matvec(q, p)
        pq = float(lv.dot(p, q))
        a = rr / pq
        rr_new = float(lv.fused((u, u + a * p), (r, r - a * q), r * r))
        if rr_new <= tol * tol * rr0:
            rr = rr_new
            break
        beta = rr_new / rr
        p.assign(r + beta * p)
        rr = rr_new
    return u, k, (rr / rr0) ** 0.5


class DeviceCG:
    """The same CG iteration with every scalar kept on the device
    (DeviceScalar): no host synchronisation per iteration, so step() can be
    captured in a CUDA graph and replayed."""

    def __init__(self, b: lv.DenseVector):
        n = len(b)
        self.u = lv.DenseVector.zeros(n, "f64")
        self.r = lv.DenseVector.zeros(n, "f64")
        self.r.assign(b)
        self.p = lv.DenseVector.zeros(n, "f64")
        self.p.assign(self.r)
        self.q = lv.DenseVector.zeros(n, "f64")
        self.rr = lv.dot(self.r, self.r, lazy=True)

    def step(self):
        u, r, p, q = self.u, self.r, self.p, self.q
        matvec(q, p)
        alpha = self.rr / lv.dot(p, q, lazy=True)
        rr_new = lv.fused((u, u + alpha * p), (r, r - alpha * q), r * r, lazy=True)
        p.assign(r + (rr_new / self.rr) * p)
        self.rr.copy_(rr_new)  # in place: a captured graph re-reads the same address


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    g = np.random.default_rng(0)
    b = lv.DenseVector.from_values(g.standard_normal(a.n), "f64")
    cg(b, 2)  # warm-up: first-use kernel builds (NVRTC) are not part of the timing
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, k, rel = cg(b, a.iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    # independent check of the residual with torch ops
    ut, bt = u.tensor, b.tensor
    au = 2 * ut
    au[1:] -= ut[:-1]
    au[:-1] -= ut[1:]
    res = float(torch.linalg.vector_norm(bt - au) / torch.linalg.vector_norm(bt))
    print(f"host-scalar CG: n={a.n} iterations={k} relative residual (CG recurrence) {rel:.3e}, "
          f"recomputed {res:.3e}, {dt * 1e3:.1f} ms ({dt / k * 1e6:.1f} us/iteration)")

    # device-resident scalars, eager and captured in a CUDA graph
    cg_dev = DeviceCG(b)
    cg_dev.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        cg_dev.step()
    torch.cuda.synchronize()
    de = time.perf_counter() - t0
    cg_g = DeviceCG(b)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cg_g.step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        cg_g.step()
    graph.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        graph.replay()
    torch.cuda.synchronize()
    dg = time.perf_counter() - t0
    print(f"device-scalar CG: {de / k * 1e6:.1f} us/iteration eager, "
          f"{dg / k * 1e6:.1f} us/iteration as a CUDA graph")


if __name__ == "__main__":
    main()
