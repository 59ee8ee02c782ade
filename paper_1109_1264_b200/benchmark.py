"""GPU size sweeps with the reference's CSV contract (`salt-bench`).

The reference's `lanevec-bench` (pkg/src/lanevec/bench.py:1-349) sweeps the
level-1 ops over sizes and variants and writes
`op,variant,type,n,reps,best_s,median_s,gflops,gbytes`.  This module keeps
that CLI and CSV (same header, same accounting for the shared ops,
bench.py:9-15 / :49-50) and times on the device:

  variants
    engine          fused sm_100a kernel, device-resident vectors (CUDA events)
    engine-U1..U8   accepted for CLI compatibility: the plan is validated,
                    the kernel is the same fused kernel
    engine-host     pinned host vectors streamed through the GPU (end to end,
                    wall clock around the blocking call)
    torch           the same tree as one torch eager op per node with
                    materialised temporaries — "BLAS composition", the
                    baseline the paper's fusion claim is measured against
    naive           the reference's name for its unfused baseline (scalar
                    loops there, bench.py:121-132): here the same unfused
                    torch composition as `torch`
  ops
    dot scal axpy scaled_copy            (reference OPS, bench.py:46)
    sum norm2 t1 t2 etree axpy_dot       (BASELINE configs; --op extended)

--flush-l2 overwrites a 256 MiB buffer (> 126 MB L2) between reps, outside
the timed region, for HBM claims.  --extended adds pct_hbm (of the
measured copy peak), device, gpus, bytes and pct_hbm_nominal (of 8 TB/s)
columns.
"""

import argparse
import json
import statistics
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = ["BenchRecord", "OPS", "EXTENDED_OPS", "VARIANTS", "run_sweep", "emit_csv", "parse_csv",
           "main", "bytes_moved", "flop_count", "default_sizes", "gpu_sizes", "simd_available", "record_lines",
           "measure", "CSV_HEADER"]

OPS = ("dot", "scal", "axpy", "scaled_copy")
EXTENDED_OPS = OPS + ("sum", "norm2", "t1", "t2", "etree", "axpy_dot")
VARIANTS = ("engine", "engine-host", "torch", "naive", "engine-U1", "engine-U2", "engine-U4", "engine-U8")
CSV_HEADER = "op,variant,type,n,reps,best_s,median_s,gflops,gbytes"
# + gpus, bytes (algorithmic, per call), % of the
# measured and of the nominal (8 TB/s) HBM peak, device
EXT_HEADER = CSV_HEADER + ",pct_hbm,device,gpus,bytes,pct_hbm_nominal"
NOMINAL_HBM_GBS = 8000.0

# per element: (flops, distinct vectors read + written)
_ACCOUNT = {
    "dot": (2, 2), "scal": (1, 2), "axpy": (2, 3), "scaled_copy": (1, 2), "sum": (1, 1),
    "norm2": (2, 1), "t1": (2, 4), "t2": (4, 4), "etree": (7, 5), "axpy_dot": (4, 4),
}
_ALPHA, _BETA, _GAMMA = 1.25, -0.75, 0.5


@dataclass(frozen=True)
class BenchRecord:
    op: str
    variant: str
    type: str
    n: int
    reps: int
    best_s: float
    median_s: float
    gflops: float
    gbytes: float
    # GPU extras (--extended CSV columns).  They take no part in equality, so
    # a record read back from the reference's 9-column CSV equals the one
    # written (reference test_bench.py:90-100).
    pct_hbm: float = field(default=float("nan"), compare=False)
    device: str = field(default="", compare=False)
    gpus: int = field(default=1, compare=False)
    bytes: int = field(default=0, compare=False)
    pct_hbm_nominal: float = field(default=float("nan"), compare=False)


def default_sizes() -> list:
    """The reference's sweep (bench.py:72-82): every power of two 2^6 .. 2^22
    with its +-1 neighbours.  Device-scale sweeps: gpu_sizes()."""
    out = set()
    for p in range(6, 23):
        out.update(((1 << p) - 1, 1 << p, (1 << p) + 1))
    return sorted(out)


def gpu_sizes() -> list:
    """2^6 .. 2^28 by 4x, each with its +-1 neighbours (`--sizes gpu`): up to
    the HBM-resident sizes where the roofline applies."""
    out = set()
    for p in range(6, 29, 2):
        out.update(((1 << p) - 1, 1 << p, (1 << p) + 1))
    return sorted(out)


def flop_count(op, n):
    return _ACCOUNT[op][0] * n


def bytes_moved(op, n, dtype):
    from .lanes import as_dtype

    return _ACCOUNT[op][1] * n * as_dtype(dtype).itemsize


def simd_available(dtype="f32") -> bool:
    """True when a batched lane backend is active for this element type
    (the reference's gate for its performance smoke test, bench.py:92-94);
    the lane descriptor here is the same validated plan descriptor."""
    from .lanes import default_backend

    return default_backend(dtype).caps.specialized


def _hbm_peak():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def _operands(op, n, dt, device, seed):
    import paper_1109_1264_b200 as lv

    g = np.random.default_rng([seed, n, EXTENDED_OPS.index(op)])
    count = {"dot": 2, "scal": 1, "axpy": 2, "scaled_copy": 1, "sum": 1, "norm2": 1, "t1": 3,
             "t2": 3, "etree": 4, "axpy_dot": 3}[op]
    vecs = [lv.DenseVector.from_values(g.uniform(-1, 1, n), dt, device=device) for _ in range(count)]
    out = lv.DenseVector.zeros(n, dt, device=device) if op in ("scaled_copy", "t1", "t2", "etree") else None
    return vecs, out


def _make_data(op, n, dtype, seed, device=None):
    """(x, y, out) of a reference op, seeded as the reference seeds them
    (bench.py:97-106: stream [seed, n, op index], x then y, out zeros)."""
    vecs, out = _operands(op, n, dtype, device if device is not None else "cuda", seed)
    return vecs[0], (vecs[1] if len(vecs) > 1 else None), out


def _engine_call(op, x, y, out, alpha, options):
    """Zero-argument callable running a reference op once (reference
    bench.py:109-118)."""
    import paper_1109_1264_b200 as lv

    if op == "dot":
        return lambda: lv.dot(x, y, lazy=True, **options)
    if op == "scal":
        return lambda: lv.scal(alpha, x, **options)
    if op == "axpy":
        return lambda: lv.axpy(alpha, x, y, **options)
    if op == "scaled_copy":
        return lambda: lv.scaled_copy(alpha, x, out, **options)
    raise ValueError(f"unknown op {op!r}")


def _engine_call_ext(op, v, out, options):
    """The BASELINE-config ops (and the reference ops) over operand list v."""
    import paper_1109_1264_b200 as lv

    if op == "dot":
        return lambda: lv.dot(v[0], v[1], lazy=True, **options)
    if op == "sum":
        return lambda: lv.sum(v[0], lazy=True, **options)
    if op == "norm2":
        return lambda: lv.norm2(v[0], lazy=True, **options)
    if op == "scal":
        return lambda: lv.scal(_ALPHA, v[0], **options)
    if op == "axpy":
        return lambda: lv.axpy(_ALPHA, v[0], v[1], **options)
    if op == "scaled_copy":
        return lambda: lv.scaled_copy(_ALPHA, v[0], out, **options)
    if op == "t1":
        return lambda: out.assign(v[0] + (v[1] - v[2]), **options)
    if op == "t2":
        return lambda: out.assign(_ALPHA * v[0] + _BETA * (v[1] - v[2]), **options)
    if op == "etree":
        return lambda: out.assign(
            _ALPHA * (v[0] + v[1]) - _BETA * (v[2] - v[3]) + _GAMMA * v[0], **options)
    if op == "axpy_dot":
        return lambda: lv.axpy_dot(_ALPHA, v[0], v[1], v[2], lazy=True, **options)
    raise ValueError(f"unknown op {op!r}")


def _torch_call(op, v, out):
    """One torch eager kernel per node, temporaries materialised in HBM."""
    import torch

    t = [x.tensor for x in v]
    dt = t[0].dtype
    a, b, g = (torch.tensor(s, dtype=dt).item() for s in (_ALPHA, _BETA, _GAMMA))
    if op == "dot":
        return lambda: torch.sum(torch.mul(t[0], t[1]))
    if op == "sum":
        return lambda: torch.sum(t[0])
    if op == "norm2":
        return lambda: torch.sqrt(torch.sum(torch.mul(t[0], t[0])))
    if op == "scal":
        return lambda: t[0].copy_(torch.mul(t[0], a))
    if op == "axpy":
        return lambda: t[1].copy_(torch.add(t[1], torch.mul(t[0], a)))
    if op == "scaled_copy":
        return lambda: out.tensor.copy_(torch.mul(t[0], a))
    if op == "t1":
        return lambda: out.tensor.copy_(torch.add(t[0], torch.sub(t[1], t[2])))
    if op == "t2":
        return lambda: out.tensor.copy_(torch.add(torch.mul(t[0], a), torch.mul(torch.sub(t[1], t[2]), b)))
    if op == "etree":
        return lambda: out.tensor.copy_(torch.add(torch.sub(torch.mul(torch.add(t[0], t[1]), a),
                                                            torch.mul(torch.sub(t[2], t[3]), b)),
                                                  torch.mul(t[0], g)))
    if op == "axpy_dot":
        def f():
            t[1].copy_(torch.add(t[1], torch.mul(t[0], a)))
            return torch.sum(torch.mul(t[1], t[2]))
        return f
    raise ValueError(op)


def measure(op, variant, n, dtype="f32", reps=25, warmup=5, seed=0, packages=None, flush_l2=False):
    import torch

    from .lanes import as_dtype, dtype_name

    dt = as_dtype(dtype)
    host = variant == "engine-host"
    device = "cpu" if host else "cuda"
    vecs, out = _operands(op, n, dt, device, seed)
    options = {}  # validated by the engine exactly as the reference's (bench.py:135-141)
    if variant.startswith("engine-U"):
        options["unroll"] = int(variant[len("engine-U"):])
    if packages is not None:
        options["packages"] = packages
    unfused = variant in ("torch", "naive")
    if unfused:
        call = _torch_call(op, vecs, out)
    elif op in OPS:  # through the module global, so a spy can wrap it (reference test_bench.py:190-212)
        call = _engine_call(op, vecs[0], vecs[1] if len(vecs) > 1 else None, out, _ALPHA, options)
    else:
        call = _engine_call_ext(op, vecs, out, options)
    mutated = {"scal": 0, "axpy": 1, "axpy_dot": 1}.get(op)
    pristine = vecs[mutated].tensor.clone() if mutated is not None and n else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if flush_l2 else None

    def restore():
        if pristine is not None:
            vecs[mutated].tensor.copy_(pristine)
        if flush is not None:
            flush.fill_(1)

    for _ in range(warmup):
        restore()
        call()
    torch.cuda.synchronize()
    # Device variants without an L2 flush: below 64 MB of traffic a call
    # lasts a few microseconds, close to the ~1-2 us tick of the event
    # clock, so one rep times `inner` back-to-back calls and divides.
    # In-place ops (scal, axpy, axpy_dot) keep one call per rep, so every
    # call starts from the restored operand, as in the reference
    # (bench.py:156-170).
    inner = 1 if host or flush is not None or mutated is not None or bytes_moved(op, n, dt) >= (64 << 20) \
        else 16
    times = []
    for _ in range(reps):
        restore()
        if host:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            call()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        else:
            # queue ~50 us of GPU work per call first so the events bracket device time,
            # not the host's launch latency
            torch.cuda._sleep(100_000 * inner)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(inner):
                call()
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e) / 1e3 / inner)
    best = min(times)
    med = statistics.median(times)
    gbytes = bytes_moved(op, n, dt) / best / 1e9
    return BenchRecord(op, variant, dtype_name(dt), n, reps, best, med, flop_count(op, n) / best / 1e9,
                       gbytes, gbytes / _hbm_peak(), torch.cuda.get_device_name(), 1,
                       bytes_moved(op, n, dt), gbytes / NOMINAL_HBM_GBS)


def run_sweep(ops, variants, sizes, dtype="f32", reps=25, warmup=5, seed=0, packages=None, flush_l2=False):
    for op in ops:
        if op not in EXTENDED_OPS:
            raise ValueError(f"unknown op {op!r}; choose from {', '.join(EXTENDED_OPS)}")
    for v in variants:
        if v not in VARIANTS:
            raise ValueError(f"unknown variant {v!r}; choose from {', '.join(VARIANTS)}")
    return [measure(op, v, n, dtype, reps, warmup, seed, packages, flush_l2)
            for op in ops for v in variants for n in sizes]


def _lines(records, extended):
    yield EXT_HEADER if extended else CSV_HEADER
    for r in records:
        vals = [r.op, r.variant, r.type, r.n, r.reps, r.best_s, r.median_s, r.gflops, r.gbytes]
        if extended:
            vals += [r.pct_hbm, r.device.replace(",", " "), r.gpus, r.bytes, r.pct_hbm_nominal]
        yield ",".join(repr(v) if isinstance(v, float) else str(v) for v in vals)


def record_lines(records):
    """Header + one CSV row per record (the reference's record_lines,
    bench.py:222-231)."""
    return _lines(records, False)


def emit_csv(records, destination, extended=False) -> None:
    if destination == "-":
        for ln in _lines(records, extended):
            sys.stdout.write(ln + "\n")
        return
    with open(destination, "w") as f:
        for ln in _lines(records, extended):
            f.write(ln + "\n")


def parse_csv(text: str) -> list:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] not in (CSV_HEADER, EXT_HEADER):
        raise ValueError("missing or malformed CSV header")
    ext = lines[0] == EXT_HEADER
    out = []
    for ln in lines[1:]:
        p = ln.split(",")
        extra = [float(p[9]), p[10], int(p[11]), int(p[12]), float(p[13])] if ext else []
        rec = BenchRecord(p[0], p[1], p[2], int(p[3]), int(p[4]), float(p[5]), float(p[6]),
                          float(p[7]), float(p[8]), *extra)
        out.append(rec)
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="salt-bench",
                                 description="Sweep fused BLAS-1 kernels on the GPU and emit CSV.")
    ap.add_argument("--op", default="all", help="one op, 'all' (reference ops) or 'extended'")
    ap.add_argument("--type", default="f32", choices=("f32", "f64"))
    ap.add_argument("--variants", default="engine,torch")
    ap.add_argument("--sizes", default="default",
                    help="'default' (the reference's 2^6..2^22 sweep), 'gpu' (2^6..2^28 by 4x) or a comma list")
    ap.add_argument("--reps", type=int, default=25)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--csv", default="-")
    ap.add_argument("--packages", type=int, default=None,
                    help="accepted and validated like the reference's (bench.py:294-295)")
    ap.add_argument("--cache-sizes", default=None,
                    help="comma list of cache sizes in bytes, written to <csv>.meta for plotting "
                         "(reference bench.py:295-297; ignored on stdout)")
    ap.add_argument("--flush-l2", action="store_true")
    ap.add_argument("--extended", action="store_true")
    a = ap.parse_args(argv)
    ops = list(OPS) if a.op == "all" else list(EXTENDED_OPS) if a.op == "extended" else [a.op]
    for op in ops:
        if op not in EXTENDED_OPS:
            ap.error(f"unknown op {op!r}")
    variants = [v for v in a.variants.split(",") if v]
    for v in variants:
        if v not in VARIANTS:
            ap.error(f"unknown variant {v!r}; choose from {', '.join(VARIANTS)}")
    if a.sizes == "default":
        sizes = default_sizes()
    elif a.sizes == "gpu":
        sizes = gpu_sizes()
    else:
        try:
            sizes = [int(s) for s in a.sizes.split(",") if s]
        except ValueError:
            ap.error(f"--sizes expects integers or 'default', got {a.sizes!r}")
        if not sizes or any(s < 0 for s in sizes):
            ap.error("--sizes expects non-negative integers")
    if a.reps < 1 or a.warmup < 0:
        ap.error("--reps must be >= 1 and --warmup >= 0")
    caches = None
    if a.cache_sizes is not None:
        try:
            caches = [int(c) for c in a.cache_sizes.split(",") if c]
        except ValueError:
            ap.error(f"--cache-sizes expects integers, got {a.cache_sizes!r}")
    records = run_sweep(ops, variants, sizes, a.type, a.reps, a.warmup, a.seed, packages=a.packages,
                        flush_l2=a.flush_l2)
    try:
        emit_csv(records, a.csv, a.extended)
    except OSError as exc:
        print(f"error: cannot write CSV to {a.csv}: {exc}", file=sys.stderr)
        return 1
    if caches is not None:
        if a.csv == "-":
            print("note: --cache-sizes ignored when the CSV goes to stdout", file=sys.stderr)
            return 0
        try:
            Path(a.csv + ".meta").write_text("cache_sizes_bytes," + ",".join(map(str, caches)) + "\n")
        except OSError as exc:
            print(f"error: cannot write {a.csv}.meta: {exc}", file=sys.stderr)
            return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
