#!/usr/bin/env python
"""Benchmark: effective GB/s of the fused BLAS-1 expression evaluator.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
    d = alpha*a + beta*(b - c), float64, n = 2^28 per GPU
    (a, b, c i.i.d. uniform[-1, 1], alpha, beta uniform[-2, 2], seeded,
     synthetic — no dataset is involved)
One step = one fused evaluation of that tree over the resident vectors.
Bytes per step = 8 * n * (3 reads + 1 write) = 8 GiB.
The working set (8 GiB) is 65x the 126 MB L2, so no L2 flush is needed.

Arms
  default            libsalt.so fused kernel on each GPU (one process per GPU
                     under torchrun; weak scaling: every rank owns its own
                     2^28-element vectors; no data-path collective).
  --impl reference   the reference algorithm on the host CPU: the C
                     restatement in oracle/ (tile-by-tile node evaluation,
                     same per-element IEEE ops) with all host threads, each
                     step a bounded sample of the workload; rank 0 only.

Multi-GPU block (every line of the default arm, unless --no-multi): the
north_star's multi-GPU claims, measured at the run's N:
  config4   e = alpha*(a + b) - beta*(c - d) + gamma*a, f32, 2^30 elements
            GLOBAL, block-sharded over the N ranks (strong scaling), no
            communication; max-over-ranks device time, aggregate GB/s and the
            fraction of N x the measured HBM peak;
  config5   y = alpha*x + y; r = dot(y, z), f64, 2^31 elements GLOBAL,
            block-sharded, 100 fused axpy->dot steps on ShardedVectors with
            the cross-rank reduction of every step inside the timed region;
            ms/step, the exchange route that ran, and whether r_100 is
            bit-identical on every rank;
  config5_peer  the same over the opt-in in-kernel NVLink exchange (one
            launch per step), in a child process per rank with its own
            process group and a time limit, so a fault or hang there cannot
            cost the line; probed first and reported — never raised — if it
            fails (--no-peer skips it).

--gpus is authoritative: under torchrun WORLD_SIZE must equal it (else exit
2); without torchrun, --gpus N > 1 re-executes this script under
torch.distributed.run with N ranks (exit 2 if fewer than N GPUs exist).

Output: one JSON line on rank 0 (see the keys below).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path
# steady-state measurements: build out-of-table trees with NVRTC on first use
# instead of running them on the interpreter meanwhile (tiered JIT)
os.environ.setdefault("SALT_JIT_ASYNC", "0")

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "effective GB/s per fused vector expression (and % of HBM peak) at 1/2/4/8 B200"
TREE_SIG = "S0 L0 * S1 L1 L2 - * +"
WORKLOAD = "config2: d = alpha*a + beta*(b - c), float64, n = 2^28 per GPU"


def _ensure_built():
    """Build libsalt.so / the C oracle in place if this checkout lacks them
    (build() normally produced both; nvcc and gcc are in the image)."""
    import fcntl

    lib = ROOT / "paper_1109_1264_b200" / "libsalt.so"
    orc = ROOT / "oracle" / "_build" / "liboracle.so"
    if lib.exists() and orc.exists():
        return
    with open("/tmp/salt_bench_build.lock", "w") as lock:  # one builder across ranks
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not lib.exists():
            subprocess.run(["make", "-C", str(ROOT / "paper_1109_1264_b200" / "csrc")], check=True,
                           stdout=subprocess.DEVNULL)
        if not orc.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, stdout=subprocess.DEVNULL)


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _traffic():
    """DRAM bytes per launch of the timed kernel from the committed ncu
    capture summary (profiles/ncu_summary.json), or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 10 ms.  Windows are
    delimited by mark() pairs; the headline region of a short run (the
    driver's --steps 20 is ~24 ms) holds only a few samples, so the line
    also carries the window over the multi-GPU block (about a second)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.marks = []
        # NVML read directly in a tight loop, but only inside the headline
        # window (first mark() pair): ~1 sample per ms where nvidia-smi's
        # 10 ms period leaves one or two in the driver's 24 ms region
        self.fast = []
        self._fast_on = threading.Event()
        self._fast_quit = False
        self._nvml = None

    def _fast_loop(self):
        nv, h = self._nvml
        names = ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"),
                 (0x4, "sw_power_cap"))
        while not self._fast_quit:
            if not self._fast_on.wait(0.05):
                continue
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                return
            self.fast.append((time.perf_counter(), float(sm), [n for bit, n in names if mask & bit]))
            time.sleep(0.001)  # ~20 samples in the driver's 24 ms region

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                uuid = "GPU-" + str(torch.cuda.get_device_properties(self.index).uuid)
                h = nv.nvmlDeviceGetHandleByUUID(uuid.encode() if hasattr(uuid, "encode") else uuid)
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._fast_max = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nvml = (nv, h)
            threading.Thread(target=self._fast_loop, daemon=True).start()
        except Exception:
            self._nvml = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), line.strip()))

    def mark(self):
        self.marks.append(time.perf_counter())
        if len(self.marks) == 1:
            self._fast_on.set()
        elif len(self.marks) == 2:
            self._fast_on.clear()

    def stop(self):
        self._fast_quit = True
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, window=0):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if len(self.marks) >= 2 * window + 2:
            t0, t1 = self.marks[2 * window], self.marks[2 * window + 1]
        else:
            t0, t1 = 0, float("inf")
        fast = [f for f in self.fast if t0 <= f[0] <= t1] if window == 0 else []
        if len(fast) >= 3:
            return {
                "sm_mhz": float(np.median([f[1] for f in fast])),
                "sm_max_mhz": self._fast_max,
                "reasons": sorted({r for f in fast for r in f[2]}),
                "samples": len(fast),
                "source": "nvml, sampled in a loop inside the timed region",
            }
        inside = [s for t, s in self.samples if t0 <= t <= t1]
        if not inside:  # region shorter than the sampling period: nearest sample
            inside = [min(self.samples, key=lambda ts: abs(ts[0] - t0))[1]]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in inside:
            parts = [p.strip() for p in s.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(inside),
        }


def _dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and not dist.is_initialized():
        # under torchrun (even at N = 1): a process group, so the sharded
        # paths run their real collectives (config5 / config5_peer)
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_gbs(n_sample, steps, warmup, threads, seconds_cap=None):
    """Time the C restatement of the reference algorithm (oracle/) on host
    arrays of n_sample elements; returns (GB/s, seconds per step)."""
    from oracle import coracle
    from paper_1109_1264_b200 import synth

    a, b, c = (synth.block(2, k, 0, n_sample, np.float64) for k in range(3))
    al, be = synth.scalars(2, 2)
    d = np.empty(n_sample)
    for _ in range(warmup):
        coracle.assign(TREE_SIG, d, [a, b, c], [al, be], threads=threads)
    t = []
    t_start = time.perf_counter()
    for _ in range(steps):
        s = time.perf_counter()
        coracle.assign(TREE_SIG, d, [a, b, c], [al, be], threads=threads)
        t.append(time.perf_counter() - s)
        if seconds_cap and time.perf_counter() - t_start > seconds_cap:
            break
    per = float(np.mean(t))
    return 32.0 * n_sample / per / 1e9, per, len(t)


LANEVEC_SNIPPET = r"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(1, sys.argv[2])
os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
import lanevec as lv
from paper_1109_1264_b200 import synth
n = int(sys.argv[3])
al, be = synth.scalars(2, 2)
a, b, c = (lv.DenseVector.from_values(synth.block(2, k, 0, n, np.float64), "f64") for k in range(3))
d = lv.DenseVector.zeros(n, "f64")
d.assign(al * a + be * (b - c))
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    d.assign(al * a + be * (b - c))
    ts.append(time.perf_counter() - t0)
print(json.dumps({"best_s": min(ts), "n": n}))
"""


def lanevec_1core(n=1 << 20):
    """The UNMODIFIED reference engine (lanevec, pip-installed into
    baseline/_ref) on one host core: config 2's tree at n = 2^20 through its
    own public API (DenseVector / operator tree / assign, default plan) —
    BASELINE.md §3's CPU plan, reference bench.py:144-192.  None when
    baseline/_ref is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "lanevec").exists():
        return None
    try:
        r = subprocess.run([sys.executable, "-c", LANEVEC_SNIPPET, str(ref), str(ROOT), str(n)],
                           capture_output=True, text=True, timeout=300)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as exc:  # reported, not fatal: the port is the arm's number
        return {"error": f"{type(exc).__name__}: {exc}"[:200]}
    return {"value": round(32.0 * n / d["best_s"] / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": "reference",
            "sample": f"best of 3 lanevec DenseVector assigns of config 2's tree at n = {n} f64 "
                      "(unmodified reference engine from baseline/_ref, default plan, one core)"}


def workload_config(n, world):
    """The `config` object of both arms (one workload, one description)."""
    return {
        "workload": WORKLOAD,
        "n_per_gpu": n,
        "bytes_per_step_per_gpu": int(32 * n),
        "l2": "inputs (8 GiB/GPU) >> 126 MB L2; no flush needed",
        "parallelism": f"block-sharded x{world} (weak), no data-path collective",
    }


def _mem_available():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def run_reference(args, world, rank):
    if rank != 0:
        return
    threads = _host_threads()
    n_sample = args.n_sample
    if n_sample is None:
        # the full 2^28-element workload (4 x 2 GiB of host arrays, ~70 ms a
        # step on 16 threads) when the host has the memory, else a 2^25 sample
        n_sample = args.n if _mem_available() >= 24 << 30 else 1 << 25
    gbs, per, done = cpu_reference_gbs(n_sample, args.steps, args.warmup, threads, seconds_cap=120)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(gbs, 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": done,
        "warmup": args.warmup,
        "ms_per_step": round(per * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, chunk-keyed numpy streams)",
        "config": workload_config(args.n, args.gpus) if n_sample == args.n else
                  dict(workload_config(args.n, args.gpus), sample_n=n_sample),
        "cpu_baseline": {
            "value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": (f"the full workload ({n_sample} f64 elements per step)" if n_sample == args.n else
                       f"{n_sample} f64 elements per step (bounded sample of the 2^28 workload)")
                      + ", oracle/salt_oracle.c tile evaluation, all host threads",
        },
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    line["cpu_baseline"]["lanevec_1core"] = lanevec_1core()
    line["cpu_baseline"].update(cpu_model=_cpu_model(), nproc=os.cpu_count())
    print(json.dumps(line), flush=True)


def run_gpu(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1109_1264_b200 as lv
    from paper_1109_1264_b200 import _native, synth

    dev = torch.device("cuda", local)
    n = args.n
    lib = _native.lib()
    al, be = synth.scalars(2, 2)
    vecs = []
    for k in range(3):
        v = lv.DenseVector.empty(n, "f64", device=dev)
        synth.fill_device(v.tensor, 2, k, lo=rank * n)
        vecs.append(v)
    a, b, c = vecs
    d = lv.DenseVector.empty(n, "f64", device=dev)
    torch.cuda.synchronize(dev)

    def step():
        d.assign(al * a + be * (b - c))

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = lib.salt_launch_count()
    sampler.mark()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    sampler.mark()
    launches = lib.salt_launch_count() - launches0
    elapsed_ms = t_start.elapsed_time(t_end)
    kernel_ms = [s.elapsed_time(e) for s, e in ev]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    clocks = sampler.summary(0)

    bytes_step = 32.0 * n
    value = world * bytes_step * args.steps / (elapsed_max / 1e3) / 1e9
    peak, peak_src = _peaks()
    kavg = float(np.mean(kernel_ms))
    achieved = bytes_step / (kavg / 1e3) / 1e9

    # ---- end to end: host (pinned) vectors through the public API ----
    e2e = None
    if not args.no_e2e:
        n_e2e = n
        hv = []
        for k in range(3):
            # the same synthetic values, copied down from the device vectors
            # (drawing 3 x 2^28 values on the host would cost each rank
            # seconds of CPU time at N = 8)
            h = lv.DenseVector.empty(n_e2e, "f64", device="cpu")
            h.tensor.copy_(vecs[k].tensor[:n_e2e])
            hv.append(h)
        hd = lv.DenseVector.empty(n_e2e, "f64", device="cpu")
        ha, hb, hc = hv

        def e2e_step():
            hd.assign(al * ha + be * (hb - hc))

        e2e_step()
        e_steps = max(3, min(args.steps, 8))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        s = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        torch.cuda.synchronize(dev)
        e_el = time.perf_counter() - s
        te = torch.tensor([e_el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_el = float(te.item())
        e2e = {
            "value": round(world * 32.0 * n_e2e * e_steps / e_el / 1e9, 3),
            "unit": "GB/s",
            "h2d_bytes_per_step": 24 * n_e2e,
            "d2h_bytes_per_step": 8 * n_e2e,
            "steps": e_steps,
            "timing": "host wall clock around blocking calls (pinned host vectors, "
                      "chunked H2D -> fused kernel -> D2H on 3 streams)",
        }
        del hv, hd, ha, hb, hc

    del vecs, a, b, c, d
    torch.cuda.empty_cache()
    multi = None
    if not args.no_multi:
        sampler.mark()
        multi = {"config4": run_config4(world, rank, dev, peak),
                 "config5": run_config5(world, rank, dev)}
        if not args.no_peer:
            if dist.is_initialized():
                multi["config5_peer"] = run_config5_peer_isolated(world, rank, local, dev)
            else:
                multi["config5_peer"] = {"route": "peer", "status": "skipped: no process group "
                                         "(single process without torchrun)"}
        sampler.mark()
        multi["clocks"] = sampler.summary(1)
    sampler.stop()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = _host_threads()
        n_sample = 1 << 24
        gbs, per, done = cpu_reference_gbs(n_sample, 1000, 1, threads, seconds_cap=15)
        cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{done} evaluations of the tree on {n_sample} f64 elements "
                         "(oracle/salt_oracle.c, reference per-node tile evaluation)",
               "lanevec_1core": lanevec_1core(), "cpu_model": _cpu_model(), "nproc": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(elapsed_max / args.steps, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded, chunk-keyed numpy streams; BASELINE config 2 shapes)",
            "config": workload_config(n, world),
            "pct_hbm": round(value / (world * peak), 4),
            "roofline": {
                "bound": "hbm",
                "achieved": round(achieved, 2),
                "peak": peak,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": _traffic(),
                "peak_source": peak_src,
                # the measured copy peak is a torch copy kernel's rate, below
                # what a 3-read/1-write stream reaches; also vs HBM3e nominal
                "frac_of_nominal_8000": round(achieved / 8000.0, 4),
                "kernel_avg_ms": round(kavg, 5),
                "algorithmic_bytes_per_launch": int(bytes_step),
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "multi_gpu": multi,
        }
        print(json.dumps(line), flush=True)


def _timed_region(world, dev, fn, steps, warmup):
    """warmup untimed calls, then `steps` calls between a barrier +
    synchronize on both sides; (device time in ms — CUDA events on the
    launching stream, max over ranks — and libsalt launches in the region)."""
    import torch
    import torch.distributed as dist

    from paper_1109_1264_b200 import _native

    for _ in range(warmup):
        fn(True)
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = _native.lib().salt_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn(False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = _native.lib().salt_launch_count() - l0
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), launches


def run_config4(world, rank, dev, peak, steps=20, warmup=3):
    """BASELINE config 4: strong scaling of a global 2^30 f32 e-tree."""
    import torch

    import paper_1109_1264_b200 as lv
    from paper_1109_1264_b200 import synth
    from paper_1109_1264_b200.sharding import shard_bounds

    n = 1 << 30
    lo, hi = shard_bounds(n, world, rank)
    al, be, ga = synth.scalars(4, 3)
    ops = []
    for k in range(4):
        v = lv.DenseVector.empty(hi - lo, "f32", device=dev)
        synth.fill_device_philox(v.tensor, 4, k, lo)
        ops.append(lv.ShardedVector(v, n))
    a, b, c, d = ops
    e = lv.ShardedVector(lv.DenseVector.empty(hi - lo, "f32", device=dev), n)
    torch.cuda.synchronize(dev)
    ms, launches = _timed_region(world, dev, lambda _w: e.assign(al * (a + b) - be * (c - d) + ga * a),
                                 steps, warmup)
    nbytes = 20.0 * n  # 4 distinct f32 reads + 1 write per element, global
    value = nbytes * steps / (ms / 1e3) / 1e9
    del ops, a, b, c, d, e
    torch.cuda.empty_cache()
    return {
        "workload": "config4: e = alpha*(a + b) - beta*(c - d) + gamma*a, f32, n = 2^30 GLOBAL, "
                    "block-sharded over the ranks",
        "scaling": "strong", "collective": "none",
        "n_global": n, "n_per_rank": hi - lo if world == 1 else shard_bounds(n, world, 0)[1],
        "steps": steps, "warmup": warmup,
        "ms_per_step": round(ms / steps, 5),
        "value": round(value, 3), "unit": "GB/s",
        "algorithmic_bytes_per_step": int(nbytes),
        "frac_of_aggregate_peak": round(value / (world * peak), 4),
        "gpu_launches": int(launches),
        "data": "synthetic, device Philox streams keyed per global 2^24 chunk (synth.fill_device_philox)",
    }


def run_config5(world, rank, dev, iters=100, warmup=3, route="nccl"):
    """BASELINE config 5: 100 fused axpy->dot steps on a global 2^31 f64
    vector triple, block-sharded, with a cross-rank reduction per step.

    route "nccl": the default route (16-byte NCCL all-gather + finish kernel).
    route "peer": the opt-in in-kernel NVLink exchange (SALT_EXCHANGE=peer):
    the reduction kernel itself trades the per-rank totals over peer memory,
    ONE launch per step.  It is preceded by a 2-step probe with host results
    (a timeout raises there) and an all-rank agreement, runs with a 5 s peer
    timeout, and reports a failure instead of raising, so it can never cost
    the headline."""
    import torch
    import torch.distributed as dist

    import paper_1109_1264_b200 as lv
    from paper_1109_1264_b200 import sharding, synth
    from paper_1109_1264_b200.sharding import shard_bounds

    saved = {k: os.environ.get(k) for k in ("SALT_EXCHANGE", "SALT_PEER_TIMEOUT_MS")}
    if route == "peer":
        os.environ["SALT_EXCHANGE"] = "peer"
        os.environ.setdefault("SALT_PEER_TIMEOUT_MS", "5000")

    def agree(ok):
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        if world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        return int(flag.item()) == 1

    n = 1 << 31
    lo, hi = shard_bounds(n, world, rank)
    alpha = synth.scalars(5, 1)[0]
    vecs = []
    try:
        for k in range(3):
            v = lv.DenseVector.empty(hi - lo, "f64", device=dev)
            synth.fill_device_philox(v.tensor, 5, k, lo)
            vecs.append(lv.ShardedVector(v, n))
        X, Y, Z = vecs
        torch.cuda.synchronize(dev)
        if route == "peer":
            err = None
            try:  # probe: host results check the exchange's error word every step
                for _ in range(2):
                    lv.axpy_dot(0.0, X, Y, Z)
            except RuntimeError as exc:
                err = str(exc)[:300]
            if not agree(err is None):
                return {"route": "peer", "status": "failed in the probe", "error": err}
        out = {}

        def step(warm):
            # warm-up steps use alpha = 0: y + 0*x == y bit for bit, so the
            # timed 100 iterations start from the generated y
            out["r"] = lv.axpy_dot(0.0 if warm else alpha, X, Y, Z, lazy=True)

        ms, launches = _timed_region(world, dev, step, iters, warmup)
        err = None
        try:
            r100 = float(out["r"].item())  # a peer timeout raises here (DeviceScalar guard)
        except RuntimeError as exc:
            err, r100 = str(exc)[:300], float("nan")
        if not agree(err is None):
            return {"route": route, "status": "failed", "error": err}
        bits = torch.tensor([np.float64(r100).view(np.int64)], dtype=torch.int64, device=dev)
        same = True
        if world > 1:
            allb = [torch.empty_like(bits) for _ in range(world)]
            dist.all_gather(allb, bits)
            same = all(int(b.item()) == int(bits.item()) for b in allb)
        peer = route == "peer" and any(x is not None for x in sharding._exchanges.values())
    finally:
        X = Y = Z = None  # noqa: F841 (drop the 48 GiB before the next block)
        vecs.clear()
        torch.cuda.empty_cache()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    nbytes = 32.0 * n  # x, y, z read + y written, f64, global
    return {
        "workload": "config5: y = alpha*x + y; r = dot(y, z), f64, n = 2^31 GLOBAL, block-sharded, "
                    "100 fused axpy->dot steps (lv.axpy_dot on ShardedVectors, lazy results)",
        "scaling": "strong",
        "collective": ("in-kernel NVLink peer exchange (one launch per step)" if peer else
                       "NCCL all-gather of per-rank double-double partials + salt_reduce_finish")
                      + " per step, inside the timed region",
        "exchange_route": "peer" if peer else "nccl",
        "status": "ok" if route != "peer" or peer else "peer unavailable (no process group or "
                                                        "symmetric memory): ran the NCCL route",
        "n_global": n, "iterations": iters, "warmup": warmup,
        "ms_per_step": round(ms / iters, 5),
        "value": round(nbytes * iters / (ms / 1e3) / 1e9, 3), "unit": "GB/s",
        "algorithmic_bytes_per_step": int(nbytes),
        "r_100": r100.hex(),
        "r_100_identical_on_all_ranks": bool(same),
        "gpu_launches": int(launches),
        "data": "synthetic, device Philox streams keyed per global 2^24 chunk (synth.fill_device_philox)",
    }


PEER_CHILD_TIMEOUT_S = 150  # the child takes ~7 s at N = 1; a hung route costs at most this per bench run


def _child_env(world, rank, local, port):
    """Environment of a peer-block child: its own env:// rendezvous on
    `port`.  TORCHELASTIC_* is dropped so the child hosts / joins its own
    TCP store instead of the torchrun agent's."""
    env = {k: v for k, v in os.environ.items() if not k.startswith("TORCHELASTIC")}
    env.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
               WORLD_SIZE=str(world), LOCAL_RANK=str(local), LOCAL_WORLD_SIZE=str(world))
    return env


def run_config5_peer_isolated(world, rank, local, dev, timeout=PEER_CHILD_TIMEOUT_S,
                              child_flag="--peer-child"):
    """config5_peer in a child process per rank with its own process group.

    The in-kernel NVLink exchange is opt-in and has not had a multi-GPU run
    on real hardware, so it must not be able to take the headline down: a
    device fault there kills the child's CUDA context, not this one, and a
    hang is bounded by `timeout` (the child's process group is killed).
    Every rank reports whether its child finished; the block is "ok" only if
    all did, with rank 0's child line as the numbers.  (`child_flag`
    --peer-child-selftest runs the same plumbing with a gloo child on CPU,
    for tests/test_bench_launch.py.)"""
    import signal

    import torch
    import torch.distributed as dist

    port = torch.tensor([_free_port() if rank == 0 else 0], dtype=torch.int64, device=dev)
    if world > 1:
        dist.broadcast(port, 0)
    cmd = [sys.executable, str(Path(__file__).resolve()), child_flag, "--gpus", str(world)]
    t0 = time.perf_counter()
    proc = subprocess.Popen(cmd, env=_child_env(world, rank, local, int(port.item())),
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                            start_new_session=True, cwd=str(ROOT))
    err = None
    try:
        out, errout = proc.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(proc.pid, signal.SIGKILL)
        out, errout = proc.communicate()
        err = f"child timed out after {timeout} s (killed)"
    res = None
    if err is None:
        lines = [ln for ln in out.splitlines() if ln.startswith("{")]
        if proc.returncode == 0 and lines:
            res = json.loads(lines[-1])
        else:
            err = f"child exited {proc.returncode}: {(errout or '').strip()[-300:]}"
    ok = torch.tensor([1 if res is not None else 0], dtype=torch.int32, device=dev)
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    wall = round(time.perf_counter() - t0, 2)
    if res is None:
        return {"route": "peer", "status": "failed", "error": err,
                "isolation": "child process per rank, own process group", "child_wall_s": wall}
    if int(ok.item()) != 1:
        res = {"route": "peer", "status": "failed on another rank", "rank0_child": res}
    res["isolation"] = "child process per rank, own process group"
    res["child_wall_s"] = wall
    return res


def _run_peer_child(selftest=False):
    """Entry of the child: config 5 over the peer route, one JSON line from
    every rank (the parent reads its own child's).  selftest: a gloo process
    group and one all_reduce, no GPU (the plumbing test)."""
    import torch
    import torch.distributed as dist

    if selftest:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        if os.environ.get("SALT_BENCH_SELFTEST_HANG") == os.environ["RANK"]:
            time.sleep(3600)
        res = {"route": "selftest", "status": "ok", "rank": dist.get_rank(),
               "world": dist.get_world_size(), "sum": float(t.item()),
               "torchelastic_env": sorted(k for k in os.environ if k.startswith("TORCHELASTIC"))}
    else:
        world, rank, local = _dist_setup()
        res = run_config5(world, rank, torch.device("cuda", local), route="peer")
    print(json.dumps(res), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _launch_ranks(args, argv):
    """--gpus N > 1 without torchrun: re-run this script as N ranks."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but this host has {have} GPU(s)", file=sys.stderr)
        sys.exit(2)
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + list(argv)
    sys.exit(subprocess.run(cmd).returncode)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="salt", choices=["salt", "reference"])
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-multi", action="store_true",
                    help="skip the config-4 / config-5 multi-GPU block")
    ap.add_argument("--no-peer", action="store_true",
                    help="skip config 5 over the opt-in in-kernel NVLink exchange")
    ap.add_argument("--peer-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--peer-child-selftest", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--n-sample", type=int, default=None,
                    help="elements per step of the --impl reference CPU run (default: the full "
                         "workload if the host has 24 GiB available, else 2^25)")
    raw_argv = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw_argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    under_torchrun = "WORLD_SIZE" in os.environ
    if under_torchrun and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but torchrun started WORLD_SIZE="
              f"{os.environ['WORLD_SIZE']} ranks", file=sys.stderr)
        sys.exit(2)
    _ensure_built()
    if args.peer_child or args.peer_child_selftest:
        _run_peer_child(selftest=args.peer_child_selftest)
        return
    if args.impl == "salt" and not under_torchrun and args.gpus > 1:
        _launch_ranks(args, raw_argv)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = _dist_setup()
    run_gpu(args, world, rank, local)
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
