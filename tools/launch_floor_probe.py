#!/usr/bin/env python
"""Single-launch latency floor vs BASELINE config 1 (daxpy, n = 2^20 f64).

Same methodology as tools/profile_target.py --time: ~50 us of queued GPU
work (torch.cuda._sleep) so the launch is issued ahead, then CUDA events
around ONE launch; best and median of --reps.  Rows:

  empty         torch.cuda._sleep(0): an (almost) empty kernel — the
                launch/completion floor of any event-timed single kernel
  axpy_n1       lv.axpy on 1 element: the product's floor (its launch path)
  daxpy20_hot   config 1, operands L2-resident (previous call touched them)
  daxpy20_cold  config 1 after writing a 256 MiB buffer (L2 full of dirty
                lines, config_sweep's flush) — the reference-comparable case
  daxpy20_rdflush  after READING a 256 MiB buffer (L2 full of clean lines)

ideal = 24 B x 2^20 / measured HBM peak (MEASURED_PEAKS.json).
    python tools/launch_floor_probe.py > profiles/r02_launch_floor.json
"""

import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1109_1264_b200 as lv  # noqa: E402


def timed(fn, pre=None, reps=30):
    ts = []
    for _ in range(reps):
        if pre is not None:
            pre()
        torch.cuda._sleep(100_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return {"best_us": round(min(ts), 3), "median_us": round(statistics.median(ts), 3)}


def main():
    n = 1 << 20
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    x = lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda"))
    y = lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda"))
    x1 = lv.DenseVector.from_tensor(torch.rand(1, dtype=torch.float64, device="cuda"))
    y1 = lv.DenseVector.from_tensor(torch.rand(1, dtype=torch.float64, device="cuda"))
    junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        lv.axpy(1e-3, x, y)
        lv.axpy(1e-3, x1, y1)
    torch.cuda.synchronize()
    res = {"gpu": torch.cuda.get_device_name(0), "n": n, "peak_gbs": peak,
           "ideal_us": round(24 * n / peak / 1e3, 3)}
    res["empty"] = timed(lambda: torch.cuda._sleep(0))
    res["axpy_n1"] = timed(lambda: lv.axpy(1e-3, x1, y1))
    res["daxpy20_hot"] = timed(lambda: lv.axpy(1e-3, x, y))
    res["daxpy20_cold"] = timed(lambda: lv.axpy(1e-3, x, y), pre=lambda: junk.fill_(1))
    res["daxpy20_rdflush"] = timed(lambda: lv.axpy(1e-3, x, y), pre=lambda: junk.sum())
    for k in ("daxpy20_hot", "daxpy20_cold", "daxpy20_rdflush"):
        res[k]["over_ideal"] = round(res[k]["best_us"] / res["ideal_us"], 3)
        res[k]["over_floor_plus_ideal"] = round(res[k]["best_us"] / (res["axpy_n1"]["best_us"] + res["ideal_us"]), 3)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
