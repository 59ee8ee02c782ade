#!/usr/bin/env python
"""Summarise an ncu capture (.ncu-rep, read here with `ncu -i`) and/or a
launch list (--csv --log-file) into profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof_t2.ncu-rep \
        --launches gpurun_out/launches.csv --bytes 8589934592 --out profiles/r01_t2

Writes <out>.json (machine readable) and <out>.txt (one screen).
"""

import argparse
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_ncu_peak",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_ghz",
    "dram__cycles_elapsed.avg.per_second": "dram_clock_ghz",
}
UNITS = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Gbyte": 1e9, "Mbyte": 1e6,
         "Kbyte": 1e3, "Tbyte": 1e12, "byte": 1.0, "GB": 1e9, "MB": 1e6}


def _raw(rep):
    out = subprocess.run([os.environ.get("NCU", "ncu"), "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")}
        for metric, name in KEYS.items():
            if metric in d and d[metric] not in ("", "n/a"):
                try:
                    v = float(d[metric].replace(",", ""))
                except ValueError:
                    continue
                k[name] = v * UNITS.get(u.get(metric, ""), 1.0) if u.get(metric) in UNITS else v
        kernels.append(k)
    return kernels


def _launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = {}
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = UNITS.get(d.get("Metric Unit", "ns"), 1e-9)
        agg.setdefault(d["Kernel Name"], []).append(float(d["Metric Value"].replace(",", "")) * unit)
    total = sum(sum(v) for v in agg.values())
    return [
        {"kernel": k, "launches": len(v), "avg_s": sum(v) / len(v), "share": sum(v) / total}
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))
    ]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--bytes", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args(argv)
    res = {"note": a.note}
    lines = [a.note] if a.note else []
    if a.rep:
        ks = _raw(a.rep)
        res["kernels"] = ks
        for k in ks:
            traffic = k.get("dram_read", 0) + k.get("dram_write", 0)
            k["dram_bytes"] = traffic
            if k.get("duration"):
                k["dram_gbs"] = traffic / k["duration"] / 1e9
            if a.bytes:
                k["algorithmic_bytes"] = a.bytes
                k["traffic_over_algorithmic"] = traffic / a.bytes
                if k.get("duration"):
                    k["algorithmic_gbs"] = a.bytes / k["duration"] / 1e9
            lines.append(f"kernel: {k['kernel'][:150]}")
            for key in ("duration", "dram_read", "dram_write", "dram_bytes", "dram_gbs",
                        "algorithmic_gbs", "traffic_over_algorithmic", "dram_pct_of_ncu_peak",
                        "registers_per_thread", "grid", "achieved_occupancy_pct",
                        "sm_throughput_pct", "fp64_pipe_pct", "fp64_pipe_cycles_pct", "l2_hit_pct", "sm_clock_ghz"):
                if key in k:
                    lines.append(f"  {key:28s} {k[key]:.6g}")
        if ks:
            res["dram_bytes_per_launch"] = ks[0]["dram_bytes"]
    if a.launches:
        ls = _launches(a.launches)
        res["launch_list"] = ls
        lines.append("launch list (cold-cache, serialised; compare shares):")
        for l in ls:
            lines.append(f"  {l['launches']:4d} x {l['avg_s']*1e3:9.4f} ms  share {l['share']*100:5.1f}%  {l['kernel'][:110]}")
    open(a.out + ".json", "w").write(json.dumps(res, indent=1))
    open(a.out + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
