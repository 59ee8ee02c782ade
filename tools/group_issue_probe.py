#!/usr/bin/env python
"""Cross-device issue skew of the single-process multi-GPU path
(devicegroup.py): G launches of config 4's e-tree block, issued

  serial      from one host thread, one salt_fused per member in turn (the
              round-1 DeviceGroup loop, C ABI calls only — no Python
              lowering counted);
  group       by salt_group_fused: one persistent host thread per member,
              all released at once (csrc/salt_abi_group.inc).

Skew = (last member's issue end) - (first member's issue end) per call, in
us; p50 / p99 over the calls.  With one GPU every member uses device 0 on
its own stream (all members then share one CUDA context, whose launch path
is partly serialised — an upper bound for G separate devices).  The budget
the skew is judged against: 2 % of config 4's per-device block at G = 8
(2^30 f32 e-tree / 8 = 2.5 GiB at ~6.5 TB/s = ~0.41 ms).

    python tools/group_issue_probe.py --members 8 --calls 200 > profiles/r02_group_issue.json
"""

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1109_1264_b200 import _native  # noqa: E402

SIG = "S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +"  # config 4: al*(a+b) - be*(c-d) + ga*a


def pct(xs, q):
    return float(np.percentile(np.asarray(xs), q))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=8)
    ap.add_argument("--calls", type=int, default=200)
    ap.add_argument("--n", type=int, default=(1 << 30) // 8)
    a = ap.parse_args()
    G, n = a.members, a.n
    lib = _native.lib()
    dev = torch.device("cuda", 0)
    streams = [torch.cuda.Stream(device=dev) for _ in range(G)]
    vecs = [[torch.rand(n, dtype=torch.float32, device=dev) for _ in range(4)] for _ in range(G)]
    outs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(G)]
    scal = [1.25, -0.5, 0.75]
    sp, ks = _native.double_array(scal)
    # ---- serial: one thread, G C-ABI calls
    per_member = []
    for g in range(G):
        lp, k1 = _native.ptr_array([t.data_ptr() for t in vecs[g]])
        dp, k2 = _native.ptr_array([outs[g].data_ptr()])
        per_member.append((lp, dp, k1, k2, streams[g].cuda_stream))
    serial = []
    for c in range(a.calls + 5):
        ends = []
        t0 = time.perf_counter_ns()
        for lp, dp, _k1, _k2, st in per_member:
            _native.check(lib.salt_fused(_native.SALT_F32, SIG.encode(), None, dp, 1, lp, 4, sp, 3, None, 0,
                                         n, 0, None, 0, None, None, st))
            ends.append(time.perf_counter_ns() - t0)
        if c >= 5:
            serial.append((ends[-1] - ends[0]) / 1e3)
        if c % 20 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    # ---- group: persistent member threads
    devs = (ctypes.c_int * G)(*([0] * G))
    grp = ctypes.c_void_p()
    _native.check(lib.salt_group_create(G, ctypes.addressof(devs), ctypes.addressof(grp)))
    dsts, kd = _native.ptr_array([o.data_ptr() for o in outs])
    leaves, kl = _native.ptr_array([t.data_ptr() for g in range(G) for t in vecs[g]])
    ns, kn = _native.i64_array([n] * G)
    strs, kst = _native.ptr_array([s.cuda_stream for s in streams])
    group, group_start, call_us = [], [], []
    st = (ctypes.c_int64 * G)()
    en = (ctypes.c_int64 * G)()
    for c in range(a.calls + 5):
        t0 = time.perf_counter_ns()
        _native.check(lib.salt_group_fused(grp, _native.SALT_F32, SIG.encode(), None, dsts, 1, leaves, 4, sp, 3,
                                           None, 0, ns, 0, None, 0, None, strs))
        t1 = time.perf_counter_ns()
        _native.check(lib.salt_group_issue_times(grp, ctypes.addressof(st), ctypes.addressof(en)))
        if c >= 5:
            group.append((max(en) - min(en)) / 1e3)
            group_start.append((max(st) - min(st)) / 1e3)
            call_us.append((t1 - t0) / 1e3)
        if c % 20 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    lib.salt_group_destroy(grp)
    # correctness of the group launch: every member's result equals a serial one
    ref = torch.empty_like(outs[0])
    lp, dp, *_ = per_member[G - 1]
    rp, kr = _native.ptr_array([ref.data_ptr()])
    _native.check(lib.salt_fused(_native.SALT_F32, SIG.encode(), None, rp, 1, lp, 4, sp, 3, None, 0, n, 0,
                                 None, 0, None, None, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    same = bool(torch.equal(ref, outs[G - 1]))
    block_ms = 20.0 * n / 6547.2e9 * 1e3
    res = {
        "members": G, "n_per_member": n, "calls": a.calls, "gpu": torch.cuda.get_device_name(0),
        "block_ms_at_measured_peak": round(block_ms, 4),
        "budget_us_2pct": round(0.02 * block_ms * 1e3, 2),
        "serial_skew_us": {"p50": pct(serial, 50), "p99": pct(serial, 99)},
        "group_skew_end_us": {"p50": pct(group, 50), "p99": pct(group, 99)},
        "group_skew_start_us": {"p50": pct(group_start, 50), "p99": pct(group_start, 99)},
        "group_call_us": {"p50": pct(call_us, 50), "p99": pct(call_us, 99)},
        "group_result_equals_serial": same,
        "note": "all members on device 0 (one context): an upper bound for G devices",
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
