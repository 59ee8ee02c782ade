#!/usr/bin/env python
"""First-call latency of a tree outside the compiled-in table, cold JIT disk
cache: synchronous NVRTC build (SALT_JIT_ASYNC=0) vs the tiered path
(interpreter now, compile in the background).  Each mode runs in a fresh
process.

    python tools/jit_latency.py
"""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import time, json, torch, paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import _native
lib = _native.lib()
n = 1 << 20
v = [lv.DenseVector.from_tensor(torch.rand(n, dtype=torch.float64, device="cuda")) for _ in range(4)]
out = lv.DenseVector.zeros(n, "f64")
out.assign(v[0] + v[1]); torch.cuda.synchronize()       # CUDA context, table warm
res = {}
for name, fn in (("assign", lambda: out.assign((v[0] - v[1]) * (v[2] + v[3]) - 0.5 * v[0])),
                 ("dot", lambda: lv.dot(out - v[2], v[3]))):
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    res[name + "_first_ms"] = round((time.perf_counter() - t) * 1e3, 2)
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    res[name + "_second_ms"] = round((time.perf_counter() - t) * 1e3, 3)
lib.salt_jit_wait()
for name, fn in (("assign", lambda: out.assign((v[0] - v[1]) * (v[2] + v[3]) - 0.5 * v[0])),
                 ("dot", lambda: lv.dot(out - v[2], v[3]))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    res[name + "_compiled_ms"] = round((time.perf_counter() - t) * 1e3, 3)
res["interp_launches"] = lib.salt_interp_launch_count()
print(json.dumps(res))
"""


def main():
    rows = {}
    for mode in ("0", "1"):
        env = dict(os.environ, SALT_JIT_CACHE="off", SALT_JIT_ASYNC=mode, PYTHONPATH=str(ROOT))
        out = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env,
                             cwd=ROOT, timeout=600)
        rows["tiered" if mode == "1" else "synchronous"] = (json.loads(out.stdout.strip().splitlines()[-1])
                                                           if out.returncode == 0 else out.stderr[-500:])
    print(json.dumps({"what": "first-call latency of fresh trees (n = 2^20 f64), cold JIT cache", **rows},
                     indent=1))


if __name__ == "__main__":
    main()
