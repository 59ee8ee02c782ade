#!/usr/bin/env python
"""PCIe ceiling on this box: pinned H2D / D2H / bidirectional copy bandwidth
with torch (cudaMemcpyAsync), for sizing the end-to-end (host vector) path."""

import json
import time

import torch


def bw(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    return nbytes / min(t) / 1e9


def main():
    res = {}
    for mb in (64, 256, 1024):
        n = mb << 20
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def both():
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            s1.synchronize()
            s2.synchronize()

        def two_h2d():
            half = n // 2
            with torch.cuda.stream(s1):
                d[:half].copy_(h[:half], non_blocking=True)
            with torch.cuda.stream(s2):
                d[half:].copy_(h[half:], non_blocking=True)
            s1.synchronize()
            s2.synchronize()

        res[f"{mb}MiB"] = {
            "h2d_gbs": round(bw(lambda: d.copy_(h, non_blocking=True), n), 2),
            "d2h_gbs": round(bw(lambda: h2.copy_(d2, non_blocking=True), n), 2),
            "h2d_two_streams_gbs": round(bw(two_h2d, n), 2),
            "bidirectional_total_gbs": round(bw(both, 2 * n), 2),
        }
    # The end-to-end step's shape with no kernel at all: 3 bytes up for every
    # byte down (T2: a, b, c in; d out), both directions at once, in 8 chunks
    # so the D2H of chunk k overlaps the H2D of chunk k+1 — the ceiling of
    # bench.py's e2e number.
    n = 768 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(n // 3, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    do = torch.empty(n // 3, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def mix():
        k, ko = n // 8, n // 24
        evs = []
        for c in range(8):
            with torch.cuda.stream(s1):
                d[c * k:(c + 1) * k].copy_(h[c * k:(c + 1) * k], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
            s2.wait_event(e)
            with torch.cuda.stream(s2):
                ho[c * ko:(c + 1) * ko].copy_(do[c * ko:(c + 1) * ko], non_blocking=True)
            evs.append(e)
        s1.synchronize()
        s2.synchronize()

    res["t2_shape_3up_1down"] = {
        "effective_gbs": round(bw(mix, n + n // 3), 2),
        "note": "768 MiB H2D + 256 MiB D2H per step in 8 chunks, D2H of chunk k overlapping H2D "
                "of chunk k+1; no kernel: the ceiling of the e2e path",
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
