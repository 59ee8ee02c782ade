#!/usr/bin/env python
"""Multi-process check of the sharded path (one process per GPU, NCCL).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29531 tools/dist_check.py

Every rank builds its block of the same global vectors from the chunk-keyed
synthetic streams, evaluates an elementwise tree (no communication), a dot
and a norm2 (per-rank double-double partials -> NCCL all-gather -> fixed
rank-order finish, or the in-kernel NVLink exchange), the fused axpy->dot
and a fused CG update with a device-resident step length, and checks them against the
oracle: elementwise bit-exact on its block, reductions within 1e-12 of the
exact global value, identical on every rank.  Prints one JSON line on rank 0.
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1109_1264_b200 as lv  # noqa: E402
from oracle import coracle, restate  # noqa: E402  (checker only)
from paper_1109_1264_b200 import synth  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = (1 << 24) + 77
    mk = lambda k: (lambda lo, hi: synth.block(5, k, lo, hi, np.float64))
    X, Y, Z = (lv.ShardedVector.from_blocks(n, "f64", mk(k)) for k in range(3))
    lo, hi = X.lo, X.hi
    x, y, z = (synth.block(5, k, 0, n, np.float64) for k in range(3))
    W = lv.ShardedVector.zeros(n, "f64")
    W.assign(0.5 * X - 2.0 * (Y - Z))
    want = restate.eval_sig("S0 L0 * S1 L1 L2 - * -", [x[lo:hi], y[lo:hi], z[lo:hi]], [0.5, 2.0], "f64")
    ok_elem = W.local.to_array().tobytes() == want.tobytes()
    r = lv.dot(X, Y)
    ex = coracle.reduce_exact("L0 L1 *", [x, y], [], "f64")
    ok_dot = abs(float(r) - ex) <= 1e-12 * abs(ex)
    nr = lv.norm2(Z)
    exn = np.sqrt(coracle.reduce_exact("L0 L0 *", [z], [], "f64"))
    ok_nrm = abs(float(nr) - exn) <= 1e-12 * exn
    rr = lv.axpy_dot(0.25, X, Y, Z)
    y_new = restate.eval_sig("L0 S0 L1 * +", [y, x], [0.25], "f64")
    ex2 = coracle.reduce_exact("L0 L1 *", [y_new, z], [], "f64")
    ok_fused = abs(float(rr) - ex2) <= 1e-12 * abs(ex2) and Y.local.to_array().tobytes() == y_new[lo:hi].tobytes()
    # a CG update with a device-resident step length: one salt_fused kernel
    # per rank, total exchanged in-kernel (peer) or via the all-gather (nccl)
    a = lv.dot(X, Y, lazy=True) / lv.dot(Z, Z, lazy=True)
    av = float(a.item())
    x_new = restate.eval_sig("L0 S0 L1 * +", [x, z], [av], "f64")
    y_cg = restate.eval_sig("L0 S0 L1 * -", [y_new, x_new], [av], "f64")  # reads the new X
    cg = lv.fused((X, X + a * Z), (Y, Y - a * X), Y * Y, lazy=True)
    ex3 = coracle.reduce_exact("L0 L0 *", [y_cg], [], "f64")
    ok_cg = (abs(float(cg.item()) - ex3) <= 1e-12 * ex3
             and X.local.to_array().tobytes() == x_new[lo:hi].tobytes()
             and Y.local.to_array().tobytes() == y_cg[lo:hi].tobytes())
    # every rank must hold the identical reduction results
    mine = torch.tensor([float(r), float(nr), float(rr), float(cg.item())], dtype=torch.float64,
                        device="cuda")
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    same = all(torch.equal(v, allv[0]) for v in allv)
    flags = torch.tensor([int(bool(v)) for v in (ok_elem, ok_dot, ok_nrm, ok_fused, ok_cg, same)],
                         dtype=torch.int32, device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        res = dict(zip(["elementwise", "dot", "norm2", "axpy_dot", "cg_update_device_scalar",
                        "identical_on_ranks"],
                       [bool(v) for v in flags.tolist()]))
        res["world"] = world
        res["values"] = [float(r).hex(), float(nr).hex(), float(rr).hex(), float(cg.item()).hex()]
        from paper_1109_1264_b200 import sharding

        res["exchange"] = sharding.exchange_route()

        ex = [e for e in sharding._exchanges.values() if e is not None]
        res["peer_exchange_active"] = bool(ex)
        res["peer_epochs"] = ex[0].epoch if ex else 0
        res["ok"] = all(res[k] for k in ("elementwise", "dot", "norm2", "axpy_dot",
                                         "cg_update_device_scalar", "identical_on_ranks"))
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if bool(flags.min().item()) else 1)


if __name__ == "__main__":
    main()
