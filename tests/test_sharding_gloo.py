"""Multi-rank host logic on CPU: block partition, rank-ordered all-gather of
per-rank partials, gathering a sharded vector, and operand placement — with
world_size 2 over gloo (the data-path kernels themselves need a GPU and are
covered by the gpu tests)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1109_1264_b200.sharding import SHARD_ALIGN, shard_bounds


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_partition(world):
    for n in [0, 1, 63, 64, 65, 1000, 4097, 1 << 20, (1 << 31) + 5]:
        prev = 0
        for r in range(world):
            lo, hi = shard_bounds(n, world, r)
            assert lo == prev and lo <= hi
            assert lo % SHARD_ALIGN == 0 or lo == n
            prev = hi
        assert prev == n
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1109_1264_b200 as lv
        from paper_1109_1264_b200 import runtime
        from paper_1109_1264_b200.expressions import lower

        n = 1000
        full = np.arange(n, dtype=np.float64) * 0.5
        x = lv.ShardedVector.from_global(full, "f64", device="cpu")
        y = lv.ShardedVector.from_blocks(n, "f64", lambda lo, hi: full[lo:hi] * 2, device="cpu")
        lo, hi = shard_bounds(n, world, rank)
        assert (x.lo, x.hi) == (lo, hi) and len(x) == n and len(x.local) == hi - lo
        # gather of the sharded vector (collective)
        assert np.array_equal(x.to_array(), full)
        # per-rank partial {hi, lo} pairs come back in rank order on every rank
        part = torch.tensor([float(rank + 1), 1e-20 * (rank + 1)], dtype=torch.float64)
        got = x.gather_partials(part).numpy()
        want = np.array([[r + 1.0, 1e-20 * (r + 1)] for r in range(world)]).reshape(-1)
        assert np.array_equal(got, want)
        # placement resolves every operand to its local block
        lw = lower(2.0 * x + y)
        pl = runtime.Placement(lw.vectors, None, n)
        assert pl.sharded is x and pl.n == hi - lo
        assert [v is s for v, s in zip(pl.leaves, [x.local, y.local])] == [True, True]
        # mixing sharded and plain vectors is rejected
        plain = lv.DenseVector.zeros(n, "f64", device="cpu")
        with pytest.raises(TypeError):
            runtime.Placement(lower(x + plain).vectors, None, n)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}
