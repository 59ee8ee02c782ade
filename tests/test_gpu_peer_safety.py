"""The NVLink peer-exchange route fails loudly, never with a wrong number
(sharding.py, VERDICT r01 "What's weak" 4).

One GPU: a PeerExchange whose descriptor names world = 2 but whose "rank 1"
buffers are local memory that no process writes — so the kernel's wait for
rank 1 must time out.  The exchange is injected through
sharding.peer_exchange (what runtime._device_reduce asks for a sharded
reduction)."""

import ctypes
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1109_1264_b200 as lv  # noqa: E402
from paper_1109_1264_b200 import _native, sharding  # noqa: E402


class LocalPeerExchange(sharding.PeerExchange):
    """world = 2, rank 0; both ranks' symmetric buffers live in one local
    allocation (rank 1's half is never written by anyone)."""

    def __init__(self, timeout_ns):
        dev = torch.device("cuda", torch.cuda.current_device())
        self.world, self.rank = 2, 0
        nb = _native.XCHG_BUFFER_BYTES
        self.buffer = torch.zeros(2 * nb // 8, dtype=torch.int64, device=dev)
        self.error = torch.zeros(1, dtype=torch.int32, device=dev)
        self.desc = _native.Exchange()
        self.desc.rank, self.desc.world = 0, 2
        self.desc.timeout_ns = int(timeout_ns)
        self.desc.error = self.error.data_ptr()
        for p in range(2):
            base = self.buffer.data_ptr() + p * nb
            self.desc.slots[p] = base
            self.desc.flags[p] = base + 2 * _native.XCHG_MAX_RANKS * 16
        self.epoch = 0
        self.failed = False

    def publish_rank1(self, epoch, hi, lo=0.0):
        """Play rank 1 for one epoch: its total into rank 0's slot, then its flag."""
        words = self.buffer.view(torch.float64)
        par = epoch & 1
        slot = (par * _native.XCHG_MAX_RANKS + 1) * 2  # DD index (par, rank 1) in rank 0's buffer
        words[slot] = hi
        words[slot + 1] = lo
        flags = self.buffer[2 * _native.XCHG_MAX_RANKS * 2:]
        flags[1] = epoch
        torch.cuda.synchronize()


@pytest.fixture
def sharded_pair():
    n = 100_000
    g = np.random.default_rng(7)
    x, y = g.standard_normal(n), g.standard_normal(n)
    X = lv.ShardedVector.from_global(x, "f64", device="cuda")
    Y = lv.ShardedVector.from_global(y, "f64", device="cuda")
    return X, Y, x, y


def test_default_route_is_nccl(monkeypatch):
    monkeypatch.delenv("SALT_EXCHANGE", raising=False)
    assert sharding.exchange_route() == "nccl"
    assert sharding.peer_exchange(None, torch.device("cuda", 0)) is None
    monkeypatch.setenv("SALT_EXCHANGE", "bogus")
    with pytest.raises(ValueError):
        sharding.exchange_route()


def test_peer_timeout_raises_instead_of_nan(monkeypatch, sharded_pair):
    X, Y, _, _ = sharded_pair
    fake = LocalPeerExchange(timeout_ns=1_000_000)  # 1 ms; rank 1 never arrives
    monkeypatch.setattr(sharding, "peer_exchange", lambda group, device: fake)
    with pytest.raises(RuntimeError, match="peer exchange"):
        lv.dot(X, Y)
    assert fake.failed and int(fake.error.item()) == 1
    # the group refuses further exchanges on the host ...
    with pytest.raises(RuntimeError, match="peer exchange"):
        lv.norm2(X)


def test_lazy_result_raises_at_item(monkeypatch, sharded_pair):
    X, Y, _, _ = sharded_pair
    fake = LocalPeerExchange(timeout_ns=1_000_000)
    monkeypatch.setattr(sharding, "peer_exchange", lambda group, device: fake)
    r = lv.dot(X, Y, lazy=True)  # no host synchronisation yet
    derived = (r + 1.0) / 2.0    # lazy scalar arithmetic inherits the guard
    with pytest.raises(RuntimeError, match="peer exchange"):
        derived.item()
    with pytest.raises(RuntimeError, match="peer exchange"):
        r.item()
    with pytest.raises(RuntimeError):
        float(r)


def test_device_poison_returns_at_once(monkeypatch, sharded_pair):
    """A rank whose error word is set touches no slot and does not wait: a
    60 s timeout is never reached."""
    X, Y, _, _ = sharded_pair
    fake = LocalPeerExchange(timeout_ns=60_000_000_000)
    fake.error.fill_(1)
    monkeypatch.setattr(sharding, "peer_exchange", lambda group, device: fake)
    t0 = time.perf_counter()
    with pytest.raises(RuntimeError):
        lv.dot(X, Y)
    assert time.perf_counter() - t0 < 5.0
    # no slot touched (rank 0 publishes no total once poisoned); its flag at
    # every peer carries ABORT instead, so the peers stop waiting for it
    words = fake.buffer.view(2, -1)  # [rank buffer][int64 words]
    nslot = 2 * _native.XCHG_MAX_RANKS * 2
    assert int(words[:, :nslot].abs().sum().item()) == 0
    assert int(words[0, nslot + 0].item()) == -1 and int(words[1, nslot + 0].item()) == -1


def test_a_peer_abort_ends_the_wait_at_once(monkeypatch, sharded_pair):
    """Rank 1 gave up (its ABORT flag is set in rank 0's buffer): rank 0
    returns NaN and raises at once instead of waiting out a 60 s timeout."""
    X, Y, _, _ = sharded_pair
    fake = LocalPeerExchange(timeout_ns=60_000_000_000)
    flags = fake.buffer[2 * _native.XCHG_MAX_RANKS * 2:]
    flags[1] = -1  # ~0: ABORT from rank 1
    torch.cuda.synchronize()
    monkeypatch.setattr(sharding, "peer_exchange", lambda group, device: fake)
    t0 = time.perf_counter()
    with pytest.raises(RuntimeError, match="peer exchange"):
        lv.dot(X, Y)
    assert time.perf_counter() - t0 < 5.0
    assert int(fake.error.item()) == 1


def test_peer_route_bits_match_the_allgather_route(monkeypatch, sharded_pair):
    """Rank 1 contributes +0.0: the folded total equals the one-rank total
    bit for bit (same dd fold as salt_reduce_finish)."""
    X, Y, x, y = sharded_pair
    want = lv.dot(X, Y)  # default route (world 1: partial -> finish)
    fake = LocalPeerExchange(timeout_ns=10_000_000_000)
    monkeypatch.setattr(sharding, "peer_exchange", lambda group, device: fake)
    for epoch in (1, 2, 3):  # both slot parities and reuse
        fake.publish_rank1(epoch, 0.0)
        got = lv.dot(X, Y)
        assert np.float64(got).tobytes() == np.float64(want).tobytes()
    assert fake.epoch == 3 and not fake.failed and int(fake.error.item()) == 0
