"""Block-sharded vectors across GPUs (one process per GPU, torch.distributed).

The reference is single-process; the paper only sketches data-parallel
evaluation.  Here a global vector of length n is split
into contiguous blocks, one per rank:

    rank r owns [r*B, min(n, (r+1)*B)),  B = ceil(n / world) rounded up to a
    multiple of 64 elements, so every block base stays 256-byte aligned.

Elementwise trees over ShardedVectors run on each rank's block with no
communication.  Reductions exchange one double-double total per rank and
every rank folds them in rank order — deterministic and identical on all
ranks — by one of two routes:

  nccl  (default, and gloo on CPU): the kernel writes its partial
        (SALT_PARTIAL), a 16-byte all-gather collects them, and
        salt_reduce_finish folds them;
  peer  (opt-in: SALT_EXCHANGE=peer, GPUs with symmetric memory): the
        reduction kernel's last CTA writes its total straight into every
        peer's symmetric buffer over NVLink, raises a flag there, waits for
        all peers' flags and folds — the collective happens inside the
        reduction kernel (salt_reduce_exchange), no NCCL launch, no host
        involvement.

Both fold the same values in the same order, so they give identical bits.

Failure behaviour of the peer route (it must never return a wrong number):
  * the ranks agree on the route: after building its buffers every rank
    contributes an ok flag to one all_reduce(MIN); if any rank failed, every
    rank falls back to the all-gather;
  * a peer that does not arrive within the timeout (SALT_PEER_TIMEOUT_MS,
    default 60 s) makes the kernel write NaN and set a sticky error word;
    the host sees the NaN, reads the word and raises RuntimeError — at once
    for host results, at DeviceScalar.item() for lazy ones;
  * the error word poisons the exchange on the device: every later
    exchange kernel of that rank returns NaN at once without touching the
    peer slots (no read of a slot a later epoch has overwritten), and the
    host refuses further exchanges on that group.
"""

import os
import threading

import numpy as np
import torch
import torch.distributed as dist

from .lanes import as_dtype
from .sugar import VectorOps
from .vectors import DenseVector

__all__ = ["shard_bounds", "ShardedVector", "SHARD_ALIGN", "exchange_route"]

SHARD_ALIGN = 64


def shard_bounds(n: int, world: int, rank: int, align: int = SHARD_ALIGN):
    """[lo, hi) of `rank`'s block of a length-n vector split over `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if n < 0:
        raise ValueError(f"length must be >= 0, got {n}")
    per = -(-n // world) if n else 0
    per = -(-per // align) * align
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


class PeerExchange:
    """Symmetric NVLink buffers + epoch counter of one process group on one
    device (torch symmetric memory supplies the peer mappings)."""

    TIMEOUT_NS = 60_000_000_000  # a peer that never arrives yields NaN, not a hang

    def __init__(self, group, device, timeout_ns=None):
        import torch.distributed._symmetric_memory as symm_mem

        from ._native import XCHG_BUFFER_BYTES, XCHG_MAX_RANKS, Exchange

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > XCHG_MAX_RANKS:
            raise ValueError(f"peer exchange supports up to {XCHG_MAX_RANKS} ranks")
        name = (group or dist.group.WORLD).group_name
        try:
            symm_mem.enable_symm_mem_for_group(name)
        except Exception:  # newer torch enables it on demand
            pass
        self.buffer = symm_mem.empty(XCHG_BUFFER_BYTES // 8, dtype=torch.int64, device=device)
        self.buffer.zero_()
        self.error = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        self.handle = symm_mem.rendezvous(self.buffer, name)
        dist.barrier(group)
        ptrs = list(self.handle.buffer_ptrs)
        self.desc = Exchange()
        self.desc.rank = self.rank
        self.desc.world = self.world
        if timeout_ns is None:
            ms = os.environ.get("SALT_PEER_TIMEOUT_MS")
            timeout_ns = int(float(ms) * 1e6) if ms else self.TIMEOUT_NS
        self.desc.timeout_ns = int(timeout_ns)
        self.desc.error = self.error.data_ptr()
        for p, base in enumerate(ptrs):
            self.desc.slots[p] = base                     # DD[2][8]
            self.desc.flags[p] = base + 2 * XCHG_MAX_RANKS * 16  # u64[8]
        self.epoch = 0
        self.failed = False

    def next(self):
        """Descriptor for the next exchange (epochs advance in SPMD order)."""
        if self.failed:
            raise RuntimeError(self._message())
        self.epoch += 1
        self.desc.epoch = self.epoch
        return self.desc

    def _message(self):
        return (f"NVLink peer exchange of rank {self.rank}/{self.world} failed: a peer did not "
                f"arrive within {self.desc.timeout_ns / 1e6:.0f} ms (epoch {self.epoch}); the "
                "exchange is disabled for this group — rerun with SALT_EXCHANGE=nccl")

    def check(self, value=None):
        """Raise if the exchange timed out.  `value` is the reduction result
        (host scalar): the kernel writes NaN on a timeout, so only a NaN
        result costs a read of the device error word."""
        if value is not None and value == value:  # not NaN: cannot be a timeout
            return
        if self.failed or int(self.error.item()) != 0:
            self.failed = True
            raise RuntimeError(self._message())


_exchanges = {}
_exchange_lock = threading.Lock()


def exchange_route() -> str:
    """'nccl' (default) or 'peer' (SALT_EXCHANGE=peer)."""
    route = os.environ.get("SALT_EXCHANGE", "nccl")
    if route not in ("nccl", "peer"):
        raise ValueError(f"SALT_EXCHANGE must be 'nccl' or 'peer', got {route!r}")
    return route


def peer_exchange(group, device):
    """The PeerExchange of (group, device), or None when peer exchange is
    disabled (the default) or unavailable on any rank of the group (then
    reductions use the NCCL all-gather).  Collective on first use: every
    rank of the group must reach it (they do — reductions are SPMD)."""
    if exchange_route() != "peer" or device.type != "cuda":
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    key = (id(group), device.index)
    with _exchange_lock:
        if key not in _exchanges:
            # Agree BEFORE the collective construction (symmetric-memory
            # rendezvous): every rank must be able to reach every other
            # rank's device over peer memory and import symmetric memory;
            # otherwise no rank enters the rendezvous (a rank failing alone
            # inside it would leave the others waiting).
            if not _agree(group, device, _peer_capable(group, device)):
                _exchanges[key] = None
                return None
            try:
                xchg = PeerExchange(group, device)
            except Exception:
                xchg = None
            # one route for the whole group: peer only if every rank built it
            ok = torch.tensor([1 if xchg is not None else 0], dtype=torch.int32, device=device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            _exchanges[key] = xchg if int(ok.item()) == 1 else None
        return _exchanges[key]


def _agree(group, device, ok: bool) -> bool:
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return int(flag.item()) == 1


def _peer_capable(group, device) -> bool:
    """This rank can map every rank's device (all-gathers the device
    ordinals; same-node ranks) and has torch symmetric memory."""
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except Exception:
        return False
    world = dist.get_world_size(group)
    mine = torch.tensor([device.index], dtype=torch.int64, device=device)
    allv = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    try:
        return all(d == device.index or torch.cuda.can_device_access_peer(device.index, d)
                   for d in (int(v) for v in allv.tolist()))
    except Exception:
        return False


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


class ShardedVector(VectorOps):
    """A global vector of `global_len` elements; this rank holds `local`."""

    __slots__ = ("local", "global_len", "lo", "hi", "group", "world", "rank")

    __array_ufunc__ = None

    def __init__(self, local: DenseVector, global_len: int, group=None):
        self.group = group
        self.world, self.rank = _world(group)
        self.global_len = int(global_len)
        self.lo, self.hi = shard_bounds(self.global_len, self.world, self.rank)
        if len(local) != self.hi - self.lo:
            raise ValueError(
                f"rank {self.rank} block must hold {self.hi - self.lo} elements, got {len(local)}"
            )
        self.local = local

    @classmethod
    def zeros(cls, n: int, dtype="f32", group=None, device=None):
        world, rank = _world(group)
        lo, hi = shard_bounds(n, world, rank)
        return cls(DenseVector.zeros(hi - lo, dtype, device=device), n, group)

    @classmethod
    def from_global(cls, values, dtype="f32", group=None, device=None):
        """Take this rank's block of a host array holding the global vector."""
        arr = np.asarray(values).reshape(-1)
        world, rank = _world(group)
        lo, hi = shard_bounds(arr.shape[0], world, rank)
        return cls(DenseVector.from_values(arr[lo:hi], dtype, device=device), arr.shape[0], group)

    @classmethod
    def from_blocks(cls, n: int, dtype, make_block, group=None, device=None):
        """Build from `make_block(lo, hi) -> array` for this rank's block only
        (each rank generates just its own data)."""
        world, rank = _world(group)
        lo, hi = shard_bounds(n, world, rank)
        return cls(DenseVector.from_values(make_block(lo, hi), dtype, device=device), n, group)

    @property
    def dtype(self):
        return self.local.dtype

    def __len__(self) -> int:
        return self.global_len

    def same_partition(self, other) -> bool:
        return (
            isinstance(other, ShardedVector)
            and other.global_len == self.global_len
            and other.world == self.world
            and other.group is self.group
        )

    def gather_partials(self, part: torch.Tensor) -> torch.Tensor:
        """All-gather one {hi, lo} float64 pair per rank, in rank order (a
        16-byte NCCL all-gather per rank over NVLink; gloo on CPU)."""
        if not (dist.is_available() and dist.is_initialized()):
            return part.reshape(-1)
        out = torch.empty(self.world * part.numel(), dtype=part.dtype, device=part.device)
        if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(self.group) == "nccl":
            # one collective straight into the rank-ordered buffer (no torch.cat launch)
            dist.all_gather_into_tensor(out, part.reshape(-1), group=self.group)
            return out
        parts = list(out.view(self.world, -1).unbind(0))
        dist.all_gather(parts, part.reshape(-1), group=self.group)
        return out

    # ---- inspection (collective: every rank must call) ----
    def to_array(self) -> np.ndarray:
        if self.world == 1:
            return self.local.to_array()
        per = shard_bounds(self.global_len, self.world, 0)[1]
        dt = as_dtype(self.dtype)
        buf = torch.zeros(per, dtype=self.local.tensor.dtype, device=self.local.device)
        buf[: len(self.local)] = self.local.tensor
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        full = torch.cat(parts)[: self.global_len]
        return full.cpu().numpy().astype(dt, copy=False)

    def read_block(self, lo: int, hi: int):
        return self.to_array()[lo:hi]

    def assign(self, expression, **options) -> None:
        from .engine import execute_assign
        from .expressions import AssignNode, Leaf, as_node

        execute_assign(AssignNode(Leaf(self), as_node(expression)), **options)


    def __repr__(self):
        return (
            f"ShardedVector(len={self.global_len}, rank={self.rank}/{self.world}, "
            f"block=[{self.lo},{self.hi}), dtype={self.dtype})"
        )
