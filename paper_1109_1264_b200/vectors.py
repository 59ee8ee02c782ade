"""DenseVector: the leaves and destinations of expressions, resident in HBM.

Reference: pkg/src/lanevec/vectors.py:1-144 (a 64-byte aligned NumPy buffer).
Here the storage is a 1-D torch tensor — torch is only the allocator — that
lives either

  * on a CUDA device (the normal case: trees over device vectors run as one
    fused sm_100a kernel on that device), or
  * in pinned host memory (`device="cpu"`): trees over host vectors are
    streamed through the GPU in chunks (H2D -> fused kernel -> D2H, three
    overlapped streams, `salt_assign_host`).  This is the end-to-end path
    and also lets vectors larger than HBM be evaluated.

Storage is aligned to DEVICE_ALIGNMENT (256 B), which satisfies the
reference's CONTAINER_ALIGNMENT (64 B) and the kernels' 256-bit accesses.
Element access (get/set/read_block/...) keeps the reference's duck-typed
vector protocol (expressions.py:68-69) and copies across PCIe when the
storage is on the device; it is for inspection, not for the hot path.
"""

import numpy as np
import torch

from .lanes import DEVICE_ALIGNMENT, as_dtype
from .sugar import VectorOps

__all__ = ["DenseVector", "DeviceScalar", "default_device", "torch_dtype"]

_TORCH_DTYPES = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
_NP_DTYPES = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}


def torch_dtype(dt: np.dtype) -> torch.dtype:
    return _TORCH_DTYPES[as_dtype(dt)]


def default_device() -> torch.device:
    """The current CUDA device, or the host when this process has no GPU
    (vectors can then be built and inspected, but evaluating a tree raises:
    there is no CPU evaluation path)."""
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _as_device(device) -> torch.device:
    if device is None:
        return default_device()
    if isinstance(device, int):
        return torch.device("cuda", device)
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if dev.type not in ("cuda", "cpu"):
        raise ValueError(f"unsupported device {device!r}")
    return dev


def _aligned_empty(n: int, dt: np.dtype, device: torch.device) -> torch.Tensor:
    """Uninitialised length-n storage whose base address is 256-B aligned."""
    tdt = _TORCH_DTYPES[dt]
    pad = DEVICE_ALIGNMENT // dt.itemsize
    if device.type == "cpu":
        raw = torch.empty(n + pad, dtype=tdt, pin_memory=torch.cuda.is_available())
    else:
        raw = torch.empty(n + pad, dtype=tdt, device=device)
    start = ((-raw.data_ptr()) % DEVICE_ALIGNMENT) // dt.itemsize
    return raw[start : start + n]


class DenseVector(VectorOps):
    """Fixed-length contiguous f32/f64 vector (reference vectors.py:18-31)."""

    # _ptr/_dev/_n/_code cache what the C fast path (csrc/fastpath.c) reads
    __slots__ = ("_data", "_dtype", "_ptr", "_dev", "_n", "_code")

    def __init__(self, data: torch.Tensor, dtype):
        self._data = data
        self._dtype = as_dtype(dtype)
        self._ptr = data.data_ptr()
        self._dev = data.get_device()  # -1 for host storage
        self._n = int(data.shape[0])
        self._code = 0 if self._dtype.itemsize == 4 else 1

    # ------------------------------------------------------------ creation
    @classmethod
    def zeros(cls, n: int, dtype="f32", device=None) -> "DenseVector":
        if n < 0:
            raise ValueError(f"length must be >= 0, got {n}")
        dt = as_dtype(dtype)
        buf = _aligned_empty(int(n), dt, _as_device(device))
        buf.zero_()
        return cls(buf, dt)

    @classmethod
    def empty(cls, n: int, dtype="f32", device=None) -> "DenseVector":
        """Uninitialised vector (a destination that will be fully assigned)."""
        if n < 0:
            raise ValueError(f"length must be >= 0, got {n}")
        dt = as_dtype(dtype)
        return cls(_aligned_empty(int(n), dt, _as_device(device)), dt)

    @classmethod
    def from_values(cls, values, dtype="f32", device=None) -> "DenseVector":
        dt = as_dtype(dtype)
        src = np.ascontiguousarray(np.asarray(values, dtype=dt).reshape(-1))
        buf = _aligned_empty(src.shape[0], dt, _as_device(device))
        if src.shape[0]:
            buf.copy_(torch.from_numpy(src))
        return cls(buf, dt)

    @classmethod
    def from_tensor(cls, tensor: torch.Tensor) -> "DenseVector":
        """Wrap an existing 1-D contiguous f32/f64 tensor without copying."""
        if tensor.dim() != 1 or not tensor.is_contiguous():
            raise ValueError("from_tensor needs a 1-D contiguous tensor")
        if tensor.dtype not in _NP_DTYPES:
            raise TypeError(f"unsupported element type {tensor.dtype}; use float32 or float64")
        return cls(tensor, _NP_DTYPES[tensor.dtype])

    @classmethod
    def from_dlpack(cls, obj) -> "DenseVector":
        """Zero-copy import of any DLPack producer (CuPy, JAX, NumPy, torch)
        holding a 1-D contiguous f32/f64 array."""
        return cls.from_tensor(torch.from_dlpack(obj))

    def __dlpack__(self, **kwargs):
        return self._data.__dlpack__(**kwargs)

    def __dlpack_device__(self):
        return self._data.__dlpack_device__()

    @property
    def __cuda_array_interface__(self):
        """CUDA array interface (CuPy / Numba) for device-resident vectors."""
        if self._data.device.type != "cuda":
            raise AttributeError("host vectors have no __cuda_array_interface__")
        return self._data.__cuda_array_interface__

    # ------------------------------------------------------------ properties
    @property
    def dtype(self) -> np.dtype:
        return self._dtype

    @property
    def device(self) -> torch.device:
        return self._data.device

    @property
    def tensor(self) -> torch.Tensor:
        """The backing storage (borrowed; do not resize)."""
        return self._data

    @property
    def address(self) -> int:
        """Base address of the storage (device or pinned host)."""
        return self._data.data_ptr()

    def __len__(self) -> int:
        return int(self._data.shape[0])

    # ------------------------------------------------------------ elements
    def _check_index(self, i: int) -> None:
        if not 0 <= i < self._data.shape[0]:
            raise IndexError(f"index {i} out of range for length {len(self)}")

    def get(self, i: int):
        self._check_index(i)
        return self._dtype.type(self._data[i].item())

    def set(self, i: int, value) -> None:
        self._check_index(i)
        self._data[i] = float(self._dtype.type(value))

    def __getitem__(self, i: int):
        return self.get(i)

    def __setitem__(self, i: int, value) -> None:
        self.set(i, value)

    def to_array(self) -> np.ndarray:
        """Copy of the contents as a host NumPy array."""
        return self._data.detach().to("cpu").numpy().copy()

    def to_values(self) -> list:
        """Elements as a list of element-typed NumPy scalars."""
        return list(self.to_array())

    # Duck-typed vector protocol (reference vectors.py:88-100).  Block reads
    # return host copies.
    def read_block(self, lo: int, hi: int) -> np.ndarray:
        return self._data[lo:hi].detach().to("cpu").numpy()

    def write_block(self, lo: int, hi: int, values) -> None:
        src = torch.from_numpy(np.ascontiguousarray(np.asarray(values, dtype=self._dtype)))
        self._data[lo:hi].copy_(src)

    def read_element(self, i: int):
        return self._dtype.type(self._data[i].item())

    def write_element(self, i: int, value) -> None:
        self._data[i] = float(self._dtype.type(value))

    # ------------------------------------------------------------ evaluation
    def assign(self, expression, **plan_kwargs) -> None:
        """Evaluate a lazy expression into this vector in one fused pass."""
        if not plan_kwargs:  # the C fast path first: no AssignNode / Leaf objects
            from ._native import fastpath

            fast = fastpath()
            if fast is not None and fast.assign(self, expression):
                return
        from .engine import execute_assign
        from .expressions import AssignNode, Leaf, as_node

        execute_assign(AssignNode(Leaf(self), as_node(expression)), **plan_kwargs)

    # Arithmetic builds lazy nodes: sugar.VectorOps (reference vectors.py:109-138).

    __array_ufunc__ = None

    def __repr__(self):
        n = len(self)
        head = self._data[:6].detach().to("cpu").tolist() if n else []
        shown = ", ".join(repr(float(v)) for v in head)
        tail = ", ..." if n > 6 else ""
        return f"DenseVector([{shown}{tail}], len={n}, dtype={self._dtype}, device={self.device})"


class DeviceScalar:
    """An element-typed scalar that lives in device memory.

    Returned by reductions called with `lazy=True` (no host
    synchronisation).  It can scale an expression like a Python number —
    `a * p` with `a` a DeviceScalar builds a ScaleNode whose alpha the fused
    kernel reads from device memory — and DeviceScalars combine with + - * /
    and unary minus.  Those combinations are LAZY: `alpha = rr / pq` records
    the operation instead of launching anything.  Used as an operand of a
    fused tree it is compiled into the kernel's scalar program and computed
    once per thread in that kernel's prologue (salt_fused_prog), so a whole
    solver iteration (dots -> alpha = rr / pq -> fused update) is one launch
    per reduction and one per update, with no host round trip, and can be
    captured in a CUDA graph.  Anything that needs the value itself
    (`.item()`, float(), `.tensor`, `.address`) materialises it once with
    1-element torch ops.  Either way every operation is one IEEE
    round-to-nearest op in the element type, so both give the same bits.
    `.item()` / float() return the element-typed NumPy scalar the reference
    returns (test_ops.py:29-31).
    """

    __slots__ = ("_tensor", "dtype", "guard", "_expr", "_version", "_seen")

    __array_ufunc__ = None

    # a lazy scalar with more operations than this is materialised instead
    # of being compiled into a kernel's scalar program (32 ops, stack 8)
    MAX_PROGRAM_OPS = 24

    def __init__(self, tensor, dtype, guard=None, _expr=None):
        self._tensor = tensor
        self.dtype = as_dtype(dtype)
        # guard(value): raises if the producing collective failed (a peer
        # exchange that timed out writes NaN; see sharding.PeerExchange.check)
        self.guard = guard
        # (op, operand[, operand]) for a lazy result: op in + - * / neg,
        # operands DeviceScalars or element-typed Python floats
        self._expr = _expr
        # copy_() bumps _version; a lazy result remembers its operands'
        # versions (_seen) and refuses to run on an operand changed since
        self._version = 0
        self._seen = None if _expr is None else tuple(
            a._version if isinstance(a, DeviceScalar) else None for a in _expr[1:])

    @classmethod
    def full(cls, value, dtype="f64", device=None) -> "DeviceScalar":
        dt = as_dtype(dtype)
        return cls(torch.full((1,), float(dt.type(value)), dtype=_TORCH_DTYPES[dt],
                              device=_as_device(device)), dt)

    # ---- value (materialised on demand) ----
    @property
    def lazy(self) -> bool:
        """True while this scalar is an unevaluated operation."""
        return self._tensor is None

    @property
    def tensor(self) -> torch.Tensor:
        t = self._tensor
        if t is None:
            t = self._tensor = self._materialise()
        return t

    def check_operands(self) -> None:
        """Raise if an operand of this lazy scalar was modified in place
        (copy_) after the operation was recorded: the recorded operation
        would no longer give what an eager evaluation would have given."""
        if self._tensor is not None or self._expr is None:
            return
        for a, v in zip(self._expr[1:], self._seen):
            if isinstance(a, DeviceScalar):
                if a._version != v:
                    raise RuntimeError("a DeviceScalar operand was modified in place (copy_) after this "
                                       "lazy scalar operation was recorded; use it before modifying its "
                                       "operands, or materialise it first (.tensor)")
                a.check_operands()

    def _materialise(self) -> torch.Tensor:
        self.check_operands()
        op, *args = self._expr
        ref = next(a for a in args if isinstance(a, DeviceScalar)).tensor
        ts = [a.tensor if isinstance(a, DeviceScalar) else torch.full_like(ref, a) for a in args]
        if op == "neg":
            return torch.neg(ts[0])
        fn = {"+": torch.add, "-": torch.sub, "*": torch.mul, "/": torch.div}[op]
        return fn(ts[0], ts[1])

    @property
    def device(self) -> torch.device:
        if self._tensor is not None:
            return self._tensor.device
        return next(a for a in self._expr[1:] if isinstance(a, DeviceScalar)).device

    def program_size(self) -> int:
        """Operations a scalar program needs to compute this scalar."""
        if self._tensor is not None or self._expr is None:
            return 1
        return 1 + sum(a.program_size() if isinstance(a, DeviceScalar) else 1 for a in self._expr[1:])

    @property
    def address(self) -> int:
        return self.tensor.data_ptr()

    def item(self):
        v = self.dtype.type(self.tensor.item())
        if self.guard is not None:
            self.guard(v)
        return v

    def __float__(self):
        return float(self.item())

    # ---- scalar arithmetic (lazy: recorded, evaluated in the consuming kernel) ----
    def _operand(self, other):
        if isinstance(other, DeviceScalar):
            if other.dtype != self.dtype:
                raise TypeError(f"mixed element types: {self.dtype} vs {other.dtype}")
            return other
        return float(self.dtype.type(other))

    def _lazy(self, op, *args):
        # a result inherits its operands' guard (a failed collective behind
        # an operand still raises at .item() of anything computed from it)
        guard = next((a.guard for a in args if isinstance(a, DeviceScalar) and a.guard is not None), None)
        return DeviceScalar(None, self.dtype, guard=guard, _expr=(op,) + args)

    def __truediv__(self, other):
        if isinstance(other, (DeviceScalar, int, float, np.floating)):
            return self._lazy("/", self, self._operand(other))
        return NotImplemented

    def __rtruediv__(self, other):
        if isinstance(other, (int, float, np.floating)):
            return self._lazy("/", self._operand(other), self)
        return NotImplemented

    def copy_(self, other) -> "DeviceScalar":
        """In-place assignment (keeps this scalar's device address, so a
        CUDA graph that reads it sees the new value on the next replay)."""
        self.tensor.copy_(other.tensor if isinstance(other, DeviceScalar) else
                          torch.tensor([float(self.dtype.type(other))], dtype=self.tensor.dtype))
        self._version += 1
        return self

    def __add__(self, other):
        if isinstance(other, (DeviceScalar, int, float, np.floating)):
            return self._lazy("+", self, self._operand(other))
        return NotImplemented

    def __radd__(self, other):
        if isinstance(other, (int, float, np.floating)):
            return self._lazy("+", self._operand(other), self)
        return NotImplemented

    def __sub__(self, other):
        if isinstance(other, (DeviceScalar, int, float, np.floating)):
            return self._lazy("-", self, self._operand(other))
        return NotImplemented

    def __rsub__(self, other):
        if isinstance(other, (int, float, np.floating)):
            return self._lazy("-", self._operand(other), self)
        return NotImplemented

    def __neg__(self):
        return self._lazy("neg", self)

    def __mul__(self, other):
        if isinstance(other, (DeviceScalar, int, float, np.floating)):
            return self._lazy("*", self, self._operand(other))
        from .expressions import scale_node

        return scale_node(self, other)  # scalar * vector expression

    def __rmul__(self, other):
        if isinstance(other, (int, float, np.floating)):
            return self._lazy("*", self._operand(other), self)
        return NotImplemented

    def __repr__(self):
        return f"DeviceScalar({self.item()!r}, dtype={self.dtype})"
