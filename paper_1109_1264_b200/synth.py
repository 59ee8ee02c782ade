"""Seeded synthetic inputs for the BASELINE.json configs.

No public dataset is involved; every operand is drawn from a keyed NumPy
stream `default_rng([SEED, cfg, operand, chunk])` with chunk = 2^24
elements, in float64, then cast to the element type (the reference's keyed
seed idiom: bench.py:97-106, test_acceptance.py:39-40, :72-73).  Chunk keying
lets any rank or checker regenerate any global range independently of how
the vector is sharded.  Scalars come from stream [SEED, cfg, 255] in order
alpha, beta, gamma.
"""

import numpy as np

__all__ = ["SEED", "CHUNK", "CONFIGS", "block", "scalars", "fill_device", "fill_device_philox"]

SEED = 1109_1264
CHUNK = 1 << 24

# cfg id -> (element distribution, scalar range)
CONFIGS = {
    1: ("uniform", 2.0),  # daxpy, n = 2^20, f64
    2: ("uniform", 2.0),  # fused sweep a + (b - c), alpha*a + beta*(b - c), f64
    3: ("normal", None),  # ddot / dnrm2, f32 and f64
    4: ("uniform", 2.0),  # e-tree, f32, sharded
    5: ("normal", 1.0),  # axpy -> dot, f64, sharded
}


def _draw(cfg: int, operand: int, chunk: int, count: int) -> np.ndarray:
    g = np.random.default_rng([SEED, cfg, operand, chunk])
    if CONFIGS[cfg][0] == "normal":
        return g.standard_normal(count)
    return g.uniform(-1.0, 1.0, count)


def block(cfg: int, operand: int, lo: int, hi: int, dtype) -> np.ndarray:
    """Elements [lo, hi) of operand `operand` of config `cfg` (global index)."""
    dt = np.dtype(dtype)
    out = np.empty(max(0, hi - lo), dtype=dt)
    pos = lo
    while pos < hi:
        c = pos // CHUNK
        c_lo = c * CHUNK
        take_hi = min(hi, c_lo + CHUNK)
        vals = _draw(cfg, operand, c, take_hi - c_lo)
        out[pos - lo : take_hi - lo] = vals[pos - c_lo :].astype(dt)
        pos = take_hi
    return out


def scalars(cfg: int, count: int = 3) -> list:
    """alpha, beta, gamma as Python floats (the API coerces them to dtype)."""
    rng_range = CONFIGS[cfg][1] or 1.0
    g = np.random.default_rng([SEED, cfg, 255])
    return [float(v) for v in g.uniform(-rng_range, rng_range, count)]


def fill_device(tensor, cfg: int, operand: int, lo: int = 0):
    """Fill a device tensor with elements [lo, lo + len) chunk by chunk (keeps
    host memory bounded for multi-GiB vectors)."""
    import torch

    n = tensor.shape[0]
    dt = {torch.float32: np.float32, torch.float64: np.float64}[tensor.dtype]
    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        tensor[s:e].copy_(torch.from_numpy(block(cfg, operand, lo + s, lo + e, dt)))
    return tensor


def fill_device_philox(tensor, cfg: int, operand: int, lo: int = 0):
    """Fill a device tensor with elements [lo, lo + len) of a DEVICE-generated
    stream: torch's Philox generator seeded per global chunk
    (SEED, cfg, operand, chunk), drawn in float64 with the config's
    distribution, then cast.  Chunk keying makes the global vector independent
    of the sharding, like block().  Used for the multi-GiB operands of the
    bench's multi-GPU block (config 5 is 3 x 16 GiB at one GPU), where the
    NumPy streams would cost a minute of host time; these values are NOT the
    NumPy streams' values (parity tests use block())."""
    import torch

    n = tensor.shape[0]
    dev = tensor.device
    normal = CONFIGS[cfg][0] == "normal"
    g = torch.Generator(device=dev)
    pos = 0
    while pos < n:
        c = (lo + pos) // CHUNK
        c_lo = c * CHUNK
        take = min(n - pos, c_lo + CHUNK - (lo + pos))
        g.manual_seed(((SEED * 16 + cfg) * 256 + operand) * (1 << 20) + c)
        full = torch.empty(CHUNK, dtype=torch.float64, device=dev)
        if normal:
            full.normal_(generator=g)
        else:
            full.uniform_(-1.0, 1.0, generator=g)
        off = lo + pos - c_lo
        tensor[pos:pos + take].copy_(full[off:off + take])
        pos += take
    return tensor
