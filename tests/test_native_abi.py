"""The C-ABI library (CPU): it loads without a GPU, exports every function
include/salt.h declares, and validates signatures / arguments before any
CUDA call (so these run with no device)."""

import ctypes
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1109_1264_b200 import _native

HEADER = ROOT / "include" / "salt.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(salt_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_native.HEADER_SYMBOLS)


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (salt_\w+)", out))
    assert set(header_functions()) <= exported


def test_abi_constants():
    lib = _native.lib()
    assert lib.salt_abi_version() == 1
    assert lib.salt_reduce_workspace_bytes() >= 256 + 16 * 1024


@pytest.mark.parametrize("sig,kind,expect", [
    ("L0", 0, 1),
    ("S0 L0 *", 0, 1),
    ("L0 S0 L1 * +", 0, 1),
    ("L0 L1 L2 - +", 0, 1),
    ("S0 L0 * S1 L1 L2 - * +", 0, 1),
    ("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", 0, 1),
    ("L0 L1 *", 1, 1),
    ("L0 L0 *", 1, 1),
    ("L0", 1, 1),
    ("L0 L1 * L2 *", 0, 2),          # not in the table: NVRTC instantiates it
    ("L0 L1 L2 L3 L4 L5 L6 L7 + + + + + + +", 0, 2),
    ("L0 +", 0, 0),                  # malformed
    ("L0 L1", 0, 0),                 # two values left
    ("L16", 0, 0),                   # leaf index out of range (SALT_MAX_LEAVES = 16)
    ("L15", 0, 2),
    ("S32 L0 *", 0, 0),
    ("L0 / L1", 0, 0),
    ("D L0 *", 0, 0),                # D only inside a fused reduce tree
    ("", 0, 0),
])
def test_signature_validation(sig, kind, expect):
    assert _native.lib().salt_signature_kind(1, sig.encode(), None, kind) == expect


def test_fused_signature_kind():
    lib = _native.lib()
    assert lib.salt_signature_kind(1, b"L0 S0 L1 * +", b"D L2 *", 2) == 1
    assert lib.salt_signature_kind(0, b"L0 S0 L1 * +", b"D D *", 2) == 1
    assert lib.salt_signature_kind(0, b"L0 L1 +", b"D L0 *", 2) == 2
    assert lib.salt_signature_kind(0, b"L0 L1 +", b"D +", 2) == 0


def test_bad_arguments_fail_before_cuda():
    lib = _native.lib()
    leaves, keep = _native.ptr_array([0x1000, 0x2000])
    sc, keep2 = _native.double_array([1.0])
    rc = lib.salt_assign(1, b"L0 L1 L2 + +", ctypes.c_void_p(0x3000), leaves, 2, sc, 1, 10, None)
    assert rc == -1 and b"3 leaves" in lib.salt_last_error()
    rc = lib.salt_assign(7, b"L0", ctypes.c_void_p(0x3000), leaves, 1, sc, 0, 10, None)
    assert rc == -1 and b"dtype" in lib.salt_last_error()
    rc = lib.salt_assign(1, b"L0 L1 ?", ctypes.c_void_p(0x3000), leaves, 2, sc, 0, 10, None)
    assert rc == -1 and b"bad token" in lib.salt_last_error()
    rc = lib.salt_reduce(1, b"L0 L1 *", leaves, 2, sc, 0, 10, 0, None, 0, ctypes.c_void_p(8), None, None)
    assert rc == -4  # workspace too small
    with pytest.raises(RuntimeError, match="libsalt error"):
        _native.check(lib.salt_assign(1, b"L0 +", None, leaves, 1, sc, 0, 1, None))
    # zero-length assignment is a no-op that never touches CUDA
    assert lib.salt_assign(1, b"L0", ctypes.c_void_p(0x3000), leaves, 1, sc, 0, 0, None) == 0
    # single-process all-reduce: arguments are validated before NCCL or CUDA
    outs, keep3 = _native.ptr_array([0x1000])
    assert lib.salt_allreduce_sum(outs, 0, 1, None, outs) == -1
    assert lib.salt_allreduce_sum(outs, 1, 7, outs, outs) == -1 and b"dtype" in lib.salt_last_error()
    assert lib.salt_allreduce_sum_flags(outs, 1, 1, outs, outs, _native.SALT_PARTIAL) == -1
    assert b"flags" in lib.salt_last_error()
    assert lib.salt_nccl_comm_init_all(0, None, outs) == -1
    assert lib.salt_nccl_comm_destroy(1, None) == -1


def test_nvrtc_instantiates_arbitrary_trees_without_a_gpu():
    """The JIT compiles the same fused-kernel template for trees outside the
    table (vector + scalar-lane variants), even after torch is imported
    (torch bundles an older NVRTC; libsalt loads the toolkit's by path)."""
    import torch  # noqa: F401

    lib = _native.lib()
    for dt in (0, 1):
        assert lib.salt_prepare(dt, b"L0 L1 * L2 * S0 L3 * -", None, 0) == 0, lib.salt_last_error()
        assert lib.salt_prepare(dt, b"L0 L1 - L2 L3 + *", None, 1) == 0, lib.salt_last_error()
        assert lib.salt_prepare(dt, b"L0 L1 +", b"D D *", 2) == 0, lib.salt_last_error()
    assert lib.salt_prepare(1, b"L0 +", None, 0) == -1


def test_jit_disk_cache(tmp_path):
    """JIT cubins are cached on disk (SALT_JIT_CACHE); a second process loads
    them instead of recompiling."""
    import os
    import sys

    code = ("import time; from paper_1109_1264_b200 import _native; l = _native.lib(); "
            "t = time.time(); assert l.salt_prepare(0, b'L0 L1 - L0 * L2 -', None, 0) == 0; "
            "print(time.time() - t)")
    env = {**os.environ, "SALT_JIT_CACHE": str(tmp_path / "jit")}
    first = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           cwd=ROOT, check=True)
    files = sorted((tmp_path / "jit").glob("*.salt"))
    assert len(files) == 2  # vector and scalar-lane variants
    second = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                            cwd=ROOT, check=True)
    assert float(second.stdout) < float(first.stdout)
    # every entry carries the format magic and is private to the user
    for f in files:
        assert f.read_bytes().startswith(b"SALTJIT2 ") and (f.stat().st_mode & 0o077) == 0
    assert ((tmp_path / "jit").stat().st_mode & 0o077) == 0
    # a corrupted entry is not trusted: it is deleted and rebuilt by NVRTC
    blob = bytearray(files[0].read_bytes())
    blob[-20] ^= 0xFF
    files[0].write_bytes(bytes(blob))
    subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT, check=True)
    assert files[0].read_bytes() != bytes(blob) and files[0].read_bytes().startswith(b"SALTJIT2 ")


def test_jit_disk_cache_refuses_a_shared_directory(tmp_path):
    """A cache directory writable by group/others is not used at all (no
    kernel is read from it or written to it); compilation still works."""
    import os
    import sys

    shared = tmp_path / "shared"
    shared.mkdir()
    os.chmod(shared, 0o777)
    (shared / "planted.salt").write_bytes(b"not a kernel")
    code = ("from paper_1109_1264_b200 import _native; l = _native.lib(); "
            "assert l.salt_prepare(0, b'L0 L1 + L0 * L2 -', None, 0) == 0")
    env = {**os.environ, "SALT_JIT_CACHE": str(shared)}
    subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT, check=True)
    assert sorted(p.name for p in shared.iterdir()) == ["planted.salt"]


def test_c_fast_path_declines_what_it_cannot_take():
    """The fast path only takes plain device vectors; everything else is
    declined (False / None) so the Python path handles it (and raises the
    reference's errors)."""
    import paper_1109_1264_b200 as lv
    from paper_1109_1264_b200.expressions import ScaleNode, as_node

    fast = _native.fastpath()
    assert fast is not None
    x = lv.DenseVector.zeros(10, "f64", device="cpu")
    y = lv.DenseVector.zeros(10, "f64", device="cpu")
    assert fast.assign(y, as_node(y) + ScaleNode(0.5, as_node(x))) is False
    assert fast.reduce(as_node(x) * as_node(y), 0) is None
    assert fast.assign_reduce(y, as_node(y) + ScaleNode(0.5, as_node(x)), as_node(y) * as_node(x), 0) is None
    cv = lv.CountingVector.zeros(10, "f64", device="cpu")
    assert fast.assign(cv, as_node(x)) is False


@pytest.mark.parametrize("prog,msg", [
    (b"p0 p1 / =0 +", b"underflow"),
    (b"p0 p1", b"leaves values"),
    (b"p0 =1", b"does not define P0"),
    (b"p5 =0", b"device scalar 5"),
    (b"S9 =0", b"host scalar 9"),
    (b"p0 % =0", b"bad scalar program token"),
    (b"p0 =9", b"output index"),
    (b" ".join([b"p0"] * 9) + b" " + b" ".join([b"+"] * 8) + b" =0", b"deeper than 8"),
])
def test_scalar_program_is_validated_before_any_launch(prog, msg):
    """salt_fused_prog rejects malformed scalar programs with SALT_EINVAL and
    a message, before touching the device (runs without a GPU)."""
    lib = _native.lib()
    dummy = ctypes.c_double(0.0)
    ptr = ctypes.addressof(dummy)
    leaves, k1 = _native.ptr_array([ptr])
    dsts, k2 = _native.ptr_array([ptr])
    ps, k3 = _native.ptr_array([ptr, ptr])
    sc, k4 = _native.double_array([1.0])
    rc = lib.salt_fused_prog(1, b"P0 L0 *", None, dsts, 1, leaves, 1, sc, 1, ps, 2, prog, 4, 0, None, 0,
                             None, None, None)
    assert rc == -1  # SALT_EINVAL
    assert msg in lib.salt_last_error(), lib.salt_last_error()


def test_traced_kernel_source_compiles_with_nvrtc():
    """salt_set_trace switches a call to the NVRTC build of its tree with
    -DSALT_TRACE.  Without a GPU the call must get past the JIT (the traced
    source compiles) and fail only at the first CUDA runtime call."""
    lib = _native.lib()
    dummy = ctypes.c_double(0.0)
    ptr = ctypes.addressof(dummy)
    leaves, k1 = _native.ptr_array([ptr, ptr])
    sc, k2 = _native.double_array([0.5])
    buf = (ctypes.c_int64 * 64)()
    assert lib.salt_set_trace(ctypes.addressof(buf), 64) == 0
    try:
        rc = lib.salt_assign(1, b"L0 S0 L1 * -", ctypes.c_void_p(ptr), leaves, 2, sc, 1, 4096, None)
        msg = lib.salt_last_error().decode()
    finally:
        assert lib.salt_set_trace(None, 0) == 0
    assert rc != 0
    assert "traced kernel" not in msg and "NVRTC" not in msg, msg
    assert lib.salt_set_trace(ctypes.addressof(buf), 2) != 0  # too small a buffer
