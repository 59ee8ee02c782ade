"""Fuzzing the C ABI's signature parser (CPU, no GPU): any byte string must
be classified without crashing, and for well-formed token streams the
verdict must match a plain postfix validator (stack discipline, index
bounds SALT_MAX_LEAVES / SALT_MAX_SCALARS)."""

import hypothesis.strategies as st
from hypothesis import HealthCheck, given, settings

from paper_1109_1264_b200 import _native

TOKENS = ([f"L{k}" for k in range(18)] + [f"S{k}" for k in range(34)] + ["+", "-", "*"] * 6)


def valid(tokens):
    depth = 0
    for t in tokens:
        if t[0] == "L":
            if int(t[1:]) >= _native.SALT_MAX_LEAVES:
                return False
            depth += 1
        elif t[0] == "S":
            if int(t[1:]) >= _native.SALT_MAX_SCALARS:
                return False
            depth += 1
        else:
            if depth < 2:
                return False
            depth -= 1
    return depth == 1


@settings(max_examples=400, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(st.sampled_from(TOKENS), min_size=0, max_size=40), st.sampled_from([0, 1]),
       st.sampled_from([0, 1]))
def test_token_streams_match_a_postfix_validator(tokens, kind, dtype):
    sig = " ".join(tokens).encode()
    got = _native.lib().salt_signature_kind(dtype, sig, None, kind)
    assert got in (0, 1, 2)
    assert (got != 0) == valid(tokens), (sig, got)


@settings(max_examples=300, deadline=None)
@given(st.binary(min_size=0, max_size=200), st.binary(min_size=0, max_size=60),
       st.sampled_from([0, 1, 2]))
def test_arbitrary_bytes_never_crash(sig, rsig, kind):
    sig = sig.replace(b"\x00", b" ")
    rsig = rsig.replace(b"\x00", b" ")
    got = _native.lib().salt_signature_kind(1, sig, rsig if kind == 2 else None, kind)
    assert got in (0, 1, 2)
