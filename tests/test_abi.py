"""CPU-side checks of the C ABI: libldbp.so loads, exports every symbol include/ldbp.h declares,
and validates arguments before touching the GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2010_14258_b200 import _lib

    return _lib


def header_functions():
    src = open(os.path.join(ROOT, "include", "ldbp.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|size_t)\s+(ldbp_\w+)\(", src, flags=re.M)))


def test_header_symbols_exported(L):
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L.lib, name), name
    assert sorted(L.EXPORTED) == names
    assert L.lib.ldbp_abi_version() == 1


def test_validation_before_launch(L):
    lib = L.lib
    P = ctypes.c_void_p
    fake = P(0x10000)  # never dereferenced: validation fails first

    def fwd(d, x=fake, y=P(0x20000), taps=fake, gamma=fake):
        return lib.ldbp_forward(ctypes.byref(d), x, y, taps, gamma, None, 0, None)

    assert fwd(L.dims(1, 16, 2, 4)) == -2           # even T
    assert fwd(L.dims(1, 16, 2, 17)) == -2          # T > LDBP_MAX_TAPS
    assert fwd(L.dims(1, 4, 2, 5)) == -2            # T > n
    assert fwd(L.dims(1, 16, 0, 3)) == -2           # M < 1
    assert fwd(L.dims(-1, 16, 2, 3)) == -2          # B < 0
    assert fwd(L.dims(1, 0, 2, 3)) == -2            # n < 1
    d = L.dims(1, 16, 2, 3)
    d.reserved = 1
    assert fwd(d) == -1
    assert fwd(L.dims(1, 16, 2, 3, flags=8)) == -1  # unknown flag
    assert fwd(L.dims(1, 16, 2, 3), x=None) == -1
    assert fwd(L.dims(1, 16, 2, 3), x=P(0x10004)) == -3  # misaligned complex64
    assert fwd(L.dims(1, 16, 2, 3), y=fake) == -1   # y aliases x
    assert b"aliases" in lib.ldbp_last_error() or b"alias" in lib.ldbp_last_error()
    assert fwd(L.dims(0, 16, 2, 3)) == 0            # empty batch: no-op
    for s in (0, -1, -2, -3, -4, -5):
        assert lib.ldbp_status_string(s).startswith(b"LDBP")


def test_forward_workspace_and_launch_plan(L):
    lib = L.lib
    out = ctypes.c_size_t(123)
    d = L.dims(256, 16384, 25, 5, 1)
    assert lib.ldbp_workspace_bytes(ctypes.byref(d), 0, ctypes.byref(out)) == 0
    assert out.value == 0  # one launch, no ping-pong buffer
    nl = ctypes.c_int(0)
    assert lib.ldbp_launch_count(ctypes.byref(d), 0, ctypes.byref(nl)) == 0 and nl.value == 1
    d = L.dims(4096, 16384, 100, 15, 1)
    assert lib.ldbp_workspace_bytes(ctypes.byref(d), 0, ctypes.byref(out)) == 0
    assert out.value >= 4096 * 16384 * 8  # chained launches need one ping-pong buffer
    assert lib.ldbp_launch_count(ctypes.byref(d), 0, ctypes.byref(nl)) == 0 and nl.value >= 2
    assert lib.ldbp_workspace_bytes(ctypes.byref(d), 9, ctypes.byref(out)) == -1
