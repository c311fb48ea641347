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
    assert L.lib.ldbp_abi_version() == 2


def test_validation_before_launch(L):
    lib = L.lib
    P = ctypes.c_void_p
    fake = P(0x10000)  # never dereferenced: validation fails first

    def fwd(d, x=fake, y=P(0x20000), taps=fake, gamma=fake):
        return lib.ldbp_forward(ctypes.byref(d), x, y, taps, gamma, None, 0, None)

    assert fwd(L.dims(1, 16, 2, 4)) == -2           # even T
    assert fwd(L.dims(1, 64, 2, 33)) == -2          # T > LDBP_MAX_TAPS (31)
    assert fwd(L.dims(1, 4, 2, 5)) == -2            # T > n
    assert fwd(L.dims(1, 16, 0, 3)) == -2           # M < 1
    assert fwd(L.dims(-1, 16, 2, 3)) == -2          # B < 0
    assert fwd(L.dims(1, 0, 2, 3)) == -2            # n < 1
    d = L.dims(1, 16, 2, 3)
    d.reserved = 1
    assert fwd(d) == -1
    assert fwd(L.dims(1, 16, 2, 3, flags=16)) == -1  # unknown flag
    assert lib.ldbp_status_string(-6).startswith(b"LDBP_ENONFINITE")
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


def test_store_all_schedule_workspace(L):
    """Backward / loss_grad / train use the store-all schedule when B*n >= 2^20 and the
    activations fit the budget: the workspace holds all M activations; tiny or over-budget
    problems use the checkpoint schedule (ldbp.h)."""
    lib = L.lib
    out = ctypes.c_size_t(0)
    d = L.dims(512, 16384, 50, 9, 1)  # C3
    assert lib.ldbp_workspace_bytes(ctypes.byref(d), 2, ctypes.byref(out)) == 0
    assert out.value >= 50 * 512 * 16384 * 8
    d1 = L.dims(4, 1024, 4, 3, 1)  # C1: segments
    assert lib.ldbp_workspace_bytes(ctypes.byref(d1), 2, ctypes.byref(out)) == 0
    assert out.value < 4 * 4 * 1024 * 8
    os.environ["LDBP_BWD_MODE"] = "0"
    try:
        assert lib.ldbp_workspace_bytes(ctypes.byref(d), 2, ctypes.byref(out)) == 0
        assert out.value < 50 * 512 * 16384 * 8 // 4
    finally:
        del os.environ["LDBP_BWD_MODE"]


def test_tiny_fused_step_plan(L):
    """C1-sized problems (M <= 5 or more than one recompute segment, the per-CTA activations fit
    shared memory) train in ONE launch
    (ldbp_tiny.cuh); LDBP_TINY=0 restores the segment schedule; over-size or long models never
    take the fused kernel by default."""
    lib = L.lib
    nl = ctypes.c_int(0)
    d1 = L.dims(4, 1024, 4, 3, 1)  # C1
    for op in (2, 3):
        assert lib.ldbp_launch_count(ctypes.byref(d1), op, ctypes.byref(nl)) == 0 and nl.value == 1
    assert lib.ldbp_launch_count(ctypes.byref(d1), 1, ctypes.byref(nl)) == 0 and nl.value > 1  # backward: no
    os.environ["LDBP_TINY"] = "0"
    try:
        assert lib.ldbp_launch_count(ctypes.byref(d1), 3, ctypes.byref(nl)) == 0 and nl.value > 2
    finally:
        del os.environ["LDBP_TINY"]
    d16 = L.dims(4, 1024, 16, 3, 1)  # two recompute segments in the segment schedule: fused instead
    assert lib.ldbp_launch_count(ctypes.byref(d16), 3, ctypes.byref(nl)) == 0 and nl.value == 1
    for d in (L.dims(4, 1024, 8, 3, 1), L.dims(64, 4096, 4, 3, 1), L.dims(2, 1 << 16, 2, 3, 1)):
        assert lib.ldbp_launch_count(ctypes.byref(d), 3, ctypes.byref(nl)) == 0 and nl.value > 1


def test_rx_essm_ssfm_validation(L):
    """The NEXT-row entry points validate shapes and pointers before any launch."""
    lib = L.lib
    P = ctypes.c_void_p
    f = P(0x10000)
    out = ctypes.c_size_t(0)
    # receiver chain: n % sps, MF length, sps range
    assert lib.ldbp_rx_workspace_bytes(2, 1001, 2, ctypes.byref(out)) == -2
    assert lib.ldbp_rx_workspace_bytes(2, 1024, 5, ctypes.byref(out)) == -2
    assert lib.ldbp_rx_workspace_bytes(2, 1024, 2, ctypes.byref(out)) == 0 and out.value > 0
    assert lib.ldbp_rx_loss_grad(2, 1024, 2, 600, f, f, f, f, f, None, f, 1 << 20, None) == -2  # 2L+1 > n
    assert lib.ldbp_rx_loss_grad(2, 1024, 2, 64, None, f, f, f, f, None, f, 1 << 20, None) == -1
    assert lib.ldbp_rx_loss_grad(2, 1024, 2, 64, f, f, f, f, f, f, f, 1 << 20, None) == -1  # gy aliases y
    assert lib.ldbp_rx_loss_grad(2, 1024, 2, 64, f, f, f, f, f, None, f, 0, None) == -4   # workspace
    assert lib.ldbp_rx_loss_grad(0, 1024, 2, 64, None, None, None, None, None, None, None, 0, None) == 0
    # ESSM: kappa range and filter length
    d = L.dims(2, 32, 3, 5, 1)
    assert lib.ldbp_essm_workspace_bytes(ctypes.byref(d), 33, 0, ctypes.byref(out)) == -2
    assert lib.ldbp_essm_workspace_bytes(ctypes.byref(d), 16, 0, ctypes.byref(out)) == -2  # 33 > n
    assert lib.ldbp_essm_workspace_bytes(ctypes.byref(d), 4, 2, ctypes.byref(out)) == 0
    assert out.value >= 3 * 2 * 32 * 8
    assert lib.ldbp_essm_workspace_bytes(ctypes.byref(d), 4, 1, ctypes.byref(out)) == -1  # no BACKWARD op
    # SSFM: power-of-two n <= 2^16 (2- and 4-CTA clusters above 2^14), at most 64 steps per span
    assert lib.ldbp_ssfm_workspace_bytes(1000, 4, ctypes.byref(out)) == -2
    assert lib.ldbp_ssfm_workspace_bytes(1 << 17, 4, ctypes.byref(out)) == -2
    assert lib.ldbp_ssfm_workspace_bytes(1 << 16, 65, ctypes.byref(out)) == -2
    assert lib.ldbp_ssfm_workspace_bytes(1 << 16, 4, ctypes.byref(out)) == 0 and out.value >= 4 * (1 << 16) * 8
    assert lib.ldbp_ssfm_workspace_bytes(1 << 14, 4, ctypes.byref(out)) == 0 and out.value >= 4 * (1 << 14) * 8
