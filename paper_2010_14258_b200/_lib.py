"""ctypes loader for libldbp.so (the C ABI declared in include/ldbp.h).

Argument marshalling only.  If the shared library is missing this module raises at import
time: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LDBP_LIB", os.path.join(_HERE, "libldbp.so"))

LDBP_SYMMETRIC = 1
LDBP_PRECISE = 2
LDBP_CHECK_FINITE = 4
LDBP_STREAM_PIPELINE = 8
OP_FORWARD, OP_BACKWARD, OP_LOSS_GRAD, OP_TRAIN_STEP = 0, 1, 2, 3

# Every symbol include/ldbp.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "ldbp_abi_version",
    "ldbp_status_string",
    "ldbp_last_error",
    "ldbp_workspace_bytes",
    "ldbp_launch_count",
    "ldbp_forward",
    "ldbp_backward",
    "ldbp_loss_grad",
    "ldbp_adam_update",
    "ldbp_train_step",
    "ldbp_trace_begin",
    "ldbp_trace_end",
    "ldbp_rx_workspace_bytes",
    "ldbp_rx_loss_grad",
    "ldbp_rx_train_workspace_bytes",
    "ldbp_rx_train_grad",
    "ldbp_essm_workspace_bytes",
    "ldbp_essm_forward",
    "ldbp_essm_loss_grad",
    "ldbp_rx_exact_loss_grad",
    "ldbp_rx_exact_train_workspace_bytes",
    "ldbp_rx_exact_train_grad",
    "ldbp_ssfm_workspace_bytes",
    "ldbp_ssfm_link",
    "ldbp_tx_waveform",
)

K_FORWARD, K_BACKWARD, K_REDUCE, K_ADAM, K_REVERSE, K_RX, K_ESSM, K_SSFM, K_TINY = 1, 2, 3, 4, 5, 6, 7, 8, 9


class LdbpDims(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("steps", ctypes.c_int32),
        ("taps", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("reserved", ctypes.c_int32),
    ]


class TraceRecord(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("steps", ctypes.c_int32),
        ("samples", ctypes.c_int64),
        ("ms", ctypes.c_float),
        ("reserved", ctypes.c_int32),
    ]


class LdbpError(RuntimeError):
    def __init__(self, status: int, func: str, detail: str):
        super().__init__(f"{func} failed with status {status}: {detail}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libldbp.so not found at {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    D = ctypes.POINTER(LdbpDims)
    dbl = ctypes.c_double
    sig = {
        "ldbp_abi_version": (ctypes.c_int, []),
        "ldbp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "ldbp_last_error": (ctypes.c_char_p, []),
        "ldbp_workspace_bytes": (ctypes.c_int, [D, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_launch_count": (ctypes.c_int, [D, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "ldbp_forward": (ctypes.c_int, [D, P, P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_backward": (ctypes.c_int, [D, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_loss_grad": (ctypes.c_int, [D, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_adam_update": (ctypes.c_int, [D, P, dbl, P, P, P, ctypes.c_int64, dbl, dbl, dbl, dbl, P, P, P, P, P]),
        "ldbp_train_step": (ctypes.c_int, [D, P, P, P, P, P, P, P, ctypes.c_int64, dbl, dbl, dbl, dbl, P, P, P, P,
                                           ctypes.c_size_t, P]),
        "ldbp_trace_begin": (ctypes.c_int, [ctypes.c_int]),
        "ldbp_trace_end": (ctypes.c_int, [ctypes.POINTER(TraceRecord), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "ldbp_rx_workspace_bytes": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                   ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_rx_loss_grad": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                             P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_rx_train_workspace_bytes": (ctypes.c_int, [D, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_rx_train_grad": (ctypes.c_int, [D, P, P, P, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P,
                                              ctypes.c_size_t, P]),
        "ldbp_rx_exact_loss_grad": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_float,
                                                   P, P, P, P, P, P, P]),
        "ldbp_rx_exact_train_workspace_bytes": (ctypes.c_int, [D, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_rx_exact_train_grad": (ctypes.c_int, [D, P, P, P, P, ctypes.c_int32, ctypes.c_float, P, P, P, P, P,
                                                    ctypes.c_size_t, P]),
        "ldbp_essm_workspace_bytes": (ctypes.c_int, [D, ctypes.c_int32, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_essm_forward": (ctypes.c_int, [D, ctypes.c_int32, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_essm_loss_grad": (ctypes.c_int, [D, ctypes.c_int32, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "ldbp_tx_waveform": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, P, P,
                                            ctypes.c_int32, P, P, P, P, P]),
        "ldbp_ssfm_workspace_bytes": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]),
        "ldbp_ssfm_link": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_double), dbl, dbl, dbl, dbl, dbl, dbl, P,
                                          ctypes.c_uint64, ctypes.c_int64, P, P, ctypes.c_int32, dbl, P,
                                          ctypes.c_size_t, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int, func: str) -> None:
    if status != 0:
        detail = lib.ldbp_last_error().decode(errors="replace")
        raise LdbpError(status, func, f"{lib.ldbp_status_string(status).decode()} ({detail})")


def dims(batch: int, n: int, steps: int, taps: int, flags: int = 0) -> LdbpDims:
    return LdbpDims(int(batch), int(n), int(steps), int(taps), int(flags), 0)
