"""Thin Python binding of libldbp (same names as the C ABI, include/ldbp.h).

PyTorch is plumbing only: tensors provide device memory, the current CUDA stream and (in
``dp.py``) the process group.  Every step of the hot path runs inside libldbp's kernels.
"""
from __future__ import annotations

import contextlib
import ctypes
import functools
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (LDBP_CHECK_FINITE, LDBP_PRECISE, LDBP_STREAM_PIPELINE, LDBP_SYMMETRIC, OP_BACKWARD, OP_FORWARD,
                   OP_LOSS_GRAD, OP_TRAIN_STEP, check, lib)

_VP = ctypes.c_void_p


def _p(t):
    return None if t is None else _VP(t.data_ptr())


def _stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return _VP(s.cuda_stream)


def _flags(symmetric: bool, precise: bool, check_finite: bool = False) -> int:
    return ((LDBP_SYMMETRIC if symmetric else 0) | (LDBP_PRECISE if precise else 0)
            | (LDBP_CHECK_FINITE if check_finite else 0))


def _need(t, name, dtype, shape=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libldbp has no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def make_dims(B, n, M, T, symmetric=True, precise=False, check_finite=False):
    return _lib.dims(B, n, M, T, _flags(symmetric, precise, check_finite))


def workspace_bytes(d, op: int) -> int:
    out = ctypes.c_size_t(0)
    check(lib.ldbp_workspace_bytes(ctypes.byref(d), op, ctypes.byref(out)), "ldbp_workspace_bytes")
    return int(out.value)


def launch_count(d, op: int) -> int:
    out = ctypes.c_int(0)
    check(lib.ldbp_launch_count(ctypes.byref(d), op, ctypes.byref(out)), "ldbp_launch_count")
    return int(out.value)


class Workspace:
    """Grow-only device scratch buffer (allocated by torch's caching allocator, outside any call)."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int, device):
        if nbytes == 0:
            return None
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return self.buf


_default_ws = {}


def _ws(device, nbytes, ws):
    """Scratch for one call, enqueued on torch's current stream (the call's stream: see _on_stream).
    Default workspaces are private per (device, stream, thread), so concurrent calls on different
    streams or threads never share scratch; a caller-supplied ``ws`` used on several streams is
    protected against early reuse by record_stream (the caching allocator then waits for every
    stream that used the buffer before handing its memory out again)."""
    cur = torch.cuda.current_stream(device)
    if ws is None:
        key = (str(device), cur.cuda_stream, threading.get_ident())
        ws = _default_ws.setdefault(key, Workspace())
    b = ws.get(nbytes, device)
    if b is not None and not torch.cuda.is_current_stream_capturing():
        b.record_stream(cur)
    return b, nbytes


def _on_stream(fn):
    """Run a binding with ``stream=`` made torch's current stream, so that every output and
    scratch tensor is allocated on (and its memory ordered by) the stream the kernels run on."""

    @functools.wraps(fn)
    def wrapper(*args, stream=None, **kw):
        ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            return fn(*args, stream=stream, **kw)

    return wrapper


def _check_buf(buf, length, device):
    """Caller-supplied gradient buffer: float64, contiguous, exactly ``length`` long, on ``device``."""
    if buf is None:
        return torch.empty(length, dtype=torch.float64, device=device)
    _need(buf, "buf", torch.float64, (length,))
    if buf.device != device:
        raise ValueError(f"buf is on {buf.device}, expected {device}")
    return buf


def _check_model(x, taps, gamma):
    _need(x, "x", torch.complex64)
    if x.dim() != 2:
        raise ValueError("x must be [B][n]")
    _need(taps, "taps", torch.complex64)
    if taps.dim() != 2:
        raise ValueError("taps must be [M][T]")
    M, T = taps.shape
    _need(gamma, "gamma", torch.float32, (M,))
    return x.shape[0], x.shape[1], M, T


@_on_stream
def ldbp_forward(x, taps, gamma, *, symmetric=True, precise=False, check_finite=False, pipeline=False, out=None,
                 ws=None, stream=None):
    """y = f_theta(x) (Eq. 7) for complex64 x [B][n], taps [M][T], gamma [M].  check_finite:
    raise LdbpError (LDBP_ENONFINITE, with the first failing step) on NaN/Inf activations.
    pipeline: LDBP_STREAM_PIPELINE (ldbp.h) — the caller guarantees that no earlier, possibly still
    running kernel on the stream writes x/taps/gamma or touches out (a rotation of >= 3 buffers)."""
    B, n, M, T = _check_model(x, taps, gamma)
    d = make_dims(B, n, M, T, symmetric, precise, check_finite)
    if pipeline:
        d.flags |= LDBP_STREAM_PIPELINE
    y = torch.empty_like(x) if out is None else out
    _need(y, "out", torch.complex64, x.shape)
    nb = workspace_bytes(d, OP_FORWARD)
    w, nb = _ws(x.device, nb, ws)
    check(lib.ldbp_forward(ctypes.byref(d), _p(x), _p(y), _p(taps), _p(gamma), _p(w), nb, _stream_handle(stream)),
          "ldbp_forward")
    return y


@_on_stream
def ldbp_backward(x, gy, taps, gamma, *, symmetric=True, precise=False, need_gx=True, ws=None, stream=None):
    """Reverse mode for incoming gy = dL/dy.  Returns (dtaps complex128 [M][T], dgamma f64 [M], gx or None)."""
    B, n, M, T = _check_model(x, taps, gamma)
    _need(gy, "gy", torch.complex64, x.shape)
    d = make_dims(B, n, M, T, symmetric, precise)
    dt = torch.empty((M, T, 2), dtype=torch.float64, device=x.device)
    dg = torch.empty((M,), dtype=torch.float64, device=x.device)
    gx = torch.empty_like(x) if need_gx else None
    nb = workspace_bytes(d, OP_BACKWARD)
    w, nb = _ws(x.device, nb, ws)
    check(lib.ldbp_backward(ctypes.byref(d), _p(x), _p(gy), _p(taps), _p(gamma), _p(dt), _p(dg), _p(gx), _p(w), nb,
                            _stream_handle(stream)), "ldbp_backward")
    return torch.view_as_complex(dt), dg, gx


@_on_stream
def ldbp_loss_grad(x, target, taps, gamma, *, mask=None, symmetric=True, precise=False, check_finite=False,
                   buf=None, ws=None, stream=None):
    """[sum|e|^2 | dgamma[M] | dtaps[M][T][2]] (float64, unscaled, this device's blocks only)."""
    B, n, M, T = _check_model(x, taps, gamma)
    _need(target, "target", torch.complex64, x.shape)
    if mask is not None:
        _need(mask, "mask", torch.uint8, (M, T))
    d = make_dims(B, n, M, T, symmetric, precise, check_finite)
    out = _check_buf(buf, 1 + M + 2 * M * T, x.device)
    nb = workspace_bytes(d, OP_LOSS_GRAD)
    w, nb = _ws(x.device, nb, ws)
    check(lib.ldbp_loss_grad(ctypes.byref(d), _p(x), _p(target), _p(taps), _p(gamma), _p(mask), _p(out), _p(w), nb,
                             _stream_handle(stream)), "ldbp_loss_grad")
    return out


def ldbp_loss_grad_state(state, x, target, *, buf=None, ws=None, stream=None):
    """ldbp_loss_grad on a TrainState's working copies.  When the mask leaves only the central
    active_T < T taps (progressive pruning), the call runs on that central window (the
    T'-tap kernels; masked taps are exactly zero, so the result is the same computation) and the
    gradient is laid out back into the full [1 + M + 2 M T] buffer with zeros for the pruned taps."""
    M, T = state.taps.shape
    Ta = state.active_T
    if state.mask is None or Ta is None or Ta >= T:
        return ldbp_loss_grad(x, target, state.taps, state.gamma, mask=state.mask, symmetric=state.symmetric,
                              precise=state.precise, buf=buf, ws=ws, stream=stream)
    lo = (T - Ta) // 2
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        taps_c = state.taps[:, lo:lo + Ta].contiguous()
        mask_c = state.mask[:, lo:lo + Ta].contiguous()
        bc = ldbp_loss_grad(x, target, taps_c, state.gamma, mask=mask_c, symmetric=state.symmetric,
                            precise=state.precise, ws=ws, stream=stream)
        out = _check_buf(buf, 1 + M + 2 * M * T, x.device)
        out.zero_()
        out[:1 + M] = bc[:1 + M]
        out[1 + M:].view(M, T, 2)[:, lo:lo + Ta] = bc[1 + M:].view(M, Ta, 2)
    return out


@dataclass
class AdamConfig:
    lr: float = 1e-3  # Table I
    b1: float = 0.9   # reading G13 (paper silent)
    b2: float = 0.999
    eps: float = 1e-8


@dataclass
class TrainState:
    """Parameters + Adam state on the device: fp64 master, fp32 working copies (row a10)."""

    taps: torch.Tensor          # complex64 [M][T] working copy
    gamma: torch.Tensor         # float32 [M] working copy
    master: torch.Tensor        # float64 [2MT + M]
    m: torch.Tensor
    v: torch.Tensor
    t: int = 0
    mask: torch.Tensor | None = None            # uint8 [M][T]
    gamma_learnable: torch.Tensor | None = None  # uint8 [M]
    active_T: int | None = None                  # host-known: every tap outside the central active_T is masked
    symmetric: bool = True
    precise: bool = False
    adam: AdamConfig = field(default_factory=AdamConfig)

    @staticmethod
    def create(taps, gamma, *, device="cuda", mask=None, gamma_learnable=None, symmetric=True, precise=False,
               adam=None):
        taps = torch.as_tensor(taps).to(torch.complex128)
        gamma = torch.as_tensor(gamma).to(torch.float64)
        M, T = taps.shape
        master = torch.cat([torch.view_as_real(taps).reshape(-1), gamma]).to(device)
        z = torch.zeros_like(master)
        st = TrainState(taps=taps.to(torch.complex64).to(device).contiguous(),
                        gamma=gamma.to(torch.float32).to(device).contiguous(), master=master.contiguous(),
                        m=z.clone(), v=z.clone(), symmetric=symmetric, precise=precise, adam=adam or AdamConfig())
        if mask is not None:
            st.set_mask(mask)
        if gamma_learnable is not None:
            st.gamma_learnable = torch.as_tensor(gamma_learnable, dtype=torch.uint8).to(device).contiguous()
        return st

    def set_mask(self, mask):
        """Install a (host) tap mask; records the narrowest odd window that holds every unmasked tap,
        so that training runs the shorter-filter kernels (§8(f) NEXT-3: pruned taps cost nothing)."""
        m = np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask, dtype=np.uint8)
        if self.mask is None:
            self.mask = torch.from_numpy(m).to(self.taps.device).contiguous()
        else:
            self.mask.copy_(torch.from_numpy(m), non_blocking=False)
        kh = (m.shape[1] - 1) // 2
        cols = np.nonzero(m.any(axis=0))[0]
        k = int(max(abs(cols - kh).max(), 0)) if len(cols) else 0
        self.active_T = 2 * k + 1

    @property
    def M(self):
        return self.taps.shape[0]

    @property
    def T(self):
        return self.taps.shape[1]


@_on_stream
def ldbp_adam_update(state: TrainState, buf_reduced, n_global: float, *, stream=None):
    """One Adam step on the device from an (all-reduced) gradient buffer."""
    _need(buf_reduced, "buf_reduced", torch.float64, (1 + state.M + 2 * state.M * state.T,))
    state.t += 1
    d = make_dims(1, state.T, state.M, state.T, state.symmetric, state.precise)
    a = state.adam
    check(lib.ldbp_adam_update(ctypes.byref(d), _p(buf_reduced), float(n_global), _p(state.master), _p(state.m),
                               _p(state.v), int(state.t), a.lr, a.b1, a.b2, a.eps, _p(state.mask),
                               _p(state.gamma_learnable), _p(state.taps), _p(state.gamma), _stream_handle(stream)),
          "ldbp_adam_update")


@_on_stream
def ldbp_train_step(state: TrainState, x, target, *, buf=None, ws=None, stream=None):
    """Single-process step: loss_grad on the working copies then Adam with n_global = B*n."""
    B, n, M, T = _check_model(x, state.taps, state.gamma)
    _need(target, "target", torch.complex64, x.shape)
    d = make_dims(B, n, M, T, state.symmetric, state.precise)
    out = _check_buf(buf, 1 + M + 2 * M * T, x.device)
    nb = workspace_bytes(d, OP_TRAIN_STEP)
    w, nb = _ws(x.device, nb, ws)
    state.t += 1
    a = state.adam
    check(lib.ldbp_train_step(ctypes.byref(d), _p(x), _p(target), _p(state.taps), _p(state.gamma), _p(state.master),
                              _p(state.m), _p(state.v), int(state.t), a.lr, a.b1, a.b2, a.eps, _p(state.mask),
                              _p(state.gamma_learnable), _p(out), _p(w), nb, _stream_handle(stream)),
          "ldbp_train_step")
    return out


def _check_rx(y_like, symbols, power_w, h_mf, sps):
    B, n = y_like.shape
    if n % sps:
        raise ValueError(f"n = {n} is not a multiple of sps = {sps}")
    _need(symbols, "symbols", torch.complex64, (B, n // sps))
    _need(power_w, "power_w", torch.float32, (B,))
    _need(h_mf, "h_mf", torch.float32)
    if h_mf.dim() != 1 or h_mf.numel() % 2 == 0:
        raise ValueError("h_mf must be 1-D with an odd number of taps (2L+1)")
    return B, n, (h_mf.numel() - 1) // 2


@_on_stream
def ldbp_rx_loss_grad(y, symbols, power_w, h_mf, *, sps=2, need_grad=True, ws=None, stream=None):
    """Receiver-chain symbol loss (§8(f) NEXT-1): matched filter + downsample + genie phase.
    Returns (errs float64 [B], gy complex64 [B][n] or None); L = sum(errs)."""
    _need(y, "y", torch.complex64)
    B, n, L = _check_rx(y, symbols, power_w, h_mf, sps)
    errs = torch.empty(B, dtype=torch.float64, device=y.device)
    gy = torch.empty_like(y) if need_grad else None
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_rx_workspace_bytes(B, n, sps, ctypes.byref(nb)), "ldbp_rx_workspace_bytes")
    w, nbv = _ws(y.device, int(nb.value), ws)
    check(lib.ldbp_rx_loss_grad(B, n, sps, L, _p(y), _p(symbols), _p(power_w), _p(h_mf), _p(errs), _p(gy), _p(w),
                                nbv, _stream_handle(stream)), "ldbp_rx_loss_grad")
    return errs, gy


@_on_stream
def ldbp_rx_train_grad(x, symbols, power_w, h_mf, taps, gamma, *, sps=2, mask=None, symmetric=True, precise=False,
                       buf=None, ws=None, stream=None):
    """[sum errs | dgamma[M] | dtaps[M][T][2]] of the receiver-chain loss through LDBP (float64,
    unscaled, this device's blocks only)."""
    B, n, M, T = _check_model(x, taps, gamma)
    _, _, L = _check_rx(x, symbols, power_w, h_mf, sps)
    if mask is not None:
        _need(mask, "mask", torch.uint8, (M, T))
    d = make_dims(B, n, M, T, symmetric, precise)
    out = _check_buf(buf, 1 + M + 2 * M * T, x.device)
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_rx_train_workspace_bytes(ctypes.byref(d), sps, ctypes.byref(nb)), "ldbp_rx_train_workspace_bytes")
    w, nbv = _ws(x.device, int(nb.value), ws)
    check(lib.ldbp_rx_train_grad(ctypes.byref(d), _p(x), _p(symbols), _p(power_w), sps, L, _p(h_mf), _p(taps),
                                 _p(gamma), _p(mask), _p(out), _p(w), nbv, _stream_handle(stream)),
          "ldbp_rx_train_grad")
    return out


@_on_stream
def ldbp_rx_exact_loss_grad(y, symbols, power_w, *, sps=2, rolloff=0.1, weights=None, need_grad=True, stream=None):
    """Receiver-chain symbol loss with the exact circulant matched filter (§8(f) NEXT-1, Eq. (12)).
    Returns (errs float64 [B] unweighted, gy complex64 [B][n] = dL/dy of L = sum_b w_b errs_b, or None)."""
    _need(y, "y", torch.complex64)
    B, n = y.shape
    if n % sps:
        raise ValueError(f"n = {n} is not a multiple of sps = {sps}")
    _need(symbols, "symbols", torch.complex64, (B, n // sps))
    _need(power_w, "power_w", torch.float32, (B,))
    if weights is not None:
        _need(weights, "weights", torch.float32, (B,))
    errs = torch.empty(B, dtype=torch.float64, device=y.device)
    gy = torch.empty_like(y) if need_grad else None
    check(lib.ldbp_rx_exact_loss_grad(B, n, sps, float(rolloff), _p(y), _p(symbols), _p(power_w), _p(weights),
                                      _p(errs), _p(gy), _stream_handle(stream)), "ldbp_rx_exact_loss_grad")
    return errs, gy


@_on_stream
def ldbp_tx_waveform(codes, constellation, power_w, *, sps=2, rolloff=0.1, shift=None, phase=None, out=None,
                     stream=None):
    """Transmitted waveform [B][K sps] complex64 from symbol codes (uint8 [B][K] into `constellation`,
    complex64 [Q]) on the device: sqrt(P_b) sps e^{j phase_b} (RRC-shaped periodic frame, Eq. (11)),
    circularly shifted by shift_b samples (int32) — the waveform-MSE training target."""
    _need(codes, "codes", torch.uint8)
    B, K = codes.shape
    n = K * sps
    _need(constellation, "constellation", torch.complex64)
    q = constellation.numel()
    _need(power_w, "power_w", torch.float32, (B,))
    if shift is not None:
        _need(shift, "shift", torch.int32, (B,))
    if phase is not None:
        _need(phase, "phase", torch.float32, (B,))
    if out is None:
        out = torch.empty((B, n), dtype=torch.complex64, device=codes.device)
    else:
        _need(out, "out", torch.complex64, (B, n))
    check(lib.ldbp_tx_waveform(B, n, sps, float(rolloff), _p(codes), _p(constellation), q, _p(power_w), _p(shift),
                               _p(phase), _p(out), _stream_handle(stream)), "ldbp_tx_waveform")
    return out


@_on_stream
def ldbp_rx_exact_train_grad(x, symbols, power_w, taps, gamma, *, sps=2, rolloff=0.1, weights=None, mask=None,
                             symmetric=True, precise=False, buf=None, ws=None, stream=None):
    """[sum_b w_b errs_b | dgamma[M] | dtaps[M][T][2]] of the exact receiver-chain loss through LDBP."""
    B, n, M, T = _check_model(x, taps, gamma)
    _need(symbols, "symbols", torch.complex64, (B, n // sps))
    _need(power_w, "power_w", torch.float32, (B,))
    if weights is not None:
        _need(weights, "weights", torch.float32, (B,))
    if mask is not None:
        _need(mask, "mask", torch.uint8, (M, T))
    d = make_dims(B, n, M, T, symmetric, precise)
    out = _check_buf(buf, 1 + M + 2 * M * T, x.device)
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_rx_exact_train_workspace_bytes(ctypes.byref(d), sps, ctypes.byref(nb)),
          "ldbp_rx_exact_train_workspace_bytes")
    w, nbv = _ws(x.device, int(nb.value), ws)
    check(lib.ldbp_rx_exact_train_grad(ctypes.byref(d), _p(x), _p(symbols), _p(power_w), _p(weights), sps,
                                       float(rolloff), _p(taps), _p(gamma), _p(mask), _p(out), _p(w), nbv,
                                       _stream_handle(stream)), "ldbp_rx_exact_train_grad")
    return out


def _check_eta(eta, M):
    _need(eta, "eta", torch.float32)
    if eta.dim() != 2 or eta.shape[0] != M or eta.shape[1] % 2 == 0:
        raise ValueError("eta must be float32 [M][2*kappa+1]")
    return (eta.shape[1] - 1) // 2


@_on_stream
def ldbp_essm_forward(x, taps, gamma, eta, *, symmetric=True, precise=False, out=None, ws=None, stream=None):
    """Learned ESSM forward (§8(f) NEXT-4): y = f_theta(x) with filtered nonlinear steps."""
    B, n, M, T = _check_model(x, taps, gamma)
    kappa = _check_eta(eta, M)
    d = make_dims(B, n, M, T, symmetric, precise)
    y = torch.empty_like(x) if out is None else out
    _need(y, "out", torch.complex64, x.shape)
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_essm_workspace_bytes(ctypes.byref(d), kappa, OP_FORWARD, ctypes.byref(nb)), "ldbp_essm_workspace_bytes")
    w, nbv = _ws(x.device, int(nb.value), ws)
    check(lib.ldbp_essm_forward(ctypes.byref(d), kappa, _p(x), _p(y), _p(taps), _p(gamma), _p(eta), _p(w), nbv,
                                _stream_handle(stream)), "ldbp_essm_forward")
    return y


@_on_stream
def ldbp_essm_loss_grad(x, target, taps, gamma, eta, *, symmetric=True, precise=False, buf=None, ws=None,
                        stream=None):
    """[sum|e|^2 | dgamma[M] | dtaps[M][T][2] | deta[M][2kappa+1]] (float64, unscaled)."""
    B, n, M, T = _check_model(x, taps, gamma)
    kappa = _check_eta(eta, M)
    _need(target, "target", torch.complex64, x.shape)
    d = make_dims(B, n, M, T, symmetric, precise)
    out = _check_buf(buf, 1 + M + 2 * M * T + M * (2 * kappa + 1), x.device)
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_essm_workspace_bytes(ctypes.byref(d), kappa, OP_LOSS_GRAD, ctypes.byref(nb)),
          "ldbp_essm_workspace_bytes")
    w, nbv = _ws(x.device, int(nb.value), ws)
    check(lib.ldbp_essm_loss_grad(ctypes.byref(d), kappa, _p(x), _p(target), _p(taps), _p(gamma), _p(eta), _p(out),
                                  _p(w), nbv, _stream_handle(stream)), "ldbp_essm_loss_grad")
    return out


@_on_stream
def ldbp_ssfm_link(u, deltas_km, *, spans, span_km, alpha_np, beta2, gamma, fs_hz, ase_sigma=0.0, noise=None,
                   ase_seed=None, block0=0, decim=0, cutoff=0.5, ws=None, stream=None):
    """GPU SSFM channel generator (§8(f) NEXT-2): propagates u [B][n] (complex64, n a power of two
    <= 65536, in place) over `spans` spans of len(deltas_km) steps each, EDFA + ASE.  ASE draws:
    ``noise`` [spans][B][n] CN(0,1), or (noise None, ase_sigma != 0) Philox draws keyed by
    (ase_seed, global block block0 + b, span, sample) — ldbp_inputs.ase_cn_philox.
    decim > 0 returns the low-passed (|fftfreq| <= cutoff), decimated output [B][n // decim]."""
    _need(u, "u", torch.complex64)
    B, n = u.shape
    if noise is not None:
        _need(noise, "noise", torch.complex64, (spans, B, n))
    elif ase_sigma != 0.0 and ase_seed is None:
        raise ValueError("ase_sigma != 0 needs either noise draws or an ase_seed")
    d = (ctypes.c_double * len(deltas_km))(*[float(v) for v in deltas_km])
    nb = ctypes.c_size_t(0)
    check(lib.ldbp_ssfm_workspace_bytes(n, len(deltas_km), ctypes.byref(nb)), "ldbp_ssfm_workspace_bytes")
    w, nbv = _ws(u.device, int(nb.value), ws)
    r = torch.empty((B, n // decim), dtype=torch.complex64, device=u.device) if decim > 0 else None
    check(lib.ldbp_ssfm_link(B, n, spans, len(deltas_km), d, span_km, alpha_np, beta2, gamma, fs_hz, ase_sigma,
                             _p(noise), int(ase_seed or 0) & 0xFFFFFFFFFFFFFFFF, int(block0), _p(u), _p(r), int(decim),
                             float(cutoff), _p(w), nbv, _stream_handle(stream)), "ldbp_ssfm_link")
    return r if decim > 0 else u


class trace:
    """Context manager: per-launch CUDA-event timing of libldbp kernels on this thread.

    >>> with trace() as t:
    ...     ldbp_forward(x, taps, gamma)
    >>> t.records  # [(kind, steps, samples, ms), ...]
    """

    def __init__(self, capacity: int = 4096):
        self.capacity = capacity
        self.records = []
        self.count = 0

    def __enter__(self):
        check(lib.ldbp_trace_begin(self.capacity), "ldbp_trace_begin")
        return self

    def __exit__(self, *exc):
        arr = (_lib.TraceRecord * self.capacity)()
        cnt = ctypes.c_int(0)
        check(lib.ldbp_trace_end(arr, self.capacity, ctypes.byref(cnt)), "ldbp_trace_end")
        self.count = cnt.value
        self.records = [(r.kind, r.steps, r.samples, r.ms) for r in arr[: min(cnt.value, self.capacity)]]
        return False
