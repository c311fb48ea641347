"""§8(f) NEXT-2: GPU split-step channel generator vs the oracle channel (oracle/channel.py:
Kerr with L_eff at each segment start, lossy dispersion, EDFA gain + ASE, brick-wall LPF +
decimation; §IV-A) on the same inputs and ASE draws.

Tolerance from the arithmetic: fp32 radix-2 FFTs with exact twiddles err ~ log2(n) 2^-24 per
transform; 2 transforms per step, errors add as a random walk, so
tol = 10 * sqrt(2 * spans * steps) * log2(n) * 2^-24 (<= 1e-4 for the cases below), rel-L2 per block.
"""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import channel, physics, steps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2010_14258_b200 as P

    return P


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def link_params(rho_a=4):
    a = physics.alpha_np_per_km(0.2)
    return dict(alpha_np=a, beta2=physics.ps2_per_km(-21.7), gamma=1.3, fs_hz=rho_a * 10.7e9,
                span_km=80.0, ase_sigma=float(np.sqrt(physics.ase_psd(5.0, a, 80.0, 1.946e14) * rho_a * 10.7e9)))


def tol(spans, S, n):
    return 10 * np.sqrt(2 * spans * S) * np.log2(n) * 2.0 ** -24


@pytest.mark.parametrize("B,nsym,spans,S,decim,noisy,pdbm", [
    (2, 256, 2, 10, 0, True, 5.0),    # two spans, ASE, 5 dBm (nonlinear)
    (3, 512, 3, 6, 2, True, 2.0),     # LPF + decimation to 2 sps (rho_a = 4)
    (1, 4096, 1, 5, 0, False, 8.0),   # n = 16384, the maximum
])
def test_ssfm_link_parity(P, B, nsym, spans, S, decim, noisy, pdbm):
    rho_a = 4
    n = nsym * rho_a
    prm = link_params(rho_a)
    pw = float(li.dbm_to_w(pdbm))
    s = np.stack([li.qam16(li.rng(71, b, "symbols"), nsym) for b in range(B)])
    x = np.stack([channel.modulate(s[b], rho_a, pw) for b in range(B)])
    deltas = steps.log_step_sizes(prm["span_km"], S, prm["alpha_np"])
    noise = np.stack([li.cn(li.rng(71, 0, "ase", sub=k), (B, n)) for k in range(spans)]) if noisy else None
    # oracle on the fp32-rounded input and draws
    u = x.astype(np.complex64).astype(np.complex128)
    nz = None if noise is None else noise.astype(np.complex64).astype(np.complex128)
    psd = prm["ase_sigma"] ** 2 / prm["fs_hz"]
    for k in range(spans):
        u = channel.ssfm(u, deltas, prm["alpha_np"], prm["beta2"], prm["gamma"], prm["fs_hz"])
        u = channel.edfa(u, prm["alpha_np"], prm["span_km"], psd, prm["fs_hz"], None if nz is None else nz[k])
    if decim:
        ref = np.stack([channel.lowpass_decimate(u[b], rho_a, rho_a // decim) for b in range(B)])
    else:
        ref = u
    ut = torch.from_numpy(x.astype(np.complex64)).cuda()
    nt = None if noise is None else torch.from_numpy(noise.astype(np.complex64)).cuda()
    out = P.ldbp_ssfm_link(ut, deltas, spans=spans, span_km=prm["span_km"], alpha_np=prm["alpha_np"],
                           beta2=prm["beta2"], gamma=prm["gamma"], fs_hz=prm["fs_hz"],
                           ase_sigma=prm["ase_sigma"] if noisy else 0.0, noise=nt, decim=decim,
                           cutoff=(rho_a // max(decim, 1)) / (2.0 * rho_a) if decim else 0.5)
    out = out.cpu().numpy().astype(np.complex128)
    t = tol(spans, S, n)
    assert t <= 1e-4
    for b in range(B):
        assert rel(out[b], ref[b]) <= t, (b, rel(out[b], ref[b]), t)


@pytest.mark.parametrize("B,nsym,spans,S,decim,block0,pdbm", [
    (2, 8192, 2, 4, 2, 0, 4.0),      # n = 2^15 (2-CTA cluster), LPF + decimation (C2-C4 block size)
    (1, 16384, 1, 3, 2, 5, 6.0),     # n = 2^16 (4-CTA cluster), global block index 5 (C5 block size)
    (2, 1024, 2, 4, 0, 7, 3.0),      # single CTA, keyed draws
])
def test_ssfm_link_cluster_and_philox_ase(P, B, nsym, spans, S, decim, block0, pdbm):
    """Blocks longer than one CTA's shared memory (cluster four-step DFT over distributed shared
    memory) and ASE drawn inside the kernel by the counter-based generator, against the oracle
    channel fed ldbp_inputs.ase_cn_philox — the same Philox4x32-10 draws in numpy."""
    rho_a = 4
    n = nsym * rho_a
    prm = link_params(rho_a)
    pw = float(li.dbm_to_w(pdbm))
    seed = 201014258
    s = np.stack([li.qam16(li.rng(72, b, "symbols"), nsym) for b in range(B)])
    x = np.stack([channel.modulate(s[b], rho_a, pw) for b in range(B)])
    deltas = steps.log_step_sizes(prm["span_km"], S, prm["alpha_np"])
    u = x.astype(np.complex64).astype(np.complex128)
    psd = prm["ase_sigma"] ** 2 / prm["fs_hz"]
    for k in range(spans):
        u = channel.ssfm(u, deltas, prm["alpha_np"], prm["beta2"], prm["gamma"], prm["fs_hz"])
        nz = np.stack([li.ase_cn_philox(seed, block0 + b, k, n) for b in range(B)])
        u = channel.edfa(u, prm["alpha_np"], prm["span_km"], psd, prm["fs_hz"], nz)
    ref = np.stack([channel.lowpass_decimate(u[b], rho_a, rho_a // decim) for b in range(B)]) if decim else u
    ut = torch.from_numpy(x.astype(np.complex64)).cuda()
    out = P.ldbp_ssfm_link(ut, deltas, spans=spans, span_km=prm["span_km"], alpha_np=prm["alpha_np"],
                           beta2=prm["beta2"], gamma=prm["gamma"], fs_hz=prm["fs_hz"], ase_sigma=prm["ase_sigma"],
                           ase_seed=seed, block0=block0, decim=decim,
                           cutoff=(rho_a // max(decim, 1)) / (2.0 * rho_a) if decim else 0.5)
    out = out.cpu().numpy().astype(np.complex128)
    t = tol(spans, S, n) + 1e-6  # + the fp32 Box-Muller of the draws (relative ~1e-7 per draw)
    for b in range(B):
        assert rel(out[b], ref[b]) <= t, (b, rel(out[b], ref[b]), t)


def test_ssfm_philox_draws_shard_invariant(P):
    """The keyed in-kernel draws depend only on the global block index: blocks [0, 4) in one call
    equal blocks [0, 2) + [2, 4) (block0 = 2) in two calls, bit for bit."""
    rho_a, nsym, spans, S = 4, 1024, 2, 3
    n = nsym * rho_a
    prm = link_params(rho_a)
    s = np.stack([li.qam16(li.rng(73, b, "symbols"), nsym) for b in range(4)])
    x = torch.from_numpy(np.stack([channel.modulate(s[b], rho_a, 1e-3) for b in range(4)]).astype(np.complex64)).cuda()
    deltas = steps.log_step_sizes(prm["span_km"], S, prm["alpha_np"])
    kw = dict(spans=spans, span_km=prm["span_km"], alpha_np=prm["alpha_np"], beta2=prm["beta2"], gamma=prm["gamma"],
              fs_hz=prm["fs_hz"], ase_sigma=prm["ase_sigma"], ase_seed=9)
    full = P.ldbp_ssfm_link(x.clone(), deltas, block0=0, **kw).cpu()
    a = P.ldbp_ssfm_link(x[:2].clone(), deltas, block0=0, **kw).cpu()
    b = P.ldbp_ssfm_link(x[2:].clone(), deltas, block0=2, **kw).cpu()
    assert torch.equal(torch.cat([a, b]), full)
